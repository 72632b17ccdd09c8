# one tuning iteration on the GPU box: parity over every compiled launch variant, then a sweep
# usage: bash tools/gpu_iter.sh TAG "sweep spec"
TAG=$1; SPEC=$2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "every_launch_variant" > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
bash tools/sweep.sh $TAG "$SPEC" > /dev/null 2>&1
