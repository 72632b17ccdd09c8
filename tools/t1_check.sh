# n=1 one-thread-per-point variants: parity over every variant, then a timing sweep
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "every_launch_variant or n1 or 1-" > gpurun_out/t1_tests.log 2>&1
echo "rc=$?" >> gpurun_out/t1_tests.log
bash tools/sweep.sh t1 "1:0,5,6,7,8 2:0" > /dev/null 2>&1
