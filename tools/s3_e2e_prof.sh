timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" > gpurun_out/s3b_hosttests.log 2>&1; echo "rc=$?" >> gpurun_out/s3b_hosttests.log
timeout 600 python bench.py --no-per-n --no-cpu-baseline --no-mc --no-configs > gpurun_out/s3b_bench.json 2> gpurun_out/s3b_bench.err
bash tools/prof_s3.sh
