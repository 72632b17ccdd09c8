timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/racecheck_full.log 2>&1; echo "rc=$?" >> gpurun_out/racecheck_full.log
timeout 600 python -m pytest tests/test_mc.py -m gpu -x -q > gpurun_out/r47_tests.log 2>&1; echo rc=$? >> gpurun_out/r47_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-per-n --no-cpu-baseline --no-e2e > gpurun_out/bench_r47.json 2>gpurun_out/bench_r47.err
