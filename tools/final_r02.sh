# round-2 closing run, part 1 (one GPU): full gpu tests, smoke, bench line, sanitizers
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_final.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
bash tools/sanitize.sh > gpurun_out/sanitize_final.txt 2>&1
