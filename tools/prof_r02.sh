NCU=/usr/local/cuda/bin/ncu
common="--steps 2 --warmup 3 --no-per-n --no-cpu-baseline --no-e2e --no-mc"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:qed_ -s 3 -c 1 -o gpurun_out/full_r02_n1 -f python bench.py --n 1 $common > gpurun_out/full_r02_n1.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:qed_ -s 3 -c 1 -o gpurun_out/full_r02_n3 -f python bench.py --n 3 --points 2097152 $common > gpurun_out/full_r02_n3.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:qed_ -s 3 -c 1 -o gpurun_out/full_r02_n4 -f python bench.py --n 4 --points 1048576 $common > gpurun_out/full_r02_n4.log 2>&1
