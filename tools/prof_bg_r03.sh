NCU=/usr/local/cuda/bin/ncu
common="--steps 1 --warmup 3 --no-per-n --no-cpu-baseline --no-e2e --no-mc --no-configs"
cap() { timeout 600 $NCU --set full --clock-control none --import-source on -k regex:qed_eval -s 3 -c 1 -o gpurun_out/p_$1 -f python bench.py $2 $common > gpurun_out/p_$1.log 2>&1;
  python tools/ncu_lines_wf.py gpurun_out/p_$1.ncu-rep 40 > gpurun_out/lineswf_$1.txt 2>&1;
  python tools/ncu_sass_top.py gpurun_out/p_$1.ncu-rep > gpurun_out/sass_$1.txt 2>&1;
  $NCU -i gpurun_out/p_$1.ncu-rep --page raw --csv > gpurun_out/raw_$1.csv 2>&1; rm -f gpurun_out/p_$1.ncu-rep; }
cap bg3 "--n 3 --points 2097152 --algorithm bg"
cap bg4 "--n 4 --points 1048576 --algorithm bg"
cap bg5 "--n 5 --points 524288 --algorithm bg"
cap n3 "--n 3 --points 2097152"
