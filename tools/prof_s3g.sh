# session-3 closing profile set (one GPU): launch list of the default bench command (no per_n / MC legs),
# ncu --set full of the headline kernel (n = 2, bench config) and of BG n = 3 (kept as .ncu-rep for the
# SASS-level L1 analysis here); reports above 28 MB are summarised on the box and deleted.
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_s3g.csv python bench.py --steps 3 --warmup 3 --no-per-n --no-cpu-baseline --no-mc --no-configs \
  > gpurun_out/launches_s3g.log 2>&1
common="--steps 2 --warmup 3 --no-per-n --no-cpu-baseline --no-e2e --no-mc --no-configs"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:qed_ -s 3 -c 1 \
  -o gpurun_out/full_s3g_n2 -f python bench.py --n 2 $common > gpurun_out/full_s3g_n2.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:qed_ -s 3 -c 1 \
  -o gpurun_out/full_s3g_bg3 -f python bench.py --n 3 --points 2097152 --algorithm bg $common > gpurun_out/full_s3g_bg3.log 2>&1
for r in n2 bg3; do
  $NCU -i gpurun_out/full_s3g_$r.ncu-rep --page raw --csv > gpurun_out/raw_s3g_$r.csv 2>&1
  python tools/ncu_sass_top.py gpurun_out/full_s3g_$r.ncu-rep > gpurun_out/sass_s3g_$r.txt 2>&1
  python tools/ncu_lines.py gpurun_out/full_s3g_$r.ncu-rep > gpurun_out/lines_s3g_$r.txt 2>&1
  $NCU -i gpurun_out/full_s3g_$r.ncu-rep --page source --csv --print-source sass > gpurun_out/srcsass_s3g_$r.csv 2>&1
  gzip -f gpurun_out/srcsass_s3g_$r.csv
  sz=$(stat -c %s gpurun_out/full_s3g_$r.ncu-rep); if [ "$sz" -gt 28000000 ]; then rm -f gpurun_out/full_s3g_$r.ncu-rep; fi
done
ls -la gpurun_out | grep s3g
