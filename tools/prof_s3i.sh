# closing profile set after the per-spin ubar specialisation (one GPU): launch list of the bench command and
# ncu --set full of the headline kernel
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_s3i.csv python bench.py --steps 3 --warmup 3 --no-per-n --no-cpu-baseline --no-mc --no-configs \
  > gpurun_out/launches_s3i.log 2>&1
common="--steps 2 --warmup 3 --no-per-n --no-cpu-baseline --no-e2e --no-mc --no-configs"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:qed_ -s 3 -c 1 \
  -o gpurun_out/full_s3i_n2 -f python bench.py --n 2 $common > gpurun_out/full_s3i_n2.log 2>&1
$NCU -i gpurun_out/full_s3i_n2.ncu-rep --page raw --csv > gpurun_out/raw_s3i_n2.csv 2>&1
python tools/ncu_lines.py gpurun_out/full_s3i_n2.ncu-rep > gpurun_out/lines_s3i_n2.txt 2>&1
ls -la gpurun_out | grep s3i
