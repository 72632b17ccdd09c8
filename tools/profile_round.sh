#!/bin/bash
# Round profile set (run under gpurun on ONE GPU): launch list of the default bench command and one
# `ncu --set full` capture of the timed kernel for the bench config (n=2, 2^22 points), n=5 CDAG and n=5 BG.
TAG=${1:-r01}
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-per-n --no-cpu-baseline --no-mc \
  > gpurun_out/launches_${TAG}.log 2>&1
common="--steps 2 --warmup 3 --no-per-n --no-cpu-baseline --no-e2e --no-mc"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:qed_ -s 3 -c 1 \
  -o gpurun_out/full_${TAG}_n2 -f python bench.py --n 2 $common > gpurun_out/full_${TAG}_n2.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:qed_ -s 3 -c 1 \
  -o gpurun_out/full_${TAG}_n5 -f python bench.py --n 5 --points 262144 $common > gpurun_out/full_${TAG}_n5.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:qed_ -s 3 -c 1 \
  -o gpurun_out/full_${TAG}_bg5 -f python bench.py --n 5 --points 1048576 --algorithm bg $common > gpurun_out/full_${TAG}_bg5.log 2>&1
ls -la gpurun_out | grep $TAG
