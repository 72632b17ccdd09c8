#!/bin/bash
# Profiling pass on one GPU (run under gpurun).  Writes gpurun_out/{launches_*.csv, prof_*.ncu-rep}.
# usage: tools/profile.sh TAG [N POINTS]...
TAG=${1:-r01}; shift
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
# launch list of the default bench command (cold-cache, serialised: compare shares)
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 2 --no-per-n --no-cpu-baseline \
  > gpurun_out/launches_${TAG}.log 2>&1
while [ $# -ge 2 ]; do
  N=$1; P=$2; shift 2
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:qed_eval_kernel -s 2 -c 1 \
    -o gpurun_out/prof_${TAG}_n${N} -f python bench.py --n $N --points $P --steps 2 --warmup 2 --no-per-n \
    --no-cpu-baseline > gpurun_out/prof_${TAG}_n${N}.log 2>&1
done
ls -la gpurun_out
