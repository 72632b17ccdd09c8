#!/bin/bash
# Launch-variant sweep (run under gpurun): one bench line per (n, variant) -> gpurun_out/sweep_<tag>.jsonl
TAG=${1:-r01}
OUT=gpurun_out/sweep_${TAG}.jsonl
mkdir -p gpurun_out; : > $OUT
run() { n=$1; P=$2; v=$3
  QED_VARIANT=$v timeout 300 python bench.py --n $n --points $P --steps 10 --warmup 3 --no-per-n --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'n':$n,'variant':$v,'value':d['value'],'frac':d['roofline']['frac'],'sm_mhz':d['clocks']['sm_mhz']}))" >> $OUT
}
for v in 0 1 2 3 4; do run 2 4194304 $v; done
for v in 0 1 2 3 4; do run 1 4194304 $v; done
for v in 0 1 2; do run 3 2097152 $v; done
for v in 0 1 2; do run 4 1048576 $v; done
for v in 0 1 2; do run 5 262144 $v; done
cat $OUT
