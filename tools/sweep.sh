#!/bin/bash
# Launch-variant sweep (run under gpurun): one bench line per (n, variant) -> gpurun_out/sweep_<tag>.jsonl
# usage: tools/sweep.sh TAG "n:variants n:variants ..."   e.g. tools/sweep.sh r02 "2:0,1,2,3 5:0,1"
TAG=${1:-r01}
SPEC=${2:-"2:0,1,2,3,4 1:0,1,2,3,4 3:0,1,2 4:0,1,2 5:0,1,2"}
OUT=gpurun_out/sweep_${TAG}.jsonl
mkdir -p gpurun_out; : > $OUT
declare -A PTS=([1]=4194304 [2]=4194304 [3]=4194304 [4]=2097152 [5]=1048576 [6]=262144 [7]=65536 [8]=16384)
# item "n:variants" (CDAG) or "bgN:variants" (Berends-Giele)
for item in $SPEC; do
  key=${item%%:*}; vs=${item#*:}
  algo=cdag; n=$key
  if [[ $key == bg* ]]; then algo=bg; n=${key#bg}; fi
  for v in ${vs//,/ }; do
    QED_VARIANT=$v timeout 300 python bench.py --n $n --points ${PTS[$n]} --steps 10 --warmup 3 --no-per-n \
      --no-cpu-baseline --no-e2e --no-mc --no-configs --algorithm $algo 2>>gpurun_out/sweep_${TAG}.err | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'n':$n,'algorithm':'$algo','variant':$v,'value':d['value'],'frac':d['roofline']['frac'],'sm_mhz':d['clocks']['sm_mhz'],'kernel':d['config']['kernel']}))" >> $OUT
  done
done
cat $OUT
