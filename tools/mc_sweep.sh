# MC leg (configs[3]: n = 4, 2^24 points) per launch variant: gpurun_out/mc_<tag>.jsonl
TAG=$1; ALGO=$2; shift 2
for v in "$@"; do
  QED_VARIANT=$v timeout 300 python bench.py --n 4 --algorithm $ALGO --points 1048576 --steps 3 --warmup 3 --no-per-n \
    --no-cpu-baseline --no-e2e --no-configs 2>>gpurun_out/mc_$TAG.err | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['mc']; print(json.dumps({'variant':$v,'algo':'$ALGO','bg':m['bg']['value'] if m.get('bg') else None,'cdag':m['cdag']['value'] if m.get('cdag') else None,'sigma':m['bg']['sigma']}))" >> gpurun_out/mc_$TAG.jsonl
done
