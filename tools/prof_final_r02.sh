# round-2 closing run, part 2: launch list + ncu --set full of every n; summarised ON the box (the .ncu-rep
# files together exceed gpurun's 64 MiB copy-back), only the headline kernel's report is kept
TAG=r02
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-per-n --no-cpu-baseline --no-mc \
  > gpurun_out/launches_${TAG}.log 2>&1
common="--steps 2 --warmup 3 --no-per-n --no-cpu-baseline --no-e2e --no-mc"
cap() { timeout 600 $NCU --set full --clock-control none --import-source on -k regex:qed_ -s 3 -c 1 -o gpurun_out/full_${TAG}_$1 -f python bench.py $2 $common > gpurun_out/full_${TAG}_$1.log 2>&1; }
cap n1 "--n 1"
cap n2 "--n 2"
cap n3 "--n 3 --points 2097152"
cap n4 "--n 4 --points 1048576"
cap n5 "--n 5 --points 262144"
cap bg2 "--n 2 --algorithm bg"
cap bg5 "--n 5 --points 1048576 --algorithm bg"
python tools/summarize_profiles.py $TAG > gpurun_out/summarize_${TAG}.log 2>&1
mkdir -p gpurun_out/prof_${TAG}
cp profiles/${TAG}/* gpurun_out/prof_${TAG}/; cp profiles/ncu_traffic.json gpurun_out/prof_${TAG}/
for r in gpurun_out/full_${TAG}_*.ncu-rep; do b=$(basename $r .ncu-rep); python tools/ncu_lines.py $r 30 > gpurun_out/prof_${TAG}/lines_${b#full_${TAG}_}.txt 2>&1; done
for r in gpurun_out/full_${TAG}_*.ncu-rep; do [ "$r" = "gpurun_out/full_${TAG}_n2.ncu-rep" ] || rm -f $r; done
du -sh gpurun_out
