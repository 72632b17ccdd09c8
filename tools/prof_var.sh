# ncu --set full of one (n, algorithm, variant) bench kernel, summarised on the box
# usage: bash tools/prof_var.sh TAG N ALGO VARIANT POINTS
TAG=$1; N=$2; ALGO=$3; V=$4; P=$5
NCU=/usr/local/cuda/bin/ncu
QED_VARIANT=$V timeout 600 $NCU --set full --clock-control none --import-source on -k regex:qed_eval -s 3 -c 1 -o gpurun_out/p_$TAG -f \
  python bench.py --n $N --points $P --algorithm $ALGO --steps 1 --warmup 3 --no-per-n --no-cpu-baseline --no-e2e --no-mc --no-configs > gpurun_out/p_$TAG.log 2>&1
python tools/ncu_lines_wf.py gpurun_out/p_$TAG.ncu-rep 40 > gpurun_out/lineswf_$TAG.txt 2>&1
python tools/ncu_sass_top.py gpurun_out/p_$TAG.ncu-rep > gpurun_out/sass_$TAG.txt 2>&1
$NCU -i gpurun_out/p_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>&1
rm -f gpurun_out/p_$TAG.ncu-rep
