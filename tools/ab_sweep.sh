# A/B of two builds of libqed.so on one box (ab/libqed_old.so vs ab/libqed_new.so), default variants,
# alternating old/new twice: gpurun_out/ab_<tag>.jsonl
TAG=$1; SPEC=${2:-"3:0 4:0 5:0 bg3:0 bg4:0 bg5:0 bg6:0"}
LIB=paper_2511_19456_b200/lib/libqed.so
OUT=gpurun_out/ab_${TAG}.jsonl; : > $OUT
for rep in 1 2; do
  for which in old new; do
    cp ab/libqed_$which.so $LIB
    bash tools/sweep.sh ab_${TAG}_${which}_$rep "$SPEC" > /dev/null 2>&1
    sed "s/^{/{\"lib\": \"$which\", \"rep\": $rep, /" gpurun_out/sweep_ab_${TAG}_${which}_$rep.jsonl >> $OUT
  done
done
cp ab/libqed_new.so $LIB
cat $OUT
