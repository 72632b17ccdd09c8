bash tools/prof_var.sh m3 3 cdag 0 2097152
bash tools/prof_var.sh m4 4 cdag 0 1048576
bash tools/prof_var.sh m5 5 cdag 0 262144
bash tools/prof_var.sh b3 3 bg 0 2097152
