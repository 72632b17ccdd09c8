# ncu --set full of the current default kernels (BG n = 3..6, CDAG n = 2 headline), summarised on the box
bash tools/prof_var.sh s3_bg3 3 bg 0 2097152
bash tools/prof_var.sh s3_bg4 4 bg 0 1048576
bash tools/prof_var.sh s3_bg5 5 bg 0 524288
bash tools/prof_var.sh s3_bg6 6 bg 0 131072
