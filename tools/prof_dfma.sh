# ncu --set full of the DFMA peak microbenchmark (why it reads ~91 % of 148 SM x 64 DFMA/clk x f_SM)
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none -k regex:dfma_kernel -s 1 -c 1 -o gpurun_out/p_dfma -f \
  python -c "
import ctypes, os
lib = ctypes.CDLL(os.path.join('paper_2511_19456_b200', 'lib', 'libqed_peak.so'))
tf, ms = ctypes.c_double(), ctypes.c_double()
print(lib.qed_dfma_peak(4000, 8, ctypes.byref(tf), ctypes.byref(ms)), tf.value, ms.value)
" > gpurun_out/p_dfma.log 2>&1
$NCU -i gpurun_out/p_dfma.ncu-rep --page raw --csv > gpurun_out/raw_dfma.csv 2>&1
python tools/ncu_sass_top.py gpurun_out/p_dfma.ncu-rep > gpurun_out/sass_dfma.txt 2>&1
rm -f gpurun_out/p_dfma.ncu-rep
