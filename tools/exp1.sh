out=gpurun_out/exp1; mkdir -p $out
for f in -1 256 64 0; do FUSED=$f AUX_TRACE=1 timeout 300 python tools/quick_perf.py graded2049 > $out/g_$f.log 2>&1; done
AUX_TRACE=1 timeout 600 python tools/quick_perf.py jitter4097 > $out/j4097.log 2>&1
AUX_TRACE=1 timeout 600 python tools/quick_perf.py jitter1025 > $out/j1025.log 2>&1
