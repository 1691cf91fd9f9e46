out=gpurun_out/exp7; mkdir -p $out
for t in 512 1024; do
  make -C paper_1209_5421_b200/csrc -B -j32 NVEXTRA=-DAUX_FUSED_THREADS=$t > $out/build$t.log 2>&1
  AUX_TRACE=1 timeout 300 python tools/quick_perf.py graded2049 jitter1025 > $out/t$t.log 2>&1
done
make -C paper_1209_5421_b200/csrc -B -j32 > $out/build.log 2>&1
AUX_TRACE=1 timeout 300 python tools/quick_perf.py graded2049 jitter1025 > $out/t256.log 2>&1
