out=gpurun_out/exp8; mkdir -p $out
for t in 256 128 64; do AUX_TILE16_MIN=$t AUX_TRACE=1 timeout 300 python tools/quick_perf.py graded2049 > $out/t$t.log 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > $out/full.log 2>&1; echo "exit $?" >> $out/full.log
