out=gpurun_out/r2s; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_cluster16.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
bash tools/ab.sh r2s_ab jitter4097 graded2049 jitter1025 > $out/ab.txt 2>&1
for c in 1 0; do C16=$c AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter4097 > $out/qp_c16_$c.log 2>&1; done
