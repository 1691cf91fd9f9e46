out=gpurun_out/r3i; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "solve_parity or medium or tile" > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
for rep in 1 2; do for rr in 1 0; do for cfg in jitter4097 graded2049; do
  AUX_ROWS_RESTRICT=$rr AUX_TRACE=1 timeout 300 python tools/quick_perf.py $cfg > $out/rr$rr.$cfg.$rep.log 2>&1
done; done; done
