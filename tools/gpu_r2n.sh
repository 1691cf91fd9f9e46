out=gpurun_out/r2n; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_cluster16.py -x -q -m gpu -p no:cacheprovider -k "jitter_129" > $out/c16_first.log 2>&1; echo "exit $?" >> $out/c16_first.log
timeout 900 python -m pytest tests/test_gpu_cluster16.py -x -q -m gpu -p no:cacheprovider > $out/c16.log 2>&1; echo "exit $?" >> $out/c16.log
for rep in 1 2; do
for c in 1 0; do
  C16=$c AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter4097 graded2049 > $out/qp_c16_$c.$rep.log 2>&1
  echo "c16=$c rep $rep: $(grep -o 'coarse K-cycle (levels>=1) [0-9.]*' $out/qp_c16_$c.$rep.log | awk '{print $4}' | tail -4 | tr '\n' ' ')" >> $out/ab.txt
done
done
timeout 300 python bench.py > $out/bench.json 2> $out/bench.err
