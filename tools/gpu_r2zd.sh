out=gpurun_out/r2zd; mkdir -p $out
timeout 2400 python -m pytest tests -x -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "exit $?" >> $out/smoke.log
timeout 400 python bench.py > $out/bench_c3.json 2> $out/bench_c3.err
timeout 400 python bench.py --config c2 > $out/bench_c2.json 2> $out/bench_c2.err
AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter4097 graded2049 jitter1025 > $out/trace.txt 2>&1
