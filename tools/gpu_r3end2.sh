out=gpurun_out/r3end2; mkdir -p $out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 600 python bench.py > $out/bench_c3.json 2> $out/bench_c3.err
timeout 600 python bench.py --config c2 > $out/bench_c2.json 2> $out/bench_c2.err
