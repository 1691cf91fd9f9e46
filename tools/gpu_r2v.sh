out=gpurun_out/r2v; mkdir -p $out
timeout 2400 python -m pytest tests -x -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "exit $?" >> $out/smoke.log
timeout 400 python bench.py > $out/bench.json 2> $out/bench.err
