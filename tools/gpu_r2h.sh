out=gpurun_out/r2h; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py -x -q -m gpu -p no:cacheprovider -k "cluster or tile or solve_parity or cycle_options or stream or medium" > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
bash tools/ab.sh r2h_ab jitter4097 graded2049 jitter1025 > $out/ab.txt 2>&1
