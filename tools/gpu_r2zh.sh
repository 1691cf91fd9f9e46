out=gpurun_out/r2zh; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_stream.py -x -q -m gpu -p no:cacheprovider > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
bash tools/ab.sh r2zh_ab jitter4097 graded2049 > $out/ab.txt 2>&1
