out=gpurun_out/r3g; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster16.py -x -q -m gpu -p no:cacheprovider > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
bash tools/ab.sh r3g_ab jitter1025 graded2049 jitter4097 > $out/ab.txt 2>&1
