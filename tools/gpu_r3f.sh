out=gpurun_out/r3f; mkdir -p $out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_boundary.py tests/test_gpu_dist.py -x -q -m gpu -p no:cacheprovider > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
for rep in 1 2; do for v in a_head n_sync; do for cfg in jitter4097 graded2049; do
  AUX_B200_LIB=$PWD/paper_1209_5421_b200/csrc/build/var/$v.so timeout 300 python tools/step_probe.py $cfg > $out/$v.$cfg.$rep.log 2>&1
done; done; done
