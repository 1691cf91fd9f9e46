out=gpurun_out/r2i; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py tests/test_gpu_boundary.py -x -q -m gpu -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter4097 graded2049 > $out/trace.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_bgs_inv -c 16 --csv --log-file $out/bgs.csv python tools/prof_one.py jitter4097 1 > $out/ncu.log 2>&1
python tools/launch_summary.py $out/bgs.csv by_grid > $out/bgs_by_grid.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_bgs_inv -c 16 --csv --log-file $out/bgs_c2.csv python tools/prof_one.py graded2049 1 > $out/ncu2.log 2>&1
python tools/launch_summary.py $out/bgs_c2.csv by_grid > $out/bgs_c2_by_grid.txt 2>&1
