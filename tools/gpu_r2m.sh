out=gpurun_out/r2m; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -m gpu -p no:cacheprovider -k "solve_parity or setup_exports or mgs or medium or block or errors or parts_match" > $out/pytest_quick.log 2>&1; echo "pytest exit $?" >> $out/pytest_quick.log
bash tools/ab.sh r2m_ab jitter4097 graded2049 > $out/ab.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_bgs_inv -c 16 --csv --log-file $out/bgs_c3.csv python tools/prof_one.py jitter4097 1 > $out/ncu.log 2>&1
python tools/launch_summary.py $out/bgs_c3.csv by_grid > $out/bgs_c3_by_grid.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_bgs_inv -c 16 --csv --log-file $out/bgs_c2.csv python tools/prof_one.py graded2049 1 > $out/ncu2.log 2>&1
python tools/launch_summary.py $out/bgs_c2.csv by_grid > $out/bgs_c2_by_grid.txt 2>&1
