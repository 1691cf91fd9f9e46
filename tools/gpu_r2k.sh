out=gpurun_out/r2k; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "solve_parity or setup_exports or mgs or medium" > $out/pytest_quick.log 2>&1; echo "pytest exit $?" >> $out/pytest_quick.log
bash tools/ab.sh r2k_ab jitter4097 graded2049 > $out/ab.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
    --log-file $out/launches_c3.csv python tools/prof_one.py jitter4097 1 > $out/ncu_c3.log 2>&1
python tools/launch_summary.py $out/launches_c3.csv by_grid > $out/launches_c3_by_grid.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
    --log-file $out/launches_c2.csv python tools/prof_one.py graded2049 1 > $out/ncu_c2.log 2>&1
python tools/launch_summary.py $out/launches_c2.csv by_grid > $out/launches_c2_by_grid.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench exit $?" >> $out/bench.err
