out=gpurun_out/r2g; mkdir -p $out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench exit $?" >> $out/bench.err
AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter4097 graded2049 jitter1025 > $out/trace.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
    --log-file $out/launches.csv python tools/prof_one.py jitter4097 1 > $out/launches.log 2>&1
python tools/launch_summary.py $out/launches.csv by_grid > $out/launches_by_grid.txt 2>&1
