out=gpurun_out/r2final; mkdir -p $out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
for c in c3 c2 c1 c4 c5; do timeout 600 python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref_c3.json 2> $out/bench_ref_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
    --log-file $out/launches_c3.csv python tools/prof_one.py jitter4097 1 > $out/ncu_c3.log 2>&1
python tools/launch_summary.py $out/launches_c3.csv by_grid > $out/launches_c3_by_grid.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
    --log-file $out/launches_c2.csv python tools/prof_one.py graded2049 1 > $out/ncu_c2.log 2>&1
python tools/launch_summary.py $out/launches_c2.csv by_grid > $out/launches_c2_by_grid.txt 2>&1
AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter4097 graded2049 jitter1025 > $out/trace.txt 2>&1
