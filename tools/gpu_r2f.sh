out=gpurun_out/r2f; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q -m gpu -p no:cacheprovider > $out/pytest_stream.log 2>&1; echo "pytest exit $?" >> $out/pytest_stream.log
for cfg in "STREAM=-1" "STREAM=0" "STREAM=512" "STREAM=256" "STREAM=512 AUX_STREAM_PER_SM=1" "STREAM=512 AUX_STREAM_PER_SM=3"; do
  echo "== $cfg" >> $out/ab.txt
  env $cfg AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter4097 graded2049 > $out/qp.log 2>&1
  grep -E "device time|solve\[1\]" $out/qp.log | sed -n '3,4p;9,10p' >> $out/ab.txt
done
env STREAM=256 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_stream|k_tile" -c 80 --csv --log-file $out/stream_launches.csv python tools/prof_one.py jitter4097 1 > $out/ncu.log 2>&1
python tools/launch_summary.py $out/stream_launches.csv by_grid > $out/stream_by_grid.txt 2>&1
