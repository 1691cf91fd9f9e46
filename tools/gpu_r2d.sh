out=gpurun_out/r2d; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q -m gpu -p no:cacheprovider > $out/pytest_stream.log 2>&1; echo "pytest exit $?" >> $out/pytest_stream.log
for cfg in "STREAM=-1" "STREAM=0" "STREAM=512" "STREAM=256" "STREAM=512 AUX_STREAM_PER_SM=4" "STREAM=512 AUX_STREAM_PER_SM=1"; do
  echo "== $cfg" >> $out/ab.txt
  env $cfg AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter4097 graded2049 > $out/qp.log 2>&1
  grep -E "device time|solve\[1\]" $out/qp.log | tail -4 >> $out/ab.txt
done
STREAM=512 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_stream|k_tile" -c 60 --csv --log-file $out/stream_launches.csv python tools/prof_one.py jitter4097 1 > $out/ncu.log 2>&1
python tools/launch_summary.py $out/stream_launches.csv by_grid > $out/stream_by_grid.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -m gpu -p no:cacheprovider > $out/pytest_parity.log 2>&1; echo "pytest exit $?" >> $out/pytest_parity.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bgs_inv|k_stream_up|k_stream_down" -s 2 -c 4 -o $out/prof STREAM=256 python tools/prof_one.py jitter2049 1 > $out/prof.log 2>&1
