out=gpurun_out/exp2; mkdir -p $out
AUX_TRACE=1 timeout 300 python tools/quick_perf.py graded2049 > $out/fused.log 2>&1
AUX_BINV_SPLIT=1 AUX_TRACE=1 timeout 300 python tools/quick_perf.py graded2049 > $out/split.log 2>&1
AUX_BINV_SPLIT=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_rows|k_bgs_inv' -c 12 --csv --log-file $out/split.csv python tools/prof_one.py graded2049 1 > /dev/null 2>&1
