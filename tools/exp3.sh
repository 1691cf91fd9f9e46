out=gpurun_out/exp3; mkdir -p $out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $out/launches.csv python tools/prof_one.py graded2049 2 > /dev/null 2>&1
