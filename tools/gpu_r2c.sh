out=gpurun_out/r2c; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -x -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
bash tools/ab.sh r2c_ab jitter4097 graded2049 > $out/ab.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-weak-base > $out/bench.json 2> $out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_bgs_inv -c 16 --csv --log-file $out/bgs_launches.csv python tools/prof_one.py jitter4097 1 > $out/ncu.log 2>&1
