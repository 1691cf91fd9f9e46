#!/bin/bash
# Round-2 GPU call: GPU tests, bench (C3 default), the C3 trace, the reference arm,
# and an ncu launch list of a C3 solve.  Usage: bash tools/gpu_r2.sh <tag> [skip_tests]
tag=${1:-r2a}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1; nproc > $out/nproc.txt; lscpu | grep "Model name" >> $out/nproc.txt
if [ -z "$2" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
fi
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench exit $?" >> $out/bench.err
AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter4097 > $out/trace.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
    --log-file $out/launches.csv python tools/prof_one.py jitter4097 1 > $out/launches.log 2>&1
python tools/launch_summary.py $out/launches.csv by_grid > $out/launches_by_grid.txt 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
echo done
