#!/bin/bash
# Iteration loop on the GPU box: GPU tests, trace breakdown, bench (no CPU baseline).
#   bash tools/gpu_iter.sh <tag> [pytest-k-expr]
tag=${1:-it}; out=gpurun_out/$tag; mkdir -p $out
if [ -n "$2" ]; then timeout 900 python -m pytest tests -x -q -m gpu -k "$2" > $out/pytest_gpu.log 2>&1;
else timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; fi
echo "pytest exit $?" >> $out/pytest_gpu.log
AUX_TRACE=1 timeout 300 python tools/quick_perf.py graded2049 jitter1025 > $out/trace.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
if [ -n "$NCU_K" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -s ${NCU_S:-4} -c ${NCU_C:-4} \
      -o $out/prof python tools/prof_one.py graded2049 2 > $out/prof.log 2>&1
fi
