#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (N=1), launch list + ncu --set full of the top kernels.
# Usage (from the repo root on the GPU box):  bash tools/gpu_round.sh [tag]
tag=${1:-r1}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench exit $?" >> $out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file $out/launches.csv python tools/prof_one.py graded2049 2 > $out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_csr_spmv|k_rows|k_bgs_solve' -s 6 -c 6 \
    -o $out/prof python tools/prof_one.py graded2049 2 > $out/prof.log 2>&1
echo done
