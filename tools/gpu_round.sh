#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (N=1, with the reference's CPU baseline), the
# reference arm, an ncu launch list and ncu --set full captures of the dominant kernels.
# Usage (from the repo root on the GPU box):  bash tools/gpu_round.sh [tag]
tag=${1:-r1}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench exit $?" >> $out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
AUX_TRACE=1 timeout 300 python tools/quick_perf.py graded2049 jitter1025 > $out/trace.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $out/launches.csv python tools/prof_one.py graded2049 2 > $out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_bgs_inv|k_csr_spmv|k_tile_up|k_cluster_pcg|k_fused_pcg|k_mgs' -s 20 -c 10 \
    -o $out/prof python tools/prof_one.py graded2049 2 > $out/prof.log 2>&1
echo done
