#!/bin/bash
# A/B timing of alternative library builds (paper_1209_5421_b200/csrc/build/var/*.so):
#   bash tools/ab.sh <tag> [configs...]   -> gpurun_out/<tag>/<variant>.log (AUX_TRACE breakdown)
tag=${1:-ab}; shift; out=gpurun_out/$tag; mkdir -p $out
cfgs=${@:-graded2049 jitter4097}
for rep in 1 2; do
for v in paper_1209_5421_b200/csrc/build/var/*.so; do
  n=$(basename $v .so)
  AUX_B200_LIB=$PWD/$v AUX_TRACE=1 timeout 300 python tools/quick_perf.py $cfgs > $out/$n.$rep.log 2>&1
  echo "$n rep $rep: $(grep -o 'coarse K-cycle (levels>=1) [0-9.]*' $out/$n.$rep.log | awk '{print $4}' | tail -4 | tr '\n' ' ')"
done
done
# clocked builds (AUX_FUSED_CLOCKS): per-phase cycle counts of the single-CTA kernel
for v in paper_1209_5421_b200/csrc/build/varclk/*.so; do
  [ -e "$v" ] || continue
  n=$(basename $v .so)
  AUX_B200_LIB=$PWD/$v timeout 300 python tools/prof_one.py graded2049 1 > $out/clk_$n.log 2>&1
done
