#!/bin/bash
# A/B of alternative library builds on the finest-level phases (AUX_TRACE):
#   bash tools/ab_finest.sh <tag>  -> gpurun_out/<tag>/<variant>.<rep>.log
tag=$1; out=gpurun_out/$tag; mkdir -p $out
for rep in 1 2; do for v in paper_1209_5421_b200/csrc/build/var/*.so; do n=$(basename $v .so)
  AUX_B200_LIB=$PWD/$v AUX_TRACE=1 timeout 300 python tools/quick_perf.py graded2049 jitter4097 > $out/$n.$rep.log 2>&1
  echo "$n rep $rep: $(grep -o 'finest pre-smooth+restrict [0-9.]*\|finest prolong+post-smooth [0-9.]*\|outer A z + MGS + update [0-9.]*' $out/$n.$rep.log | awk '{print $NF}' | tr '\n' ' ')"
done; done
