out=gpurun_out/r2zv; mkdir -p $out
for rep in 1 2; do
for cfg in "a_cur 2" "str_minb3 2" "str_minb3 3"; do
  set -- $cfg
  AUX_STREAM_PER_SM=$2 AUX_B200_LIB=$PWD/paper_1209_5421_b200/csrc/build/var/$1.so AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter4097 > $out/$1_$2.$rep.log 2>&1
  echo "$1 per_sm=$2 rep $rep: $(grep -o 'coarse K-cycle (levels>=1) [0-9.]*' $out/$1_$2.$rep.log | awk '{print $4}' | tail -3 | tr '\n' ' ')" >> $out/ab.txt
done
done
