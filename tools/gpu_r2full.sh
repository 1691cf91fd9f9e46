out=gpurun_out/r2full; mkdir -p $out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cluster_pcg|k_c16_up|k_c16_down|k_bgs_inv\b" -s 40 -c 6 -o $out/full_c3 python tools/prof_one.py jitter4097 1 > $out/ncu.log 2>&1
ncu -i $out/full_c3.ncu-rep --page details --csv > $out/full_c3_details.csv 2>/dev/null
ncu -i $out/full_c3.ncu-rep --page raw --csv > $out/full_c3_raw.csv 2>/dev/null
