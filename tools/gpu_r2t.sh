out=gpurun_out/r2t; mkdir -p $out
timeout 600 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --import-source on --clock-control none -k regex:k_cluster_pcg -s 4 -c 3 -o $out/cluster2 python tools/prof_one.py jitter1025 1 > $out/ncu2.log 2>&1
ncu -i $out/cluster2.ncu-rep --page source --csv --print-source sass > $out/cluster2_sass.csv 2>/dev/null
ncu -i $out/cluster2.ncu-rep --page source --csv --print-source cuda > $out/cluster2_cuda.csv 2>/dev/null
