out=gpurun_out/r2z; mkdir -p $out
timeout 600 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --import-source on --clock-control none -k regex:k_bgs_inv -s 2 -c 2 -o $out/bgs python tools/prof_one.py jitter4097 1 > $out/ncu.log 2>&1
ncu -i $out/bgs.ncu-rep --page source --csv --print-source sass > $out/bgs_sass.csv 2>/dev/null
