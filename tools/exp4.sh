out=gpurun_out/exp4; mkdir -p $out
make -C paper_1209_5421_b200/csrc -B -j32 NVEXTRA=-DAUX_FUSED_CLOCKS > $out/build.log 2>&1
timeout 300 python tools/prof_one.py graded2049 1 > $out/clocks.log 2>&1
