# Fused-kernel phase clocks (debug build): bash tools/fclk.sh <tag>
out=gpurun_out/${1:-fclk}; mkdir -p $out
make -C paper_1209_5421_b200/csrc -B -j32 NVEXTRA=-DAUX_FUSED_CLOCKS > $out/build.log 2>&1
timeout 300 python tools/prof_one.py graded2049 1 > $out/clocks.log 2>&1
make -C paper_1209_5421_b200/csrc -B -j32 > $out/build2.log 2>&1
