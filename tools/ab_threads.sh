# A/B the fused kernel's CTA size (variants built by hand into the package dir)
for T in 128 256 512; do cp paper_1209_5421_b200/libauxamg_b200_f$T.so paper_1209_5421_b200/libauxamg_b200.so; echo T=$T; AUX_TRACE=1 timeout 300 python tools/quick_perf.py jitter1025 graded2049 2>&1 | grep "aux trace" | sed -n '2p;8p'; done
cp paper_1209_5421_b200/libauxamg_b200_cur.so paper_1209_5421_b200/libauxamg_b200.so
