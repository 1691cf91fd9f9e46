out=gpurun_out/r2b; mkdir -p $out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
bash tools/gpu_sanitize.sh r2b_san > /dev/null 2>&1
bash tools/fclk.sh r2b_fclk
