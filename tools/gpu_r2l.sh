out=gpurun_out/r2l; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_stream.py tests/test_runner.py tests/test_dropin.py -q -m gpu -p no:cacheprovider > $out/pytest_dist.log 2>&1; echo "pytest exit $?" >> $out/pytest_dist.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bgs_inv" -s 2 -c 2 -o $out/prof_bgs python tools/prof_one.py jitter4097 1 > $out/prof_bgs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream_up|k_stream_down" -s 0 -c 2 -o $out/prof_stream python tools/prof_one.py jitter4097 1 > $out/prof_stream.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -c "
import sys; sys.path.insert(0,'.')
from paper_1209_5421_b200 import api, problems
s = problems.jittered_p1(129)
r = api.solve(s.A, s.b, api.setup_hierarchy(s.A, s.coords, gpu=api.GpuOptions(stream_min_width=16)))
print('stream kernels', r.iterations, r.converged)
u, res, _ = api.solve_parts(s.A, s.coords, s.b, 2, gpu=api.GpuOptions(stream_min_width=32))
print('parts', res[0].iterations)
" > $out/san_${tool}_stream.log 2>&1; echo "$tool exit $?" >> $out/san_summary.txt
done
