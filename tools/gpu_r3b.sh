out=gpurun_out/r3b; mkdir -p $out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
FULL="index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
for i in 1 2 3 4 5 6; do AUX_HOSTCALL_TRACE=2 SMI_Q=$FULL SMI_MS=200 SMI_WAIT=0.15 timeout 300 python tools/stall_probe.py jitter4097 10 > $out/p_$i.log 2>&1; done
for i in 1 2 3; do timeout 400 python bench.py --no-cpu-baseline > $out/bench_c3_$i.json 2>/dev/null; done
