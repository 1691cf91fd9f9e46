out=gpurun_out/r2zy; mkdir -p $out
FULL="index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
SMI_Q=off timeout 300 python tools/stall_probe.py jitter4097 20 > $out/off.log 2>&1
SMI_Q=$FULL SMI_MS=200 timeout 300 python tools/stall_probe.py jitter4097 20 > $out/full.log 2>&1
SMI_Q=clocks.sm SMI_MS=200 timeout 300 python tools/stall_probe.py jitter4097 20 > $out/sm.log 2>&1
SMI_Q=clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap SMI_MS=200 timeout 300 python tools/stall_probe.py jitter4097 20 > $out/reasons.log 2>&1
SMI_Q=power.draw SMI_MS=200 timeout 300 python tools/stall_probe.py jitter4097 20 > $out/power.log 2>&1
SMI_Q=clocks.max.sm SMI_MS=200 timeout 300 python tools/stall_probe.py jitter4097 20 > $out/max.log 2>&1
