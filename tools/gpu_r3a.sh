out=gpurun_out/r3a; mkdir -p $out
FULL="index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
for i in 1 2 3 4 5 6; do AUX_HOSTCALL_TRACE=2 SMI_Q=$FULL SMI_MS=200 SMI_WAIT=0.15 timeout 300 python tools/stall_probe.py jitter4097 10 > $out/p_$i.log 2>&1; done
