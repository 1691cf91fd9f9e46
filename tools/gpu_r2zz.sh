out=gpurun_out/r2zz; mkdir -p $out
FULL="index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
for i in 1 2 3 4; do SMI_Q=$FULL SMI_MS=500 SMI_WAIT=0.15 timeout 300 python tools/stall_probe.py jitter4097 8 > $out/w015_$i.log 2>&1; done
for i in 1 2 3 4; do SMI_Q=$FULL SMI_MS=500 SMI_WAIT=1.5 timeout 300 python tools/stall_probe.py jitter4097 8 > $out/w150_$i.log 2>&1; done
