#!/bin/bash
# usage: tools/clocks.sh <outfile> <cmd...>: sample nvidia-smi clocks while running cmd
out=$1; shift
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 100 > "$out" &
pid=$!
"$@"
rc=$?
kill $pid
exit $rc
