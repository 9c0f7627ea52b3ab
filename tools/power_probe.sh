#!/bin/bash
# SM clock / power / throttle reasons sampled while a command runs (100 ms period).
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/power_$1.csv &
P=$!
shift
"$@"
kill $P
