#!/bin/bash
# ncu --set full captures for profiles/ (after round_profile4.sh ran the same commands without ncu)
cap() {  # name, kernel regex, skip, command...
  local name=$1 rx=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$rx" --launch-skip $skip -c 1 \
    -o gpurun_out/$name -f "$@" > gpurun_out/$name.log 2>&1
  tail -2 gpurun_out/$name.log
}
cap r2g_shift16 'k_conv_shift<.int.16>' 4 python tools/step_probe.py --iters 6
cap r2g_shift32 'k_conv_shift<.int.32>' 4 python tools/step_probe.py --iters 6
cap r2g_wide6464 'k_conv_wide<.int.64, .int.64' 4 python tools/step_probe.py --iters 6
cap r2g_shift_s2 'k_conv_shift_s2' 2 python tools/step_probe.py --iters 6
cap r2g_shift_t32 'k_conv_shift_t<.int.32>' 2 python tools/step_probe.py --iters 6
cap r2g_shift_t64 'k_conv_shift_t<.int.64>' 2 python tools/step_probe.py --iters 6
cap r2g_shift16_resid 'k_conv_shift<.int.16>' 5 python tools/conv_probe.py --B 64 --H 512 --W 1024 --side residual --softplus 0 --iters 3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_launches_c3_learned.csv python tools/step_probe.py --iters 6 > /dev/null 2>&1
ls -la gpurun_out | grep -E 'r2g|r2l'
