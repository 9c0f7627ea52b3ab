#!/bin/bash
# Round-2 evidence refresh (C3): the bench line, the launch list of a truncated learned solve, and ncu --set full
# captures of the roofline kernel class (wide conv) and of the level-0 tcgen05 conv inside that solve.
python bench.py > gpurun_out/r2f_bench.log 2>&1 || exit 1
tail -1 gpurun_out/r2f_bench.log | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches_c3_learned.csv \
  python tools/step_probe.py --iters 6 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/r2f_launches_c3_learned.csv 2>&1 | head -30
ncu --set full --clock-control none --import-source on -k regex:"k_conv_wide<64, 64" --launch-skip 4 -c 1 \
  -o gpurun_out/r2f_wide6464 -f python tools/step_probe.py --iters 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_conv_tc<16, 16" --launch-skip 4 -c 1 \
  -o gpurun_out/r2f_tc1616 -f python tools/step_probe.py --iters 6 > /dev/null 2>&1
ls gpurun_out | grep r2f
