#!/bin/bash
# Round-2 final evidence (C3): the bench line (with the CPU baseline), the reference arm, the launch list of a
# truncated learned solve, and ncu --set full captures of the tcgen05.shift convs (16 and 32 channels) and the
# 64 -> 64 wide conv inside that solve plus the residual-case level-0 conv alone.  Every capture runs after the
# same command exited 0 without ncu.
python bench.py > gpurun_out/r2g_bench.log 2>&1 || exit 1
tail -1 gpurun_out/r2g_bench.log | cut -c1-300
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2g_ref.log 2>&1; tail -1 gpurun_out/r2g_ref.log | cut -c1-300
python tools/step_probe.py --iters 6 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_launches_c3_learned.csv \
  python tools/step_probe.py --iters 6 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/r2g_launches_c3_learned.csv 2>&1 | head -24
ncu --set full --clock-control none --import-source on -k regex:"k_conv_shift<16" --launch-skip 4 -c 1 \
  -o gpurun_out/r2g_shift16 -f python tools/step_probe.py --iters 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_conv_shift<32" --launch-skip 4 -c 1 \
  -o gpurun_out/r2g_shift32 -f python tools/step_probe.py --iters 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_conv_wide<64, 64" --launch-skip 4 -c 1 \
  -o gpurun_out/r2g_wide6464 -f python tools/step_probe.py --iters 6 > /dev/null 2>&1
python tools/conv_probe.py --B 64 --H 512 --W 1024 --side residual --softplus 0 --iters 3 | tail -1
ncu --set full --clock-control none --import-source on -k regex:"k_conv_shift<16" --launch-skip 5 -c 1 \
  -o gpurun_out/r2g_shift16_resid -f python tools/conv_probe.py --B 64 --H 512 --W 1024 --side residual --softplus 0 --iters 3 > /dev/null 2>&1
python tools/cnn_probe.py --profile 2>&1 | tail -40 > gpurun_out/r2g_layers.txt
ls gpurun_out | grep r2g
