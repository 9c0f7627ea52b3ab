#!/bin/bash
# MG-only C3: launch list of a 2-window truncated solve (64 RHS) and ncu --set full of the coarse GMRES,
# the finest V-cycle legs and the Gram-Schmidt passes.
python tools/step_probe.py --precond vcycle --iters 40 --repeat 2 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mgc3_launches.csv \
  python tools/step_probe.py --precond vcycle --iters 40 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/mgc3_launches.csv 2>&1 | head -30
ncu --set full --clock-control none --import-source on -k regex:"k_coarse_gmres|k_vc_|k_arnoldi" --launch-skip 60 -c 8 \
  -o gpurun_out/mgc3_full -f python tools/step_probe.py --precond vcycle --iters 40 > gpurun_out/mgc3_full.log 2>&1
ls gpurun_out
