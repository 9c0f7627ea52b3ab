#!/bin/bash
# MG-only (V-cycle preconditioner) C2 profile: bench line, launch list, ncu --set full of the
# finest-level V-cycle legs and the Arnoldi dot pass.
set -x
python bench.py --precond vcycle --steps 3 --warmup 3 --no-cpu > gpurun_out/mg_bench.log 2>&1 || exit 1
tail -1 gpurun_out/mg_bench.log | cut -c1-400
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/mg_launches.csv \
  python bench.py --precond vcycle --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/mg_ncu1.log 2>&1
for k in k_vc_up k_vc_down k_arnoldi k_coarse_gmres; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 40 -c 1 \
    -o gpurun_out/mg_$k -f python bench.py --precond vcycle --steps 1 --warmup 1 --no-cpu --no-e2e \
    > gpurun_out/mg_ncu_$k.log 2>&1
done
ls -la gpurun_out
