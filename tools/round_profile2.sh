#!/bin/bash
# Evidence refresh: bench lines (learned default with CPU leg, MG-only, datagen, train), launch lists of the
# learned and MG-only C2 steps, and an ncu --set full capture of the roofline kernel inside the bench.
set -x
python bench.py > gpurun_out/p_bench.log 2>&1 || exit 1
python bench.py --precond vcycle --no-cpu > gpurun_out/p_bench_mg.log 2>&1 || exit 1
python bench.py --workload datagen > gpurun_out/p_bench_dg.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/p_launches_learned.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/p_launches_mg.csv \
  python bench.py --precond vcycle --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_conv_tc --launch-skip 20 -c 1 \
  -o gpurun_out/p_conv16 -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
ls gpurun_out
