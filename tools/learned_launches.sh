#!/bin/bash
# Learned C2: Krylov GPU tests, then the launch list of one step (top kernels)
timeout 600 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_multigrid.py -q -x 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/l_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/l_launches.csv 2>&1 | head -${1:-20}
