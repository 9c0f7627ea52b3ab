#!/bin/bash
# V-cycle / Krylov iteration check: GPU tests of the multigrid and Krylov paths, MG-only and learned
# C2 bench lines, and a launch list of the MG-only step.
timeout 600 python -m pytest tests/test_gpu_multigrid.py tests/test_gpu_krylov.py -q -x 2>&1 | tail -3
python bench.py --precond vcycle --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/mg_b.json
python -c "import json; d=json.load(open('gpurun_out/mg_b.json')); print('MG', d['value'], d['ms_per_step'], d['iterations_per_rhs']); print(json.dumps(d['breakdown']))"
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/mg_launches.csv \
  python bench.py --precond vcycle --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/mg_launches.csv | head -14
if [ "$1" = "full" ]; then
  python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/l_b.json
  python -c "import json; d=json.load(open('gpurun_out/l_b.json')); print('LEARNED', d['value'], d['ms_per_step'], d['iterations_per_rhs']); print(json.dumps(d['breakdown']))"
fi
