#!/bin/bash
# quick GPU check: short learned-C2 bench (value, breakdown) then the GPU test summary
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/b.json
python -c "import json; d=json.load(open('gpurun_out/b.json')); print('BENCH', d['value'], d['ms_per_step'], d['iterations_per_rhs']); print(json.dumps(d['breakdown']))"
timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
