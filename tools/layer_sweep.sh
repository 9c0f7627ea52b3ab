#!/bin/bash
# Per-layer C3 network times (tools/cnn_probe.py --profile) for the product library and each variant given.
for l in paper_2306_17486_b200/libhelmsolve_b200.so "$@"; do
  echo "== $l"
  timeout 120 python tools/cnn_probe.py --iters 10 --profile --lib $l 2>&1 | grep -E "forward|    [0-9 ][0-9] "
done
