#!/bin/bash
# stage-removal timings of the tcgen05.shift 16->16 conv at the C3 level-0 shape (variants built with
# `make variant VARIANT=sh<mask> DEFS=-DHS_SH_PROBE=<mask>`); "product" is the in-tree library
run() { timeout 120 python tools/conv_probe.py --B 64 --H 512 --W 1024 --side ${2:-residual} --softplus ${3:-0} ${1:+--lib $1} 2>&1 | tail -1; }
echo "product:"; run "" residual 0; run "" addend 1
for v in "$@"; do echo "variant $v:"; run tools/_variants/libhelmsolve_b200_$v.so residual 0; done
