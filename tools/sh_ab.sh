#!/bin/bash
# A/B timings of the tcgen05.shift 16->16 conv at the C3 level-0 shape: the product library and measurement
# variants built with `make variant VARIANT=<name> DEFS=...` (tools/_variants/); three epilogue cases each
run() { timeout 120 python tools/conv_probe.py --B 64 --H 512 --W 1024 --side $2 --softplus $3 ${1:+--lib $1} 2>&1 | tail -1; }
cases() { run "$1" none 1; run "$1" residual 0; run "$1" addend 1; }
echo "product:"; cases ""
for v in "$@"; do echo "variant $v:"; cases tools/_variants/libhelmsolve_b200_$v.so; done
