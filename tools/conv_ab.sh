#!/bin/bash
# A/B of the C3 tcgen05 conv shapes (conv_probe) for the product library and each variant given.
for l in paper_2306_17486_b200/libhelmsolve_b200.so "$@"; do
  echo "== $l"
  P="timeout 60 python tools/conv_probe.py --B 64 --lib $l"
  $P --H 512 --W 1024 --side residual --softplus 0 | tail -1
  $P --H 512 --W 1024 --side none --softplus 1 | tail -1
  $P --H 256 --W 512 --cin 32 --cout 32 --side residual --softplus 0 | tail -1
  $P --H 256 --W 512 --cin 32 --cout 32 --side none --softplus 1 | tail -1
  $P --H 512 --W 1024 --cin 16 --cout 32 --stride 2 --side addend | tail -1
  $P --H 256 --W 512 --cin 32 --cout 16 --transposed 1 --side addend | tail -1
  $P --H 128 --W 256 --cin 64 --cout 32 --transposed 1 --side addend | tail -1
done
