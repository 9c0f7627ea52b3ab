#!/bin/bash
# A/B of the C3 level-0 16-channel conv shapes, libraries interleaved twice (clocks drift under the power cap).
for rep in 1 2; do
for l in "$@"; do
  P="timeout 60 python tools/conv_probe.py --B 64 --lib $l"
  echo "$(basename $l) $($P --H 512 --W 1024 --side residual --softplus 0 | tail -1)"
  echo "$(basename $l) $($P --H 512 --W 1024 --side none --softplus 1 | tail -1)"
done
done
