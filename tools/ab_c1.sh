#!/bin/bash
# Interleaved A/B of prebuilt library variants (paper_2510_07868_b200/var_<name>.so) on the C1
# latency probe (tools/c1_latency.py).  usage: bash tools/ab_c1.sh V0 V1 ...  (GPU box)
cd "$(dirname "$0")/.."
cp paper_2510_07868_b200/libnrrs_gpu.so /tmp/lib_orig.so
for round in 1 2; do
  for v in "$@"; do
    cp "paper_2510_07868_b200/var_$v.so" paper_2510_07868_b200/libnrrs_gpu.so
    echo "== $v"; python tools/c1_latency.py 2>&1 | grep -v "^\s*$"
  done
done
cp /tmp/lib_orig.so paper_2510_07868_b200/libnrrs_gpu.so
