#!/bin/bash
# Interleaved A/B of prebuilt library variants (paper_2510_07868_b200/var_<name>.so, built with
# NRRS_EXTRA_DEFINES): each variant is swapped in as libnrrs_gpu.so and timed by bench.py twice.
# usage: bash tools/ab_variants.sh V0 V1 ...   (run on the GPU box)
cd "$(dirname "$0")/.."
cp paper_2510_07868_b200/libnrrs_gpu.so /tmp/lib_orig.so
for round in 1 2; do
  for v in "$@"; do
    cp "paper_2510_07868_b200/var_$v.so" paper_2510_07868_b200/libnrrs_gpu.so
    touch paper_2510_07868_b200/libnrrs_gpu.so
    python bench.py --no-extra --no-cpu 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,3), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k, v in d['kernels_ms'].items()})"
  done
done
cp /tmp/lib_orig.so paper_2510_07868_b200/libnrrs_gpu.so
