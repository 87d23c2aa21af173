#!/bin/bash
# Stage-3 timing of experiment builds (paper_2406_15486_b200/exp/libsa_*.so, built
# with SA_NVCC_EXTRA=-D... and build.py --out=...) against the product library.
# Usage: bash tools/k3_variants.sh OUTDIR [bench args...]
OUT=$1; shift
mkdir -p $OUT
for L in paper_2406_15486_b200/libsampleattn.so paper_2406_15486_b200/exp/libsa_*.so; do
  n=$(basename $L .so)
  SA_LIB_PATH=$PWD/$L timeout 300 python bench.py --no-dense --no-cpu --no-e2e "$@" > $OUT/$n.json 2>$OUT/$n.err
  python -c "import json,sys; d=json.load(open('$OUT/$n.json')); print('$n', d['ms_per_step'], d['stage_ms'], d['roofline']['achieved'], d['clocks']['sm_mhz'])" || tail -3 $OUT/$n.err
done
