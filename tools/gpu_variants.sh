#!/bin/bash
# bench several library variants in one GPU call: tools/gpu_variants.sh tag lib1 lib2 ...
tag=$1; shift
for lib in "$@"; do
  FPB200_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_$(basename $lib).json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/${tag}_$(basename $lib).json')); print('$lib', d['ms_per_step'], d['breakdown_ms'], round(d['roofline']['frac'],3))"
done
