#!/bin/bash
# A/B several library builds (timing probes or variants) across lengths in one GPU call, interleaved
# twice.  usage: tools/ab_probe.sh <tag> <cases> lib1 lib2 ...
tag=$1; cases=$2; shift 2
for rep in 1 2; do
  for lib in "$@"; do
    FPB200_LIB=$PWD/$lib timeout 180 python tools/ab_attn.py --tag $(basename $lib) --cases "$cases" --dense "" 2>&1 | grep '^{' >> gpurun_out/${tag}.jsonl
  done
done
cat gpurun_out/${tag}.jsonl
