#!/bin/bash
# Runs on the GPU box: bench + ncu launch list + ncu --set full of the top kernels.
# usage: tools/gpu_profile.sh <tag> [extra bench args]
tag=${1:-r1}; shift
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/${tag}_smi.txt
timeout 600 python bench.py --steps 10 --warmup 3 "$@" > $out/${tag}_bench.json 2> $out/${tag}_bench.err
tail -3 $out/${tag}_bench.err
cat $out/${tag}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fa_kernel|attention_kernel" -s 3 -c 1 \
    -o $out/${tag}_attn python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $out/${tag}_ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:discover_kernel -s 3 -c 1 \
    -o $out/${tag}_disc python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $out/${tag}_ncu_disc.log 2>&1
ls -la $out
