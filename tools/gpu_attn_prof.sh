#!/bin/bash
tag=${1:-a}; shift
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/${tag}_tests.txt; cat gpurun_out/${tag}_tests.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; cat gpurun_out/${tag}_bench.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_kernel -s 3 -c 1 \
    -o gpurun_out/${tag}_attn python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/${tag}_ncu_attn.log 2>&1
tail -2 gpurun_out/${tag}_ncu_attn.log
