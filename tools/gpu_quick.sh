#!/bin/bash
# quick GPU iteration: parity tests + short bench (no CPU baseline)
tag=${1:-q}; shift
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/${tag}_tests.txt
cat gpurun_out/${tag}_tests.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -2 gpurun_out/${tag}_bench.err; cat gpurun_out/${tag}_bench.json
