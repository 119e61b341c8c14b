#!/bin/bash
# round-2 first GPU pass: the whole GPU suite (incl. full-size reference parity and the shared-GPU
# multi-rank tests), smoke, and the default bench line
out=gpurun_out; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/r2d_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=25 > $out/r2d_tests.txt 2>&1
tail -40 $out/r2d_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/r2d_smoke.txt 2>&1; tail -3 $out/r2d_smoke.txt
timeout 900 python bench.py > $out/r2d_bench.json 2> $out/r2d_bench.err
tail -3 $out/r2d_bench.err; cat $out/r2d_bench.json
