#!/bin/bash
# round-2 first GPU pass: the whole GPU suite (incl. full-size reference parity and the shared-GPU
# multi-rank tests), smoke, and the default bench line
out=gpurun_out; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/r2e_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=25 > $out/r2e_tests.txt 2>&1
tail -40 $out/r2e_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/r2e_smoke.txt 2>&1; tail -3 $out/r2e_smoke.txt
timeout 900 python bench.py > $out/r2e_bench.json 2> $out/r2e_bench.err
tail -3 $out/r2e_bench.err; cat $out/r2e_bench.json
