#!/bin/bash
# round-2 first GPU pass: the whole GPU suite (incl. full-size reference parity and the shared-GPU
# multi-rank tests), smoke, and the default bench line
out=gpurun_out; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/${TAG:-r2e}_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=25 > $out/${TAG:-r2e}_tests.txt 2>&1
tail -40 $out/${TAG:-r2e}_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/${TAG:-r2e}_smoke.txt 2>&1; tail -3 $out/${TAG:-r2e}_smoke.txt
timeout 900 python bench.py > $out/${TAG:-r2e}_bench.json 2> $out/${TAG:-r2e}_bench.err
tail -3 $out/${TAG:-r2e}_bench.err; cat $out/${TAG:-r2e}_bench.json
