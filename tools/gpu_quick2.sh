#!/bin/bash
# quick GPU iteration: selected parity tests + short bench (no CPU legs) + launch list
out=gpurun_out; tag=${1:-q}; shift; sel=${1:-test_gpu_parity.py}; shift
timeout 900 python -m pytest $(for t in $sel; do echo tests/$t; done) -m gpu -q -x -p no:cacheprovider > $out/${tag}_tests.txt 2>&1; echo "tests rc=$?"; tail -3 $out/${tag}_tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep "$@" > $out/${tag}_bench.json 2> $out/${tag}_bench.err; tail -2 $out/${tag}_bench.err
python -c "import json; d=json.load(open('$out/${tag}_bench.json')); print(d['ms_per_step'], d['breakdown_ms'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep "$@" > /dev/null 2>&1
python tools/launch_summary.py $out/${tag}_launches.csv | head -20
