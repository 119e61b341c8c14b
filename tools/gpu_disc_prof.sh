#!/bin/bash
# ncu --set full of discover_kernel at 32K (bench inputs), 128K and 256K (sweep inputs), plus the
# bench launch list.  usage: tools/gpu_disc_prof.sh <tag>
tag=${1:-r2f}; out=gpurun_out; mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > /dev/null 2>&1
python tools/launch_summary.py $out/${tag}_launches.csv
for L in 32768 131072 262144; do
  extra=""; [ $L = 32768 ] && extra="--bench-inputs"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:discover_kernel -s 1 -c 1 \
      -o $out/${tag}_discover_kernel_${L} python tools/ncu_step.py --L $L $extra > $out/${tag}_discover_kernel_${L}.log 2>&1
  tail -1 $out/${tag}_discover_kernel_${L}.log
done
ls -la $out | grep $tag
