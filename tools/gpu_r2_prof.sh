#!/bin/bash
# ncu --set full of fa_kernel / discover_kernel at 32K (bench inputs), 128K and 256K (sweep inputs)
# plus the new/tightened tests.  usage: tools/gpu_r2_prof.sh <tag>
tag=${1:-r2b}; out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_rows.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -s -k "long_row or discover_maps" > $out/${tag}_tests.txt 2>&1
tail -3 $out/${tag}_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.txt 2>&1; tail -2 $out/${tag}_smoke.txt
for L in 32768 131072 262144; do
  extra=""; [ $L = 32768 ] && extra="--bench-inputs"
  for k in fa_kernel discover_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $out/${tag}_${k}_${L} python tools/ncu_step.py --L $L $extra > $out/${tag}_${k}_${L}.log 2>&1
    tail -1 $out/${tag}_${k}_${L}.log
  done
done
ls -la $out | grep $tag
