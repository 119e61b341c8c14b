tag=r2i; out=gpurun_out
for L in 131072 262144; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:discover_kernel -s 1 -c 1 \
      -o $out/${tag}_discover_kernel_${L} python tools/ncu_step.py --L $L > $out/${tag}_discover_kernel_${L}.log 2>&1
  tail -1 $out/${tag}_discover_kernel_${L}.log
done
