#!/bin/bash
python tools/pcie_bw.py
for c in 4 8 16 32; do
  FPB_E2E_CHUNKS=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks>=$c e2e ms', round(d['e2e']['ms'],3))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:discover_kernel -s 3 -c 1 -o gpurun_out/r4_disc python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
