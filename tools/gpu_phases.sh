#!/bin/bash
out=gpurun_out; tag=${1:-ph1}
timeout 900 python -m pytest tests/test_gpu_phases.py -m gpu -x -q -p no:cacheprovider > $out/${tag}_tests.txt 2>&1; echo "tests rc=$?"; tail -2 $out/${tag}_tests.txt
for P in 1 2; do FPB_FA_PHASES=$P timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fa_kernel -s $P -c $P python tools/ncu_step.py --L 262144 > $out/${tag}_ncu_P$P.txt 2>&1; echo "P=$P"; grep -E "dram__bytes|gpu__time" $out/${tag}_ncu_P$P.txt; done
for P in 1 2; do FPB_FA_PHASES=$P timeout 600 python tools/ab_attn.py --tag P=$P --cases "32768:0.12,262144:0.12" --dense "" 2>&1 | grep '^{' >> $out/${tag}_ab.jsonl; done; cat $out/${tag}_ab.jsonl
