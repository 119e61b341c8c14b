#!/bin/bash
out=gpurun_out; tag=${1:-ps1}
FPB200_LIB=$PWD/variants/wd.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rows.py tests/test_gpu_phases.py -m gpu -x -q -p no:cacheprovider > $out/${tag}_tests.txt 2>&1; echo "tests rc=$?"; tail -3 $out/${tag}_tests.txt
grep -o "block [0-9]* thread [0-9]* stuck on mbarrier smem+0x[0-9a-f]* parity [0-9]" $out/${tag}_tests.txt | awk '{print $2, int($4/32), $8, $10}' | sort | uniq -c | head
bash tools/ab_probe.sh ${tag}_ab "4096:0.12,32768:0.12,131072:0.12" variants/base.so variants/psmem.so
