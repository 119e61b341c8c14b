#!/bin/bash
out=gpurun_out; tag=${1:-fa4}
FPB200_LIB=$PWD/variants/wd.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rows.py -m gpu -x -q -p no:cacheprovider > $out/${tag}_tests.txt 2>&1; echo "tests rc=$?"; tail -3 $out/${tag}_tests.txt
grep -o "block [0-9]* thread [0-9]* stuck on mbarrier smem+0x[0-9a-f]* parity [0-9]" $out/${tag}_tests.txt | awk '{print $2, int($4/32), $8, $10}' | sort | uniq -c | head
FPB200_LIB=$PWD/variants/tr2.so timeout 300 python tools/trace_fa2.py 32768 > $out/${tag}_trace.txt 2>&1; cat $out/${tag}_trace.txt
for v in 0 1; do FPB_FA_V1=$v timeout 600 python tools/ab_attn.py --tag v1=$v --cases "4096:0.12,32768:0.12,131072:0.12" --dense "32768" 2>&1 | grep '^{' >> $out/${tag}_ab.jsonl; done
cat $out/${tag}_ab.jsonl
