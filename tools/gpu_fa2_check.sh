#!/bin/bash
# fa2 bring-up: watchdog build through the GPU parity suites, then v1 vs v2 timing
out=gpurun_out; tag=${1:-fa2}
FPB200_LIB=$PWD/variants/wd.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rows.py tests/test_gpu_fullsize_parity.py -m gpu -x -q -p no:cacheprovider > $out/${tag}_tests.txt 2>&1; echo "tests rc=$?"; tail -25 $out/${tag}_tests.txt
for v in 0 1; do FPB_FA_V1=$v timeout 600 python tools/ab_attn.py --tag v1=$v --cases "4096:0.12,32768:0.12,131072:0.12" --dense "32768" 2>&1 | grep '^{' >> $out/${tag}_ab.jsonl; done
cat $out/${tag}_ab.jsonl
