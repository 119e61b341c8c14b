#!/bin/bash
out=gpurun_out; tag=${1:-dO}
FPB200_LIB=$PWD/variants/wd.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rows.py tests/test_gpu_phases.py -m gpu -x -q -p no:cacheprovider > $out/${tag}_tests.txt 2>&1; echo "tests rc=$?"; tail -2 $out/${tag}_tests.txt
bash tools/ab_probe.sh ${tag}_ab "4096:0.12,8192:0.12,32768:0.12,131072:0.12" variants/dO0.so variants/dO1.so > /dev/null
python -c "
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(d['tag'], d['L'], round(d['attn_ms'],4))" $out/${tag}_ab.jsonl
