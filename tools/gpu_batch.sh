#!/bin/bash
# GPU batch: tests, bench, 2-rank torchrun smoke on one GPU, trace, ncu of fa_kernel
tag=${1:-b}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench.json 2>gpurun_out/${tag}_bench.err
python -c "import json; d=json.load(open('gpurun_out/${tag}_bench.json')); print('bench', d['ms_per_step'], d['breakdown_ms'], 'e2e', d['e2e']['ms'], 'frac', round(d['roofline']['frac'],3))"
FPB_BENCH_SHARED_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('2-rank', d['n_gpus'], d['value'], d['ms_per_step'])"
[ -f variants/libfpb200_trace.so ] && FPB200_LIB=$PWD/variants/libfpb200_trace.so timeout 300 python tools/trace_attention.py
