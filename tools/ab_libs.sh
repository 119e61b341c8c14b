#!/bin/bash
# A/B several library builds in ONE GPU call (same box): tools/ab_libs.sh tag "cases" lib1 lib2 ...
# each lib is timed twice, interleaved, with tools/ab_attn.py (discovery + attention per case)
tag=$1; cases=$2; shift 2
for rep in 1 2; do
  for lib in "$@"; do
    FPB200_LIB=$PWD/$lib timeout 300 python tools/ab_attn.py --tag "$(basename $lib)" --cases "$cases" --dense "" 2>/dev/null
  done
done > gpurun_out/${tag}_ab.jsonl
python - "$tag" <<'PY'
import json, sys, collections
rows = [json.loads(l) for l in open(f"gpurun_out/{sys.argv[1]}_ab.jsonl")]
agg = collections.defaultdict(list)
for r in rows:
    agg[(r["tag"], r["L"], r["alpha"])].append((r["disc_ms"], r["attn_ms"]))
for k, v in sorted(agg.items(), key=lambda x: (x[0][1], x[0][0])):
    print(k, "disc", [round(a, 4) for a, _ in v], "attn", [round(b, 3) for _, b in v])
PY
