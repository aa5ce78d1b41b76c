#!/bin/bash
# c5 per-change-set loop (bench.py --loop --per-set) in several trees side by side (GPU box, repo root):
#   bash tools/bisect_loop.sh DIR...   (each DIR a built tree: git archive + build)
for r in 1 2; do
  for t in "$@"; do
    (cd $t && python bench.py --config c5 --loop --per-set --steps 100 --warmup 3 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', d['value'], d['ms_per_step'], d.get('loop'), d.get('static_cache',{}).get('builds'))")
  done
done
