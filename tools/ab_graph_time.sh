#!/bin/bash
# usage (GPU box, repo root): bash tools/ab_graph_time.sh  -- ab_old/ holds the other build (git archive + build)
# A/B: new tree vs ab_old (HEAD), graph step on c4 and c5, alternating
for r in 1 2; do
  for c in c4 c5; do
    python tools/graph_time.py $c 2>&1 | tail -1 | sed "s/^/NEW /"
    (cd ab_old && python tools/graph_time.py $c 2>&1 | tail -1 | sed "s/^/OLD /")
  done
done
# eager per-kernel breakdown (kernels_ms_per_step) of both trees
for t in . ab_old; do
  (cd $t && python bench.py --config ${ABCFG:-c4} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-local-full 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', d['value'], d['kernels_ms_per_step'])")
done
