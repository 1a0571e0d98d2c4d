#!/bin/bash
# round-2 GPU pass F: solve mapping knobs (QN_SOLVE_OPTS) on c2 / c3
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
mkdir -p $O
for c in c2 c3; do for o in 0 1 2 3; do
  QN_SOLVE_OPTS=$o timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > $O/f_$c_$o.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('$O/f_$c_$o.json')); r=d['roofline']['other']; print('$c opts $o', round(d['value']), 'solve_ms', round(r['solve_ms']*1e3,1), 'in-graph', round(r['in_graph_us_per_pass']['solve'],1))"
done; done
