#!/bin/bash
# A/B of environment settings on one config: bash tools/gpu_ab_env.sh <config> "<ENV=... ENV2=...>" "<...>" ...
# prints value, stand-alone solve us, in-graph solve us per setting (two rounds, interleaved)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O; C=$1; shift
for rep in 1 2; do
  i=0
  for e in "$@"; do
    i=$((i+1))
    env $e timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu --no-e2e > $O/abe_$i.json 2>$O/abe_$i.err
    python -c "import json; d=json.load(open('$O/abe_$i.json')); r=d['roofline']['other']; g=r['in_graph_us_per_pass']; print('$C [$e]', round(d['value']), 'solve', round(r['solve_ms']*1e3,1) if r['solve_ms'] else None, 'in-graph solve', round(g['solve'],1), 'tet', round(g['tet'],1), 'grad', round(g['grad'],1))" || tail -3 $O/abe_$i.err
  done
done
