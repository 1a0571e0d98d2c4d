#!/bin/bash
# A/B of QN_SOLVE_OPTS values on a config: bash tools/gpu_ab_opts.sh "<opts list>" [config] [trace opts]
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O; C=${2:-c3}
for o in $1; do
  QN_SOLVE_OPTS=$o timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu --no-e2e > $O/ab_$o.json 2>$O/ab_$o.err
  python -c "import json; d=json.load(open('$O/ab_$o.json')); r=d['roofline']['other']; print('$C opts $o', round(d['value']), round(r['solve_ms']*1e3,1), r['in_graph_us_per_pass'])" || tail -3 $O/ab_$o.err
done
for o in $3; do
QN_SOLVE_OPTS=$o timeout 300 python tools/trace_solve.py $C plain > $O/trace_${C}_$o.txt 2>&1; echo "trace opts $o"; grep -- "---" $O/trace_${C}_$o.txt
done
