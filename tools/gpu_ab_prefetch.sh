#!/bin/bash
# A/B of the next-tile prefetch (QN_SOLVE_OPTS bit 3 disables it): parity subset, c3 bench lines, c3 trace
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_100 or c2_three or c3_frame or prefactored or twist" 2>&1 | tail -2
for o in 0 8; do
  QN_SOLVE_OPTS=$o timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e > $O/ab_$o.json 2>$O/ab_$o.err
  python -c "import json; d=json.load(open('$O/ab_$o.json')); r=d['roofline']['other']; print('c3 opts $o', round(d['value']), round(r['solve_ms']*1e3,1), r['in_graph_us_per_pass'])" || tail -3 $O/ab_$o.err
done
timeout 300 python tools/trace_solve.py c3 plain > $O/trace_c3.txt 2>&1; grep -- "---" $O/trace_c3.txt
