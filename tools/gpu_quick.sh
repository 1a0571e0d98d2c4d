#!/bin/bash
# quick GPU check: parity tests (TESTS, default the parity + line-search files), then c2 / c3 bench lines
# (value, standalone solve ms, in-graph per-pass times).  Usage: bash tools/gpu_quick.sh [tag]
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; T=${1:-q}
mkdir -p $O
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_line_search.py} -m gpu -x -q > $O/pt_$T.log 2>&1; echo "tests rc=$?"; tail -2 $O/pt_$T.log
for c in ${CONFIGS:-c2 c3}; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > $O/b_${T}_$c.json 2>$O/b_${T}_$c.err
  python -c "import json,sys; d=json.load(open('$O/b_${T}_$c.json')); r=d['roofline']['other']; g=r['in_graph_us_per_pass']; print('$c', round(d['value']), 'solve_ms', round(r['solve_ms']*1e3,1) if r['solve_ms'] else None, 'tet_ms', round(r['tet_ms']*1e3,1), 'in-graph', {k: (round(v,1) if v is not None else None) for k,v in g.items()})" || tail -3 $O/b_${T}_$c.err
done
