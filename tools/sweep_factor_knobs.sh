#!/bin/bash
# c3 factor-structure knobs on the current solve kernels (env overrides read by qn_factor.cpp)
cd "$GRAFT_REPO_ROOT" || exit 1
run() {
  env "$@" timeout 300 python bench.py --config c3 --steps 15 --warmup 3 --no-cpu --no-e2e > gpurun_out/fk.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/fk.json')); r=d['roofline']['other']; f=d['factor']; print(sys.argv[1:], round(d['value']), round(r['solve_ms']*1e3,1), f['nnz_l'], f['supernodes'], f['dense_top'])" "$@"
}
run X=0
run QN_COLLAPSE_HEIGHT=3
run QN_COLLAPSE_COLS=1024
run QN_COLLAPSE_GROWTH=4
run QN_COLLAPSE_HEIGHT=3 QN_COLLAPSE_COLS=1024 QN_COLLAPSE_GROWTH=4
run QN_ND_LEAF=128
run QN_ND_LEAF=512
run QN_RELAX_SCALE=2
run QN_TOP_MAX=2048
run QN_TOP_MAX=3000
