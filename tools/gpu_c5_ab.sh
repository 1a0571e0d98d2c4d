#!/bin/bash
# c5 A/B of environment settings: bash tools/gpu_c5_ab.sh "<ENV=..>" "<ENV=..>" ...  (it/s, V-cycle ms, CG its / step)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 600 python bench.py --config c5 --steps 2 --warmup 2 --no-cpu --no-e2e > $O/c5ab_$i.json 2>$O/c5ab_$i.err
  python -c "import json; d=json.load(open('$O/c5ab_$i.json')); r=d['roofline']['other']; v=r['vcycle']; print('[$e]', round(d['value'],2), 'it/s  vcycle ms', round(v['ms'],3), 'spmv ms', round(r['solve_ms'],3), 'cg/step', d.get('cg_iterations_per_step'), 'launches', d.get('gpu_launches'))" || tail -3 $O/c5ab_$i.err
done
