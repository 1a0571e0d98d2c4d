#!/bin/bash
# AMG V-cycle check: scaled c5 parity tests, then the c5 bench line per CSR lane count (LANES)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -m gpu -x -q -k "c5 or amg or pcg or two_level or coarse" > $O/pt_amg.log 2>&1; echo "tests rc=$?"; tail -2 $O/pt_amg.log
for k in ${LANES:-0 4 8 16}; do
  if [ "$k" = 0 ]; then unset QN_AMG_CSR_LANES; else export QN_AMG_CSR_LANES=$k; fi
  timeout 600 python bench.py --config c5 --steps 2 --warmup 2 --no-cpu --no-e2e > $O/amg_$k.json 2>$O/amg_$k.err
  python -c "import json; d=json.load(open('$O/amg_$k.json')); v=d['roofline']['other']['vcycle']; print('lanes $k', round(d['value'],2), 'vcycle ms', round(v['ms'],3), 'cg/step', d.get('cg_iterations_per_step'))" || tail -3 $O/amg_$k.err
done
