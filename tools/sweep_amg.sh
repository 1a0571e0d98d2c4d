cd "$GRAFT_REPO_ROOT"
for k in ${LANES:-8 4 16 32}; do
  QN_AMG_CSR_LANES=$k timeout 600 python bench.py --config c5 --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/amg_$k.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/amg_$k.json')); v=d['roofline']['other']['vcycle']; print('lanes $k', round(d['value'],2), 'vcycle ms', round(v['ms'],3), 'cg/step', d.get('cg_iterations_per_step'))"
done
