cd "$GRAFT_REPO_ROOT"
for e in 8192 6144 4096 3072; do
  QN_FWD_TASK_ENTRIES=$e QN_BWD_TASK_ENTRIES=$e timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/sw_$e.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sw_$e.json')); r=d['roofline']['other']; print('c3 fwd+bwd entries $e', round(d['value']), round(r['solve_ms']*1e3,1), r['in_graph_us_per_pass']['solve'])"
done
