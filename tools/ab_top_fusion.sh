cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_line_search.py tests/test_gpu_dropin.py -m gpu -x -q 2>&1 | tail -2
for o in 0 4; do
  QN_SOLVE_OPTS=$o timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab_$o.json 2>gpurun_out/ab_$o.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$o.json')); r=d['roofline']['other']; print('c3 opts $o', round(d['value']), round(r['solve_ms']*1e3,1), r['in_graph_us_per_pass'])" || tail -3 gpurun_out/ab_$o.err
done
