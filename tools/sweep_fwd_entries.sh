cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_100 or c2_three or c3_frame or prefactored or twist" 2>&1 | tail -1
for e in 8192 6144 4096; do
  QN_FWD_TASK_ENTRIES=$e timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/sw_$e.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sw_$e.json')); r=d['roofline']['other']; print('c3 fwd entries $e', round(d['value']), round(r['solve_ms']*1e3,1), r['in_graph_us_per_pass']['solve'])"
done
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/sw_c2.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/sw_c2.json')); r=d['roofline']['other']; print('c2', round(d['value']), round(r['solve_ms']*1e3,1), r['in_graph_us_per_pass']['solve'])"
