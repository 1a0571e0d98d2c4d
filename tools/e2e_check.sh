cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_line_search.py tests/test_gpu_configs.py -m gpu -q -x -k "not 400x100x100" 2>&1 | tail -2
for c in c1 c3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/e2e_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$c.json')); print('$c', round(d['value']), 'e2e', round(d['e2e']['value']))"
done
