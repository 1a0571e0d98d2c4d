#!/bin/bash
# round-2 GPU pass C: symmetric top + narrow-task solve mappings: parity tests, bench c3, trace
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_dropin.py tests/test_gpu_slab.py -m gpu -x -q > $O/pt_c.log 2>&1; echo "tests rc=$?"; tail -3 $O/pt_c.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $O/bench_c3_c.json 2> $O/bench_c3_c.err; echo "bench rc=$?"; cat $O/bench_c3_c.json
timeout 300 python tools/trace_solve.py c3 plain > $O/trace_c3_plain_c.log 2>&1; echo "trace rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"TimingIO" -c 40 --csv --log-file $O/c3_solve_launches_c.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu rc=$?"
