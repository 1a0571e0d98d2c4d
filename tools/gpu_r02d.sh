#!/bin/bash
# round-2 GPU pass D: TMA-staged task tiles in the persistent solve: parity, bench c3/c2, trace, solve launch list
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_line_search.py -m gpu -x -q > $O/pt_d.log 2>&1; echo "tests rc=$?"; tail -3 $O/pt_d.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_c3_d.json 2> $O/bench_c3_d.err; echo "bench rc=$?"; cat $O/bench_c3_d.json
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_c2_d.json 2> $O/bench_c2_d.err; echo "bench c2 rc=$?"; cat $O/bench_c2_d.json
timeout 300 python tools/trace_solve.py c3 plain > $O/trace_c3_plain_d.log 2>&1; echo "trace rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sptrsv" -c 40 --csv --log-file $O/c3_solve_launches_d.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu rc=$?"
