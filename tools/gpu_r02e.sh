#!/bin/bash
# round-2 GPU pass E: assembled forward f for multi-task supernodes: parity, bench c3/c2, trace, solve launch list
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_line_search.py -m gpu -x -q > $O/pt_e.log 2>&1; echo "tests rc=$?"; tail -3 $O/pt_e.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_c3_e.json 2> $O/bench_c3_e.err; echo "bench rc=$?"; cat $O/bench_c3_e.json
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_c2_e.json 2> $O/bench_c2_e.err; echo "bench c2 rc=$?"; cat $O/bench_c2_e.json
timeout 300 python tools/trace_solve.py c3 plain > $O/trace_c3_plain_e.log 2>&1; echo "trace rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sptrsv" -c 40 --csv --log-file $O/c3_solve_launches_e.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu rc=$?"
QN_NO_ASM=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_c3_e_noasm.json 2>/dev/null; echo "bench noasm rc=$?"; cat $O/bench_c3_e_noasm.json | cut -c1-200
timeout 300 python tools/trace_solve.py c2 plain > $O/trace_c2_plain_e.log 2>&1; echo "trace c2 rc=$?"
