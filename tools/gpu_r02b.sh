#!/bin/bash
# round-2 GPU pass B: solve traces (c2, c3), ncu --set full of the c3 timing kernels, c5 tolerance sweep
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
mkdir -p $O
timeout 300 python tools/trace_solve.py c3 plain > $O/trace_c3_plain.log 2>&1; echo "trace c3 rc=$?"
timeout 300 python tools/trace_solve.py c3 graph > $O/trace_c3_graph.log 2>&1; echo "trace c3 graph rc=$?"
timeout 300 python tools/trace_solve.py c2 graph > $O/trace_c2_graph.log 2>&1; echo "trace c2 graph rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"TimingIO|k_tet_plain" -c 6 \
  -o $O/c3_full_timing -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_full_timing.log 2>&1; echo "ncu full rc=$?"
timeout 900 python tools/c5_tol_sweep.py 40 10 10 --slabs 2 4 > $O/c5_sweep_40.log 2>&1; echo "sweep40 rc=$?"
timeout 1200 python tools/c5_tol_sweep.py 100 25 25 --frames 1 --tols 1e-10 1e-11 1e-12 > $O/c5_sweep_100.log 2>&1; echo "sweep100 rc=$?"
