#!/bin/bash
# ncu --set full of the c3 hot kernels on the current build (the stand-alone timing launches of bench.py:
# forward, top gather, symmetric top, backward, per-tet pass) + the launch list of the same command
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 5 > $O/c3_final.json 2> $O/c3_final.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file $O/c3_final_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sptrsv|k_tet|k_grad|k_solve_rhs" \
  --launch-skip 40 -c 14 -o $O/c3_final_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > $O/c3_final_ncu.log 2>&1; echo "ncu full rc=$?"
