#!/bin/bash
# end-of-round evidence on the current build: GPU suite, smoke, default bench line, launch list and
# ncu --set full of the c3 hot kernels (same commands as the round-end driver plus the profiles)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/final_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/final_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/final_bench.json 2> $O/final_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file $O/final_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sptrsv|k_tet|k_grad|k_solve_rhs" \
  --launch-skip 40 -c 12 -o $O/final_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > $O/final_ncu.log 2>&1; echo "ncu full rc=$?"
