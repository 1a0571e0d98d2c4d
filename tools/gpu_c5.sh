#!/bin/bash
# configs[4] at full size on one GPU: bench line (AMG-PCG, 1e-10), launch list (host loop, per-kernel launches)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > $O/c5_bench.json 2> $O/c5_bench.err; echo "bench rc=$?"; cut -c1-3000 $O/c5_bench.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/c5_launches.csv \
  python bench.py --config c5 --steps 1 --warmup 1 --no-cpu --no-e2e --no-graph > $O/c5_ncu.log 2>&1; echo "ncu rc=$?"
