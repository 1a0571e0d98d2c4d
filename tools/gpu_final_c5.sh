#!/bin/bash
# end-of-round evidence for configs[4]: bench line (AMG-PCG, pcg_tol 1e-10), per-kernel DRAM / L1 / L2 figures of one
# V-cycle, launch list of one host-stepped frame
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > $O/final_c5_bench.json 2> $O/final_c5_bench.err; echo "bench rc=$?"; cut -c1-400 $O/final_c5_bench.json
bash tools/gpu_vcycle_quick.sh > $O/final_c5_vcycle.txt 2>&1; tail -26 $O/final_c5_vcycle.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/final_c5_launches.csv \
  python bench.py --config c5 --steps 1 --warmup 1 --no-cpu --no-e2e --no-graph > $O/final_c5_ncu.log 2>&1; echo "launch list rc=$?"
python tools/ncu_summary.py $O/final_c5_launches.csv > $O/final_c5_launches_summary.txt 2>&1; cat $O/final_c5_launches_summary.txt
