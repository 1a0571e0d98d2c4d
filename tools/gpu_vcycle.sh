#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"k_amg|k_pcg_spmv" --launch-skip 0 -c 60 -o $O/c5_vcycle -f \
  python tools/vcycle_profile.py > $O/c5_vcycle.log 2>&1; echo "ncu rc=$?"; tail -2 $O/c5_vcycle.log
