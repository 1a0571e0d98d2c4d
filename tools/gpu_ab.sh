#!/bin/bash
# parity subset, then QN_SOLVE_OPTS A/B on c3 with traces: bash tools/gpu_ab.sh "<bench opts>" "<trace opts>" [config]
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_100 or c2_three or c3_frame or prefactored or twist" 2>&1 | tail -2
bash tools/gpu_ab_opts.sh "$1" ${3:-c3} "$2"
