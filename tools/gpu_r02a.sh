#!/bin/bash
# round-2 GPU pass A: edge-case tests, the full GPU suite, c3 bench line, c3 launch list + ncu captures, flop counts
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
mkdir -p $O
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum
timeout 600 python -m pytest tests/test_gpu_line_search.py -m gpu -x -q > $O/pt_ls.log 2>&1; echo "ls rc=$?"
timeout 1200 python -m pytest tests -m gpu -q > $O/pt_all.log 2>&1; echo "all rc=$?"; tail -3 $O/pt_all.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench rc=$?"; cat $O/bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/c3_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sptrsv|k_tet|k_grad|k_vec|k_eta" -c 7 \
  -o $O/c3_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
for w in "c1" "c3" "c5 100 25 25" "c4"; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:k_tet_plain --csv --log-file "$O/flops_${w// /_}.csv" \
    python tools/tet_flops.py $w > "$O/flops_${w// /_}.log" 2>&1; echo "flops $w rc=$?"
done
