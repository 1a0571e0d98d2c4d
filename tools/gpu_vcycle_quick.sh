#!/bin/bash
# per-kernel times and the L1 / L2 / DRAM figures of one stand-alone c5 V-cycle (the last 24 k_amg launches)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum \
  --clock-control none -k regex:"k_amg" --csv --log-file $O/vc_quick.csv python tools/vcycle_profile.py > $O/vc_quick.log 2>&1; echo "ncu rc=$?"; tail -1 $O/vc_quick.log
python - <<'P'
import csv, collections
rows = list(csv.reader(open("gpurun_out/vc_quick.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, idi, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        d.setdefault((int(r[idi]), r[ki].split("(")[0]), {})[r[mi]] = float(r[vi].replace(",", ""))
keys = list(d)[-22:]  # presmooth + 5 x (residual, restrict) + coarse + 5 x (prolong, smooth)
tot = 0
for k in keys:
    m = d[k]
    tot += m["gpu__time_duration.sum"]
    print(f"{k[1]:18s} {m['gpu__time_duration.sum']/1e3:8.1f} us  dram {(m['dram__bytes_read.sum']+m['dram__bytes_write.sum'])/1e6:7.1f} MB  "
          f"l1tex {m['l1tex__throughput.avg.pct_of_peak_sustained_elapsed']:5.1f}%  lts {m['lts__throughput.avg.pct_of_peak_sustained_elapsed']:5.1f}%  "
          f"L1hit {m['l1tex__t_sector_hit_rate.pct']:5.1f}%  sect/req {m['l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum']/max(1,m['l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum']):5.1f}")
print(f"total {tot/1e3:.1f} us")
P
