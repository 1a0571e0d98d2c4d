"""Summarise an `ncu --set full` report: per kernel duration, DRAM bytes,
throughputs, occupancy, FP64 pipe use and the top stall reasons.

    python tools/ncu_report.py gpurun_out/prof.ncu-rep [out.txt] [traffic.json key=regex ...]
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "dfma"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "dadd"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "dmul"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return float(v) * scale.get(u, 1.0)


def main(path, out_txt=None, traffic=None, keys=()):
    hdr, units, rows = raw(path)
    idx = {h: i for i, h in enumerate(hdr)}
    lines = []
    per_kernel = {}
    for r in rows:
        name = r[idx["Kernel Name"]]
        d = {}
        for m, k in METRICS:
            if m in idx and r[idx[m]] not in ("", "n/a"):
                v = r[idx[m]].replace(",", "")
                try:
                    d[k] = to_bytes(v, units[idx[m]]) if "bytes" in m else float(v)
                    if m == "gpu__time_duration.sum" and units[idx[m]] == "nsecond":
                        d[k] = float(v) / 1000.0
                    elif m == "gpu__time_duration.sum" and units[idx[m]] == "msecond":
                        d[k] = float(v) * 1000.0
                except ValueError:
                    pass
        stalls = []
        for h in hdr:
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(r[idx[h]].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        top = ", ".join(f"{n} {s / tot:.0%}" for s, n in sorted(stalls, reverse=True)[:4])
        traffic_b = d.get("dram_read", 0.0) + d.get("dram_write", 0.0)
        lines.append(f"{name[:70]}\n  duration {d.get('duration', 0):.2f} us | DRAM {traffic_b / 1e6:.2f} MB "
                     f"({d.get('dram_pct', 0):.1f}% of peak) | SM {d.get('sm_pct', 0):.1f}% | FP64 pipe "
                     f"{d.get('fp64_pipe_pct', 0):.1f}% | occupancy {d.get('occupancy_pct', 0):.1f}% | regs "
                     f"{d.get('regs', 0):.0f} | grid {d.get('grid', 0):.0f} | L2 {d.get('l2_bytes', 0) / 1e6:.2f} MB\n"
                     f"  stalls: {top}"
                     + (f"\n  fp64 flops {2 * d.get('dfma', 0) + d.get('dadd', 0) + d.get('dmul', 0):.4g} "
                        f"({(2 * d.get('dfma', 0) + d.get('dadd', 0) + d.get('dmul', 0)) / max(d.get('duration', 1), 1e-9) / 1e6:.2f} TFLOP/s)"
                        if d.get('dfma') else ""))
        per_kernel.setdefault(name, []).append(traffic_b)
    text = "\n".join(lines)
    print(text)
    if out_txt:
        with open(out_txt, "w") as fh:
            fh.write(f"source: {path}\n{text}\n")
    if traffic:
        try:
            with open(traffic) as fh:
                tj = json.load(fh)
        except (OSError, ValueError):
            tj = {}
        for kv in keys:  # key = sum over matching kernels of their mean bytes per launch
            key, rx = kv.split("=", 1)
            means = [sum(vs) / len(vs) for n, vs in per_kernel.items() if re.search(rx, n) and vs]
            if means:
                tj[key] = sum(means)
        with open(traffic, "w") as fh:
            json.dump(tj, fh, indent=1)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], a[1] if len(a) > 1 else None, a[2] if len(a) > 2 else None, a[3:])
