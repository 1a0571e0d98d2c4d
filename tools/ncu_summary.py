"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys


def summary(path, skip_prefix=()):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.defaultdict(list)
    for r in rows[hdr_i + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append((k, len(v), sum(v) / len(v) / 1000, sum(v) / tot))
    return out, tot


if __name__ == "__main__":
    out, tot = summary(sys.argv[1])
    print(f"{'kernel':70s} {'n':>5s} {'mean_us':>9s} {'share':>6s}")
    for k, n, m, s in out:
        print(f"{k:70s} {n:5d} {m:9.2f} {s:6.3f}")
    print(f"total {tot/1000:.1f} us")
