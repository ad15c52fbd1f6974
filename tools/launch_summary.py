"""Aggregate an ncu `--metrics gpu__time_duration.sum --csv` launch list per kernel name."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
             "second": 1e3, "s": 1e3}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].replace("(anonymous namespace)", "").replace("<unnamed>", "").replace("void ", "")
        name = name.split("(")[0].split("<")[0].split("::")[-1] or r[ki][:60]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values()) or 1.0
    print("kernel,launches,total_ms,share_pct")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{k},{c},{t:.3f},{100 * t / tot:.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
