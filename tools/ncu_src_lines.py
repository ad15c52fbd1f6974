"""Executed warp-instructions and stall samples per CUDA source line of an ncu --set full report
captured with --import-source on (kernels built with -lineinfo). Usage: ncu_src_lines.py rep [top]"""
import csv
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, hdr, agg, src = None, None, {}, {}
    cur = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if r[0] == "Function Name" or hdr is None or len(r) < len(hdr):
            continue
        if r[0].strip():  # a CUDA source line
            cur = (fname, int(r[0]))
            src[cur] = r[1].strip()
            continue
        if cur is None:
            continue
        f = lambda x: float(x) if x not in ("", "-") else 0.0
        a = agg.setdefault(cur, [0.0, 0.0, 0])
        a[0] += f(r[ie])
        a[1] += f(r[st])
        a[2] += 1
    ti = sum(a[0] for a in agg.values()) or 1
    ts = sum(a[1] for a in agg.values()) or 1
    print(f"total warp-instructions {ti:.4e}, stall samples {ts:.0f}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{a[0] / ti * 100:5.1f}% inst {a[1] / ts * 100:5.1f}% stall  {a[2]:4d} sass  {k[0]}:{k[1]}  {src[k][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
