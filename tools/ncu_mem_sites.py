"""Per-instruction global-memory sectors of an ncu --set full report (source page, SASS): the
load/store sites ranked by L2 theoretical sectors, with their stall share."""
import csv
import subprocess
import sys


def main(rep, top=20):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    h = rows[1]
    if "--columns" in sys.argv:
        print([c for c in h if "ector" in c or "equest" in c or "avefront" in c])
    col = {n: h.index(n) for n in ("Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed",
                                   "L2 Theoretical Sectors Global", "L2 Theoretical Sectors Global Ideal",
                                   "L1 Tag Requests Global", "L2 Theoretical Sectors Local")}
    data = []
    for r in rows[2:]:
        if len(r) < len(h) or r[0].startswith("Kernel"):
            break
        f = lambda n: float(r[col[n]] or 0) if r[col[n]] not in ("-", "") else 0.0
        data.append((r[col["Address"]], r[col["Source"]].strip(), f("Warp Stall Sampling (All Samples)"),
                     f("Instructions Executed"), f("L2 Theoretical Sectors Global"),
                     f("L2 Theoretical Sectors Global Ideal"), f("L2 Theoretical Sectors Local")))
    tot_s = sum(d[2] for d in data) or 1
    tot_g = sum(d[4] for d in data) or 1
    tot_l = sum(d[6] for d in data)
    print(f"global L2 sectors {tot_g:.3e}, local (spill) sectors {tot_l:.3e}")
    for d in sorted(data, key=lambda d: -d[4])[:top]:
        print(f"  {d[4] / tot_g * 100:5.1f}% sect {d[4]:.3e} (ideal {d[5]:.3e}) stall {d[2] / tot_s * 100:4.1f}%  {d[1][:70]}")
    # wide loads (LDG.E.ENL2.256 etc.) may not report theoretical sectors: list every global load
    # with its executed count so their traffic can be estimated (32 B per lane-load, uncoalesced)
    print("global loads/stores by executed warp-instructions:")
    for d in sorted((d for d in data if ("LDG" in d[1] or "STG" in d[1] or "ATOM" in d[1] or "RED" in d[1])),
                    key=lambda d: -d[3])[:top]:
        print(f"  exec {d[3]:.3e} sect {d[4]:.3e} stall {d[2] / tot_s * 100:4.1f}%  {d[1][:80]}")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(args[0], int(args[1]) if len(args) > 1 else 20)
