"""Opcode histogram of selected kernels in a built library (cuobjdump -sass), as committed evidence
of what the hot kernels execute: tcgen05 (UTC*), TMA/bulk copies (UBLKCP), TMEM loads (LDTM),
mbarrier sync (SYNCS), spills (STL/LDL), 256-bit loads, POPC, etc.
usage: python tools/sass_summary.py paper_1307_2982_b200/libmihg.so > profiles/r02/sass_summary.txt"""
import collections
import re
import subprocess
import sys

KERNELS = [("tc_scan_kernelILi256ELb0ELb1E", "K7 tensor-core scan, 256-bit, CTA pair"),
           ("tc_scan_kernelILi256ELb0ELb0E", "K7 tensor-core scan, 256-bit, one CTA"),
           ("mih_probe_kernelILi1ELb0ELi4E", "K4 MIH probe, 64-bit, untraced, 4 probes/lane (sparse tables)"),
           ("mih_probe_kernelILi1ELb0ELi2E", "K4 MIH probe, 64-bit, untraced, 2 probes/lane (dense tables)"),
           ("mih_piece_kernelILi1ELb0E", "K4b MIH big-bucket pieces, 64-bit"),
           ("mih_solo_kernelILi1ELb0ELi2E", "K4s one block per query (light batches), 64-bit"),
           ("scan_kernel", "K6 POPC scan")]
WATCH = ["UTCIMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "STTM", "UBLKCP", "SYNCS", "ELECT", "UCGABAR", "STL", "LDL",
         "POPC", "LDG", "STG", "ATOMG", "ATOMS", "RED", "LDS", "STS", "VIMNMX", "IMNMX", "SHFL", "VOTE", "BAR", "MEMBAR"]


def main(lib):
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    for key, desc in KERNELS:
        body = next((f for f in funcs if key in f.split("\n", 1)[0]), None)
        if body is None:
            continue
        ops = collections.Counter()
        full = collections.Counter()
        n = 0
        for line in body.splitlines():
            m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
            if m:
                op = m.group(2)
                n += 1
                full[op] += 1
                ops[op.split(".")[0]] += 1
        print(f"== {desc}: {body.split(chr(10), 1)[0].strip()[:110]}")
        print(f"   static instructions: {n}")
        print("   " + ", ".join(f"{w} {ops[w]}" for w in WATCH if ops[w]))
        wide = [o for o in full if o.startswith(("UTCIMMA", "LDTM", "UBLKCP", "LDG.E.ENL2", "UTCBAR", "SYNCS"))]
        print("   variants: " + ", ".join(f"{o} x{full[o]}" for o in sorted(wide)))


if __name__ == "__main__":
    main(sys.argv[1])
