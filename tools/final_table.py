"""Markdown rows of profiles/r02/README.md's measurement table from a directory of bench JSON lines."""
import json
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith("{")]
    return json.loads(lines[-1])


def main(d):
    def g(name):
        try:
            return load(f"{d}/{name}.json")
        except Exception:
            return None

    def fmt(x):
        return f"{x:,.0f}"

    for name in ["bench_c4", "bench_c4_k1", "bench_c4_k1000", "bench_c1", "bench_c2_k1", "bench_c2", "bench_c2_k100",
                 "bench_c3", "bench_c5", "scan_c3", "scan_c4", "scan_c5", "ref_c4", "torchrun1_c3"]:
        j = g(name)
        if not j:
            print(name, "missing")
            continue
        r = j.get("roofline") or {}
        cb = j.get("cpu_baseline") or {}
        par = j.get("parity") or {}
        ra = r.get("random_access") or {}
        tr = r.get("traffic") or {}
        print(f"| {name} | {fmt(j['value'])} | {fmt(j['e2e']['value'])} | frac {r.get('frac') and round(r['frac'], 3)} "
              f"traffic {tr.get('over_alg_bytes') and round(tr['over_alg_bytes'], 2)} "
              f"lookups/s {ra.get('achieved_lookups_per_s') and '%.2e' % ra['achieved_lookups_per_s']} vs "
              f"{ra.get('device_lookups_per_s') and '%.2e' % ra['device_lookups_per_s']} | "
              f"cpu {cb.get('value') and fmt(cb['value'])} scan {(cb.get('scan') or {}).get('qps') and round(cb['scan']['qps'], 1)} | "
              f"parity {par.get('mismatches')} / {par.get('queries')} | ms/step {round(j['ms_per_step'], 3)} | "
              f"build {(j.get('setup') or {}).get('index_build_s') and round(j['setup']['index_build_s'], 2)} s | other {j.get('other_layout') and round(j['other_layout']['value'])} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02/final")
