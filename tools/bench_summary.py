"""Print a one-line summary of bench.py JSON lines read from stdin."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r = d.get("roofline") or {}
    print(d["config"]["workload"][:28], f"{d['value']:.0f} q/s", f"e2e {d['e2e']['value']:.0f}",
          f"frac {r.get('frac', 0):.4f}", f"probe_ms {r.get('probe_ms_per_step', 0):.2f}",
          f"step_ms {d['ms_per_step']:.2f}", "launches", d.get("gpu_launches"),
          "cpu", (d.get("cpu_baseline") or {}).get("value"), "clk", d.get("clocks", {}).get("sm_mhz"))
