"""Print a compact summary of a bench.py JSON line (last line of a log)."""
import json
import sys

lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
r = json.loads(lines[-1])
print("c2", r["value"], r["unit"], r.get("kernels_ms"), "frac", r["roofline"]["frac"])
for s in r.get("secondary", []):
    keys = ("value", "unit", "ms_per_step", "kernels_ms", "gemm_TFLOPs", "TFLOPs", "error")
    print(s.get("workload", "")[:40], {k: s.get(k) for k in keys if s.get(k) is not None},
          "frac", s.get("roofline", {}).get("frac"))
