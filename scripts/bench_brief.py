"""Condense a bench.py JSON line (stdin) into one line: label, ms/answer, fallbacks, top kernels."""
import json
import sys

label = " ".join(sys.argv[1:])
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    ks = d.get("kernels_ms_per_answer", d.get("kernels_ms_per_step", {}))
    top = ", ".join(f"{k} {v:.1f}" for k, v in list(ks.items())[:5])
    e2e = d.get('e2e', {})
    cb = d.get("cpu_baseline") or {}
    ratio = f", cpu x{d['value'] / cb['value']:.0f}" if cb.get("value") else ""
    print(f"{label}: {d.get('ms_per_step', 0):.1f} ms, e2e {e2e.get('answer_ms', e2e.get('select_ms', 0)):.1f} ms{ratio}, "
          f"fallbacks {d.get('exact_fallbacks')}, decrypt {d.get('verified_decrypt')} | {top}")
