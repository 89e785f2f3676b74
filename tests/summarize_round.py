"""Markdown table of a round's bench.py JSON lines (tests/measure_round.sh
output): one row per workload and GPU count.

    python tests/summarize_round.py profiles/r01_final
"""
import json
import os
import sys


def last_json(path):
    with open(path) as f:
        lines = [ln for ln in f.read().splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def main(d):
    rows = []
    for name in sorted(os.listdir(d)):
        if not name.endswith(".json"):
            continue
        r = last_json(os.path.join(d, name))
        if not r or "ms_per_step" not in r or r.get("impl") == "reference":
            continue
        cfg, rf, st = r["config"], r.get("roofline") or {}, r.get("step_roofline") or {}
        e2e = r.get("e2e") or {}
        rows.append((cfg["workload"], r["n_gpus"], r["ms_per_step"], r["value"],
                     st.get("frac"), st.get("bound"), rf.get("kernel"), rf.get("frac"),
                     e2e.get("ms_per_step")))
    print("| workload | P | ms/step | params/s (all ranks) | step frac | dominant kernel (frac) "
          "| e2e ms (host buffers) |")
    print("|---|---|---|---|---|---|---|")
    for w, n, ms, v, sf, b, k, kf, e in sorted(rows):
        sfs = f"{sf:.3f}" + (" (NVLink)" if b == "nvlink" else "") if sf is not None else ""
        ks = f"{k} ({kf:.3f})" if k and kf is not None else (k or "")
        es = f"{e:.1f}" if e else ""
        print(f"| {w} | {n} | {ms:.3f} | {v / 1e9:.0f} G | {sfs} | {ks} | {es} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_final")
