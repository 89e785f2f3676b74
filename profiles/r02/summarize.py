"""Markdown table of the round-2 sweep (profiles/r02/sweep/*.json)."""
import glob
import json
import os

rows = []
for f in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "sweep", "*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    k = {n: round(v["avg_ms"], 3) for n, v in d.get("kernels", {}).items()}
    rows.append((d["config"]["workload"], d["n_gpus"], os.path.basename(f), d["ms_per_step"],
                 d["step_roofline"]["frac"], d["roofline"]["kernel"], d["roofline"]["frac"], k))
print("| workload | GPUs | file | ms/step | step roofline frac | dominant kernel (frac) | kernels (avg ms) |")
print("|---|---|---|---|---|---|---|")
for w, n, f, ms, fr, dk, dfr, k in rows:
    print(f"| {w} | {n} | {f} | {ms:.3f} | {fr:.3f} | {dk} ({dfr:.3f}) | {k} |")
