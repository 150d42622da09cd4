"""Markdown time-to-t_end table from a tools/runs.py JSON (profiles/runs_*.json)."""
import json
import sys

d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "profiles/runs_r01h.json"))
print("| config | scheme | t range | GPU wall | accepted / rejected | RHS evals | µs per RHS in the run "
      "| reference CPU (1 core, extrapolated) |")
print("|---|---|---|---|---|---|---|---|")
seen = {}
for r in d:  # the latest entry per (config, scheme, horizon)
    seen[(r["config"], r["stepper"], r["horizon"])] = r
for r in sorted(seen.values(), key=lambda r: (r["config"], r["horizon"], r["stepper"])):
    cpu = r.get("cpu_time_to_horizon_extrapolated_s")
    if not cpu:
        cs = "-"
    elif cpu > 2 * 86400:
        cs = f"{cpu / 86400:.1f} d"
    elif cpu > 7200:
        cs = f"{cpu / 3600:.1f} h"
    else:
        cs = f"{cpu:.1f} s"
    hz = f"{r['horizon']:g}" + ("" if r["complete"] else f" (prefix of {r['t_end_full']:g})")
    print(f"| {r['config']} | {r['stepper']} | {hz} | {r['wall_s']:.2f} s | {r['accepted']:,} / {r['rejects']:,} "
          f"| {r['rhs_evals']:,} | {r['us_per_rhs_in_run']:.1f} | {cs} |")
