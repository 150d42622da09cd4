"""Assemble profiles/parity_rNN.json (+ a markdown table on stdout) from the JSON lines the GPU
parity tests append to $AGK_PARITY_REPORT (tests/test_gpu_parity_shapes.py per-RHS / per-step
cases against oracle/_ref; tests/test_gpu_parity_runs.py full integrations against the reference's
own run() with the CPU-vs-CPU floor).
  python tools/parity_report.py gpurun_out/parity_r02x.jsonl profiles/parity_r02.json"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
out = {"per_rhs": [r for r in rows if "gpu" not in r and "restart" not in r], "runs": [r for r in rows if "gpu" in r],
       "restart_windows": [r for r in rows if "restart" in r],
       "bars": {"per_rhs": "max|got-want|/max|want| <= 1e-11 against oracle/_ref",
                "runs": "N, M1 <= 1e-8 rel; n_s <= 1e-6 normwise and element-wise where n_s > 1e-9 max n; "
                        "accepted within 2%; a bar raised to 10x the CPU-vs-CPU floor where that is above it"}}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print("| case | m | rel max diff vs _ref | note |")
print("|---|---|---|---|")
for r in out["per_rhs"]:
    v = r.get("rel_max_diff", r.get("state_rel_max_diff"))
    note = f"rejects {r['rejects']}, tau rel {r['tau_rel']:.1e}, err rel {r['err_rel']:.1e}" if "rejects" in r else ""
    print(f"| {r['case']} | {r.get('m', '2^20')} | {v:.1e} | {note} |")
print()
print("| case | accepted GPU / ref | N | M1 | n_s normwise | n_s element | accepted | raised bars (floor) |")
print("|---|---|---|---|---|---|---|---|")
for r in out["runs"]:
    g, f = r["gpu"], r["cpu_floor"]
    cell = lambda k: f"{g[k]:.1e} (floor {f[k]:.1e})"
    raised = ", ".join(f"{k}→{r['bars'][k]:.1e}" for k in r["raised"]) or "none"
    if r.get("ref_fluctuation_band"):
        raised += " (reference's own band: " + ", ".join(f"{k} {v:.1e}" for k, v in r["ref_fluctuation_band"].items() if v) + ")"
    print(f"| {r['case']} | {r['gpu_counts']['accepted']} / {r['ref_counts']['accepted']} | {cell('N')} | {cell('M1')} "
          f"| {cell('state')} | {cell('elem')} | {g['accepted']:.1e} | {raised} |")
print()
print("| restart window (device and oracle from the same device state) | accepted GPU / ref | N | M1 | n_s normwise | records in lock-step |")
print("|---|---|---|---|---|---|")
for r in out["restart_windows"]:
    d = r["restart"]
    print(f"| {r['case']} | {r['gpu_counts']['accepted']} / {r['ref_counts']['accepted']} | {d['N']:.1e} | {d['M1']:.1e} | {d['state']:.1e} | {d.get('lockstep_records', '')} |")
