"""Markdown table of a tools/configs.py JSONL (profiles/CONFIGS_*.md)."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1])]
print("| config | prec | steps/ray | solve ms | steps/s (solve) | steps/s (trace) | check |")
print("|---|---|---|---|---|---|---|")
for d in rows:
    if "total_steps" not in d:
        print(f"| {d['config']} | | | | | | σ_max slope {d['sigma_max_slope']:.3f}, "
              f"σ_median slope {d['sigma_median_slope']:.3f}, time slope {d['time_slope']:.3f} |")
        continue
    chk = ""
    if "max_err_over_peak" in d:
        chk = f"max \\|mc − slab oracle\\| = {100 * d['max_err_over_peak']:.3f} % of peak"
    if "cpu_parity" in d:
        c = d["cpu_parity"]
        chk = (f"vs reference CPU on {c['cells']} cells: {100 * c['frac_within_tol']:.2f} % within "
               f"1e-9 rel, max rel {c['max_rel']:.1e}, all within 3σ: {c['all_within_3sigma']}; "
               f"CPU {c['cpu_steps_per_s']:.3g} steps/s ({c['cpu_threads']} thr)")
    if "full_field_parity" in d:
        c = d["full_field_parity"]
        chk = (f"every cell vs reference solve(): {100 * c['frac_within_tol']:.4f} % within 1e-9 "
               f"rel, {c['bitwise_cells']} of {c['n']} bitwise, max rel {c['max_rel']:.1e}, "
               f"all within 3σ: {c['all_within_3sigma']}, total steps equal: {c['steps_equal']}; "
               f"CPU {c['cpu_steps_per_s']:.3g} steps/s ({c['cpu_threads']} thr, "
               f"{c['cpu_wall_s']:.1f} s)")
    if "vs_fp64_same_rays" in d:
        c = d["vs_fp64_same_rays"]
        chk = (f"vs fp64 (same rays): {c['violations_3sigma']} cells outside 3σ "
               f"(allowed {c['allowed']}), max rel {c['max_rel']:.1e}")
    if "sigma_max" in d and not chk:
        chk = f"σ max {d['sigma_max']:.4g}, median {d.get('sigma_median', float('nan')):.4g}"
    if "steps_per_level" in d and d.get("n_levels", 1) > 1:
        chk += f"; steps/level {d['steps_per_level']}"
    print(f"| {d['config']} | {d['precision']} | {d['steps_per_ray']:.2f} | {d['solve_ms']:.1f} | "
          f"{d['steps_per_s']:.3g} | {d['trace_steps_per_s']:.3g} | {chk} |")
