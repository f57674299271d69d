"""Summarise ncu --set full captures of the trace kernel into profiles/.

usage: python tools/ncu_summary.py <tag> <prof_fp64.ncu-rep> <prof_fp32.ncu-rep> <steps_fp64> <steps_fp32>
Writes profiles/ncu_<tag>_{fp64,fp32}.csv (raw metrics of interest) and
updates profiles/ncu_trace_summary.json (per-step DRAM traffic used by bench.py).

       python tools/ncu_summary.py --one <out.csv> <prof.ncu-rep>
Writes the metrics of one capture plus its warp-stall shares (per-instruction
samples of the source page, summed) to <out.csv>.
"""
import csv, json, subprocess, sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors.sum", "lts__t_sectors_srcunit_tex.sum"]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            out[k] = (vals[i], units[i])
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    return name, out


def to_bytes(v):
    val, unit = v
    return float(val.replace(",", "")) * UNIT.get(unit, 1.0)


def stall_shares(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[1]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = {hdr[i]: 0 for i in cols}
    for r in rows[2:]:
        for i in cols:
            tot[hdr[i]] += int(r[i] or 0)
    n = sum(tot.values()) or 1
    return {k: 100.0 * v / n for k, v in sorted(tot.items(), key=lambda x: -x[1])}, len(rows) - 2


def one(out, rep):
    name, m = metrics(rep)
    shares, n_sass = stall_shares(rep)
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["metric", "value", "unit"])
        w.writerow(["kernel", name, ""])
        w.writerow(["sass_instructions", n_sass, ""])
        for k, (v, u) in m.items():
            w.writerow([k, v, u])
        for k, v in shares.items():
            w.writerow([f"stall_share.{k}", f"{v:.2f}", "%"])


def main():
    if sys.argv[1] == "--one":
        one(sys.argv[2], sys.argv[3])
        return
    tag, r64, r32, s64, s32 = sys.argv[1:6]
    prof = Path("profiles")
    summary_path = prof / "ncu_trace_summary.json"
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {}
    for prec, rep, steps in (("fp64", r64, int(s64)), ("fp32", r32, int(s32))):
        name, m = metrics(rep)
        with open(prof / f"ncu_{tag}_{prec}.csv", "w") as f:
            w = csv.writer(f)
            w.writerow(["metric", "value", "unit"])
            w.writerow(["kernel", name, ""])
            for k, (v, u) in m.items():
                w.writerow([k, v, u])
        dram = to_bytes(m["dram__bytes_read.sum"]) + to_bytes(m["dram__bytes_write.sum"])
        summary[prec] = {"capture": tag, "kernel": name, "steps_in_launch": steps,
                         "dram_bytes_in_launch": dram, "dram_bytes_per_step": dram / steps,
                         "duration_ms": float(m["gpu__time_duration.sum"][0]),
                         "issue_active_pct": float(m["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
                         "registers": int(float(m["launch__registers_per_thread"][0]))}
        if "lts__t_sectors.sum" in m:
            l2 = float(m["lts__t_sectors.sum"][0].replace(",", "")) * 32.0
            ms = float(m["gpu__time_duration.sum"][0])
            summary[prec].update(l2_bytes_per_step=l2 / steps, l2_gb_per_s=l2 / (ms * 1e-3) / 1e9,
                                 dram_gb_per_s=dram / (ms * 1e-3) / 1e9,
                                 thread_efficiency=float(m[
                                     "smsp__thread_inst_executed_per_inst_executed.ratio"][0]) / 32,
                                 lts_throughput_pct=float(m[
                                     "lts__throughput.avg.pct_of_peak_sustained_elapsed"][0]),
                                 lsu_wavefronts_pct=float(m[
                                     "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"][0]),
                                 thread_inst_per_step=float(m["smsp__inst_executed.sum"][0].replace(",", "")) *
                                 float(m["smsp__thread_inst_executed_per_inst_executed.ratio"][0]) / steps)
    summary_path.write_text(json.dumps(summary, indent=1) + "\n")
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
