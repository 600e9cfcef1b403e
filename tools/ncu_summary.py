"""Summarise one `ncu --set full` capture (raw-page CSV exported on the GPU
box by tools/gpu_evidence.sh) into the JSON kept under profiles/: the DRAM,
L1/L2 and stall metrics the roofline discussion uses, plus the kernel's
algorithmic bytes for the captured launch.
Usage: python tools/ncu_summary.py RAW_CSV BENCH_LOG {cg|bi} LAUNCH_INDEX OUT_JSON
(LAUNCH_INDEX: position of the captured launch among the timed launches
listed in the bench line of BENCH_LOG; the bench line's bytes model gives
the index bytes per row)."""
import csv, json, re, sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "sm__cycles_elapsed.avg.per_second"]
try:  # measured HBM copy peak of this pool (driver-written), else the recipe fallback
    PEAK = json.load(open(__file__.rsplit("/", 2)[0] + "/MEASURED_PEAKS.json"))["hbm_gbs"]
except Exception:
    PEAK = 6650.0
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main(raw, log, kind, idx, out):
    rows = [r for r in csv.reader(open(raw)) if r]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    head, units, vals = rows[hi], rows[hi + 1], rows[hi + 2]
    d = {k: {"value": vals[head.index(k)], "unit": units[head.index(k)]} for k in KEYS if k in head}
    line = [l for l in open(log) if l.startswith('{"metric"')][-1]
    b = json.loads(line)
    N, K = b["config"]["cells"], b["config"]["K"]
    m = re.search(r"iters\*N\*\(8K\+([0-9.]+)\+([0-9]+)\)", b["roofline"]["bytes_model"])
    idx_row = float(m.group(1)) if m else 4.0 * K
    vec_row = float(m.group(2)) if m else 96.0
    if kind == "cg":
        it = b["cg_iterations_per_launch"][idx]
        alg = N * (12 * K + 80) + it * N * (8 * K + idx_row + vec_row)
        model = f"N(12K+80) + iters N(8K+{idx_row:g}+{vec_row:g})"
    else:
        it = b["bicgstab_iterations_per_launch"][idx]
        per_row = 600.0 - (2 * (4 * K - idx_row))
        alg = it * N * per_row
        model = f"{per_row:g} B per row and batched iteration (DESIGN.md §3)"
    t = float(d["gpu__time_duration.sum"]["value"]) * SCALE[d["gpu__time_duration.sum"]["unit"]]
    dram = sum(float(d[k]["value"]) * SCALE[d[k]["unit"]]
               for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    d["_derived"] = {"iterations_this_launch": it, "algorithmic_bytes": alg,
                     "algorithmic_model": model, "dram_bytes": dram,
                     "dram_over_algorithmic": dram / alg,
                     "dram_bytes_per_row_iteration": dram / (N * it),
                     "dram_gbs_physical": dram / t / 1e9, "frac_of_measured_peak": dram / t / 1e9 / PEAK,
                     "algorithmic_gbs": alg / t / 1e9, "duration_s": t,
                     "note": "ncu serialises and replays; SM clock under ncu as listed "
                             "(clock-control none, power cap)"}
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d["_derived"]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), sys.argv[5])
