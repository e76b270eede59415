"""Side-by-side key metrics and stall reasons of ncu raw CSV exports: python tools/ncu_cmp.py a_raw.csv b_raw.csv ..."""
import csv
import sys


def load(p):
    rows = list(csv.reader(open(p)))
    return dict(zip(rows[0], rows[2]))


ds = [load(p) for p in sys.argv[1:]]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "sm__sass_inst_executed_op_local_ld.sum", "sm__sass_inst_executed_op_local_st.sum"]
for k in keys:
    print(f"{k:62s}", " ".join(f"{d.get(k, '-'):>14s}" for d in ds))
stalls = sorted({k for d in ds for k in d if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")})
for k in stalls:
    vals = []
    for d in ds:
        try:
            vals.append(float(d.get(k, "nan")))
        except ValueError:
            vals.append(float("nan"))
    if max(vals) > 0.04:
        print(f"  stall {k.split('stalled_')[1].replace('_per_issue_active.ratio', ''):54s}",
              " ".join(f"{v:14.3f}" for v in vals))
