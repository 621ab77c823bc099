"""Summary of one kernel of an `ncu --page raw --csv` export as JSON (the keys the
profiles/*_ncu_*.json files carry).  python profiles/ab/ncu_summary.py raw.csv [note]"""
import csv
import json
import sys

KEYS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "launch__waves_per_multiprocessor",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]

rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[-1]
out = {"Kernel Name": v[h.index("Kernel Name")]}
for i, k in enumerate(h):
    if k in KEYS or ("issue_stalled" in k and k.endswith("per_issue_active.ratio")
                     and "not_issued" not in k):
        out[k] = f"{v[i]} {u[i]}".strip()
if len(sys.argv) > 2:
    out["_note"] = sys.argv[2]
print(json.dumps(dict(sorted(out.items())), indent=1))
