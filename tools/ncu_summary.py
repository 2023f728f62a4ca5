"""Summarise an ncu --set full report: key raw metrics, and per-role stall/issue
attribution over the SASS (roles are found from the source-line mapping)."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active"]


def raw(rep):
    """rep: an .ncu-rep, or the `ncu -i REP --page raw --csv` export of one (.csv)"""
    if rep.endswith(".csv"):
        with open(rep) as f:
            out = f.read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {"Kernel Name": v[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            d[k] = (v[h.index(k)] + " " + u[h.index(k)]).strip()
    return d


if __name__ == "__main__":
    res = {rep: raw(rep) for rep in sys.argv[1:]}
    print(json.dumps(res, indent=1))
