"""Copy one round's ncu evidence into profiles/: the raw-metric summaries of the
full captures (profiles/rNN_ncu_final.json), the DRAM traffic per launch that
bench.py reports as roofline.traffic (profiles/traffic.json) and the launch list.

  python tools/update_profiles.py TAG [ROUND]   (reads gpurun_out/prof_*_TAG.ncu-rep; ROUND e.g. r02)
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402


def val(s):
    x, unit = s.split()[0], s.split()[1] if len(s.split()) > 1 else ""
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(x.replace(",", "")) * mult


def main():
    tag = sys.argv[1]
    rnd = sys.argv[2] if len(sys.argv) > 2 else "r02"
    out = os.path.join(ROOT, "gpurun_out")
    reps = {}
    for c in ("c2_fp16", "c2_tf32", "c3_fp16"):
        rep = os.path.join(out, f"prof_{c}_{tag}.ncu-rep")
        reps[c] = rep if os.path.exists(rep) else os.path.join(out, f"prof_{c}_{tag}.raw.csv")
    summ, traffic = {}, {}
    for c, rep in reps.items():
        if not os.path.exists(rep):
            continue
        d = ncu_summary.raw(rep)
        summ[c] = d
        rd, wr = val(d["dram__bytes_read.sum"]), val(d["dram__bytes_write.sum"])
        traffic[c] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                      "kernel": d["Kernel Name"], "ncu_duration": d["gpu__time_duration.sum"],
                      "source": f"ncu --set full --clock-control none, one launch ({rnd}, {tag})"}
    json.dump(summ, open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_final.json"), "w"), indent=1)
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    lst = os.path.join(out, f"launches_c2_fp16_{tag}.csv")
    if os.path.exists(lst):
        shutil.copy(lst, os.path.join(ROOT, "profiles", f"{rnd}_launches_c2_fp16.csv"))
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
