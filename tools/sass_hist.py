"""SASS opcode histogram of the built libraries (CPU; cuobjdump): per kernel,
the instructions that prove the Blackwell path -- tcgen05 MMAs (UTCHMMA /
UTCQMMA, .2CTA = cta_group::2), TMEM loads/stores (LDTM / STTM), TMA
(UTMALDG / UTMASTG / UTMAPF), cluster launch control (UGETNEXTWORKID = try_cancel), the packed FP32 math of the combine (FFMA2 /
FADD2 / FMUL2) and the split's conversions (F2FP).  Writes
profiles/r02_sass_hist.json.

    python tools/sass_hist.py
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBS = ["paper_2308_15152_b200/libemusgemm.so", "probe/libtcprobe.so"]
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAPF", "FFMA2", "FADD2",
        "FMUL2", "F2FP", "HFMA2", "LDS", "STS", "LDG", "STG", "SYNCS", "ELECT", "BAR", "MEMBAR", "UGETNEXTWORKID"]


def main():
    out = {}
    for lib in LIBS:
        path = os.path.join(ROOT, lib)
        if not os.path.exists(path):
            continue
        sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
        kern = None
        per = collections.defaultdict(collections.Counter)
        for line in sass.splitlines():
            m = re.match(r"\s+Function : (\S+)", line)
            if m:
                kern = m.group(1)
                continue
            m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m and kern:
                op = m.group(1)
                base = op.split(".")[0]
                for k in KEYS:
                    if base == k or (k in ("UTCHMMA", "UTCQMMA") and base.startswith(k)):
                        per[kern][op if k in ("UTCHMMA", "UTCQMMA", "UTMALDG") else base] += 1
        total = collections.Counter()
        for c in per.values():
            total.update(c)
        demangled = {}
        names = list(per)
        if names:
            dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
            demangled = dict(zip(names, dm))
        out[lib] = {"total": dict(sorted(total.items())),
                    "kernels": {demangled.get(k, k)[:160]: dict(sorted(v.items())) for k, v in per.items()}}
    dst = os.path.join(ROOT, "profiles", "r02_sass_hist.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    for lib, v in out.items():
        print(lib, v["total"])
    print("wrote", dst, file=sys.stderr)


if __name__ == "__main__":
    main()
