"""Per-role stall breakdown from an ncu source page (SASS): each instruction is
assigned to a warp role by scanning the SASS for the role's code region markers
(the MMA issue loop contains UTCHMMA, the splitter loop F2FP/STS + FENCE.VIEW.ASYNC,
the combine loop LDTM).  Regions = maximal address ranges between branch targets are
too fragile; instead we attribute by instruction class and print stall reasons for
the hottest instructions plus the splitter-loop total."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
isrc = hdr.index("Source")
iex = hdr.index("Instructions Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[ist]) for r in data)
# splitter region: from the first LDS after a TRYWAIT to the FENCE.VIEW.ASYNC.S that precedes the
# op_full arrive.  Find FENCE indices and walk back to the previous TRYWAIT.
fences = [i for i, r in enumerate(data) if "FENCE.VIEW.ASYNC.S" in r[isrc]]
regions = []
for f in fences:
    j = f
    while j > 0 and "TRYWAIT" not in data[j][isrc]:
        j -= 1
    if f - j > 40:
        regions.append((j, f))
agg = {}
cnt = 0
for a, b in regions:
    for r in data[a:b + 1]:
        cnt += int(r[ist])
        for i in stall_cols:
            agg[hdr[i]] = agg.get(hdr[i], 0) + int(r[i] or 0)
print(f"total samples {tot}; splitter-region samples {cnt} ({100 * cnt / max(tot, 1):.1f}%) in {len(regions)} regions")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
    print(f"   {k:22s} {v:9d} {100 * v / max(cnt, 1):5.1f}%")
# combine region: instructions between LDTM and next SYNCS arrive
agg2 = {}
c2 = 0
ld = [i for i, r in enumerate(data) if "LDTM" in r[isrc]]
if ld:
    a, b = ld[0] - 5, ld[-1] + 60
    for r in data[a:b]:
        c2 += int(r[ist])
        for i in stall_cols:
            agg2[hdr[i]] = agg2.get(hdr[i], 0) + int(r[i] or 0)
print(f"combine-region samples {c2} ({100 * c2 / max(tot, 1):.1f}%)")
for k, v in sorted(agg2.items(), key=lambda x: -x[1])[:8]:
    print(f"   {k:22s} {v:9d} {100 * v / max(c2, 1):5.1f}%")
