"""Warp-stall samples of one kernel split into regions at barrier instructions (BAR.SYNC /
UCGABAR), with the dominant stall reasons per region.  python tools/ncu_regions.py REPORT KERNEL"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
iS = hdr.index("Warp Stall Sampling (All Samples)")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[iS]) for r in data)
cuts = [0] + [i + 1 for i, r in enumerate(data) if "BAR.SYNC" in r[1] or "UCGABAR_WAIT" in r[1]] + [len(data)]
print(f"{len(data)} SASS lines, {tot:.0f} samples, {len(cuts) - 2} barriers")
for a, b in zip(cuts, cuts[1:]):
    s = sum(float(r[iS]) for r in data[a:b])
    if s / tot < 0.01:
        continue
    reasons = collections.Counter()
    for r in data[a:b]:
        for i in st:
            reasons[hdr[i][6:]] += float(r[i] or 0)
    top = ", ".join(f"{k} {100 * v / max(s, 1):.0f}%" for k, v in reasons.most_common(4))
    ops = collections.Counter(r[1].split()[1 if r[1].strip().startswith("@") else 0].split(".")[0] for r in data[a:b])
    print(f"[{a:5d},{b:5d}) {100 * s / tot:5.1f}%  {top}   ops: {dict(ops.most_common(5))}")
