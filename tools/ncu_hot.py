"""Top SASS instructions of one kernel by warp-stall samples (ncu source page), with the stall
columns that dominate.  python tools/ncu_hot.py REPORT KERNEL_REGEX [N] [launch_skip]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 2 and r[0].startswith("0x")]
iS = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i != iS]
tot = sum(float(r[iS] or 0) for r in data if len(r) > iS)
print(f"{len(data)} SASS lines, {tot:.0f} samples")
order = sorted(range(len(data)), key=lambda i: -float(data[i][iS] or 0))
for i in sorted(order[:top]):
    r = data[i]
    print(f"{i:5d} {float(r[iS]):7.0f} {100*float(r[iS])/tot:5.1f}%  {r[1].strip()[:90]}")
