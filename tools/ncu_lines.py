"""Executed instructions and stall samples per CUDA source line of one kernel (ncu source page,
-lineinfo builds).  python tools/ncu_lines.py REPORT [N] [file-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
filt = sys.argv[3] if len(sys.argv) > 3 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
out, path = [], ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] and r[0] != "Line No" and r[0].isdigit():
        try:
            samp, inst = float(r[4]), float(r[7])
        except ValueError:
            continue
        out.append((path, int(r[0]), samp, inst, r[1].strip()[:90]))
ts = sum(o[2] for o in out) or 1
ti = sum(o[3] for o in out) or 1
print(f"{len(out)} lines, {ts:.0f} samples, {ti / 1e6:.1f} M warp instructions")
for p, ln, s, i, src in sorted(out, key=lambda o: -o[2])[:top]:
    if filt and filt not in p:
        continue
    print(f"{100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% inst  {p}:{ln}  {src}")
