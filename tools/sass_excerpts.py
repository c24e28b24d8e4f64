"""Opcode counts and short excerpts of the hot kernels' SASS (cuobjdump of the built library):
bulk copies (UBLKCP / UTMALDG), mbarrier traffic (SYNCS), cluster barriers (UCGABAR), FP64
tensor-core MMAs (DMMA), spills (STL / LDL).  python tools/sass_excerpts.py > profiles/...txt"""
import collections
import os
import re
import subprocess

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2605_29284_b200",
                   "librapidkrig_b200.so")
KERNELS = ["row_fwd_split_kernel", "col_split_kernel", "row_inv_split_kernel", "weights_kernel_mma<4, true>",
           "col_kernel<0, true, 1, 1>", "row_fwd_kernel<3, true, 1>", "row_inv_kernel<true, 1>",
           "cs_rowgen_kernel<false, 1, 288, 4, true>", "cs_rowgen_split_kernel<true>", "trmm_panel_kernel<false, 1>"]
KEYS = ["UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "UCGABAR", "BAR.SYNC", "DMMA", "DFMA", "SHFL", "LDG.E.ENL2.256", "STG.E.ENL2.256",
        "STL", "LDL"]

txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", txt)
out = []
for f in funcs[1:]:
    mangled = f.split("\n", 1)[0].strip()
    name = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
    short = re.sub(r"^void ", "", name).replace("rk::", "")
    if not any(k in short.replace("(bool)1", "true").replace("(bool)0", "false") or k in short for k in KERNELS):
        continue
    lines = [l for l in f.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
    ops = collections.Counter()
    for l in lines:
        ins = l.split("*/", 1)[1].strip()
        op = ins.split()[1] if ins.startswith("@") else ins.split()[0]
        for k in KEYS:
            if op.startswith(k):
                ops[k] += 1
    out.append(f"== {short[:110]}  ({len(lines)} SASS instructions)")
    out.append("   " + ", ".join(f"{k} {ops[k]}" for k in KEYS if ops[k]))
    for key in ("UBLKCP", "SYNCS", "DMMA", "UCGABAR"):
        for i, l in enumerate(lines):
            if key in l:
                for ll in lines[max(0, i - 1): i + 2]:
                    out.append("     " + re.sub(r"\s*/\*[^*]*\*/\s*$", "", ll.split("*/", 1)[1]).strip()[:100])
                break
print("\n".join(out))
