"""Drive tools/microbench on the GPU box and compare normcdfinv against scipy.special.ndtri."""
import json
import subprocess
import sys

import numpy as np
from scipy.special import ndtri

rng = np.random.default_rng(0)
k = rng.integers(0, 1 << 53, size=2_000_000, dtype=np.int64)
# include the extreme words explicitly
k[:4] = [0, 1, (1 << 53) - 1, (1 << 53) - 2]
u = (k.astype(np.float64) + 0.5) / float(1 << 53)
u.tofile("gpurun_out/u.bin")
out = subprocess.run(["./tools/microbench", "gpurun_out/u.bin", "gpurun_out/z.bin"],
                     capture_output=True, text=True, check=True)
res = json.loads(out.stdout.strip().splitlines()[0])
z = np.fromfile("gpurun_out/z.bin")
ref = ndtri(u)
rel = np.abs(z - ref) / np.maximum(np.abs(ref), 1e-300)
res["normcdfinv_max_rel_vs_ndtri"] = float(rel.max())
res["normcdfinv_max_abs_vs_ndtri"] = float(np.abs(z - ref).max())
res["normcdfinv_frac_bit_equal"] = float(np.mean(z == ref))
print(json.dumps(res))
with open("gpurun_out/microbench.json", "w") as fh:
    json.dump(res, fh, indent=1)
sys.exit(0)
