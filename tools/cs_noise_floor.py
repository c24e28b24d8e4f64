"""The reference's own floor for unconditional-field parity: the same field computed with the
circulant eigenvalues lambda = Re fft2(lag table) from numpy.fft (what simulate.py:77-100 uses)
and from scipy.fft (an equally valid FFT).  sqrt(lambda) amplifies the rounding of near-zero
eigenvalues, so the two fields differ -- any implementation that is not bit-identical to
pocketfft sits at this floor.  Usage: python tools/cs_noise_floor.py [cfg4|cfg5] [n_fields]"""
import sys

import numpy as np
import scipy.fft

sys.path.insert(0, ".")
from oracle import rk_oracle as ro
from paper_2605_29284_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 8
wl = workloads.cfg4() if name == "cfg4" else workloads.cfg5(nu=1.5, L=4, m=4096)
om = ro.Model(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
og = ro.make_grid(wl.domain, wl.dims, wl.L, wl.obs)
p1, p2, rootA = ro.embedding_root(om, og)
lam = scipy.fft.fft2(om.cov(ro.torus_lags(og, p1, p2)), workers=8).real
rootB = np.sqrt(np.clip(lam, 0, None))
print(name, "torus", (p1, p2), "max |d sqrt(lambda)|", np.abs(rootA - rootB).max(), "max sqrt(lambda)", rootA.max())
gs_a, gs_b = [], []
for j in range(nf):
    s = ro.sub_seed(ro.sub_seed(0, j), 101)
    ga = ro.uncond_field(om, og, s, (p1, p2, rootA))
    gb = ro.uncond_field(om, og, s, (p1, p2, rootB))
    gs_a.append(ga)
    gs_b.append(gb)
    print(j, "field rel diff (numpy.fft vs scipy.fft eigenvalues)", np.abs(ga - gb).max() / np.abs(ga).max(), flush=True)
if nf > 1:
    sa, sb = np.stack(gs_a).std(0, ddof=1), np.stack(gs_b).std(0, ddof=1)
    print("std of fields rel diff", np.abs(sa - sb).max() / np.abs(sa).max())
