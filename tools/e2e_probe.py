import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench, paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import workloads
case = bench.build_predict_case(pk, workloads.cfg2())
flush = bench.L2Flush()
st = case['setup']; m1, m2 = st.grid.interior_dims
ch = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory().numpy() for c in case['cs']]
xg = torch.from_numpy(np.ascontiguousarray(case['xg'])).pin_memory().numpy()
beta = np.ascontiguousarray(case['beta'])
out = torch.empty((m2, m1), dtype=torch.float64).pin_memory().numpy()
for k in range(12): pk.predict_rapid(st, ch[k % len(ch)], beta, xg, out=out)
def run(nc, fl, n=100):
    ts = []
    for k in range(n):
        if fl: flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pk.predict_rapid(st, ch[k % nc], beta, xg, out=out)
        ts.append((time.perf_counter() - t0) * 1e6)
    ts.sort(); return ts[n // 2], ts[n // 10], ts[9 * n // 10]
print('4 bufs flush', run(4, True))
print('4 bufs noflush', run(4, False))
print('1 buf noflush', run(1, False))
print('1 buf flush', run(1, True))
from paper_2605_29284_b200 import _native as N
lib = N.load(); sp = N.stream_ptr()
args = (st.handle, N.ptr(ch[0]), N.ptr(beta), 3, N.ptr(xg), N.ptr(out), sp)
ts=[]
for k in range(100):
    flush(); torch.cuda.synchronize(); t0=time.perf_counter(); lib.rk_predict_host(*args); ts.append((time.perf_counter()-t0)*1e6)
ts.sort(); print('raw ctypes flush', ts[50], ts[10], ts[90])
ms, h2d, d2h = bench.time_predict_e2e(pk, case, 50, 5, flush)
ms = sorted(ms)
print('bench e2e: mean %.1f us median %.1f min %.1f max %.1f' % (1e3 * sum(ms) / len(ms), 1e3 * ms[25], 1e3 * ms[0], 1e3 * ms[-1]))
print([round(1e3 * m) for m in ms[-8:]])
ms, h2d, d2h = bench.time_predict_e2e(pk, case, 50, 5, flush)
ms = sorted(ms)
print('bench e2e again: mean %.1f us median %.1f' % (1e3 * sum(ms) / len(ms), 1e3 * ms[25]))
print('4 bufs flush after', run(4, True))
import gc
print('gc counts', gc.get_count())
