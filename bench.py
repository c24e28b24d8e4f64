"""Benchmark of the B200 rapid-Kriging hot path (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-extra]

Headline (``value``): predicted grid points/s (fp64) on the largest single-GPU BASELINE
configuration, configs[4]'s largest cell: n = 50000 U[0,1]^2 observations, 4096 x 4096 grid,
L = 4 (M = 64), Matern nu = 2.5 (its worst-conditioned smoothness), 8748^2 circulant torus.
A step is SURVEY 8(d)'s T_predict = K1 + T_apply: the per-observation weights kernel
(stencils, Matern cross covariances, K_N substitutions) followed by predict_rapid (scatter,
3-pass FFT convolution, fixed part), from inputs resident in HBM, L2 flushed before every
step, CUDA events on the launching stream, max over ranks.  ``apply_only`` reports N/T_apply.
Under torchrun each rank runs an independent replica ("replicas only": a single predict
does not shard; the fit / setup are built on rank 0 and broadcast), and ``value`` = points of
all ranks / max-over-ranks time.  ``e2e`` = the same step through the public API on pinned
HOST buffers (H2D of c / beta, D2H of the field inside the timed region).
``extra.cs_cfg4`` / ``extra.cs_cfg5``: CS realizations/s for configs[3] (R = 1024, n = 5000,
512^2, L = 3) and configs[4]'s CS (R = 256, n = 50000, 4096^2, L = 4, nu = 1.5), realizations
sharded over the ranks (one int64 all-reduce), each with its roofline and CPU baseline.
With ``--gpus N`` and no torchrun environment the script relaunches itself under
torch.distributed.run with N processes.

``--impl reference`` times the reference algorithm's CPU implementation (the numpy oracle
port, oracle/rk_oracle.py -- /root/reference is not on the GPU box) on the box's host cores
(one process per core) on the same workload and metric, rank 0 only.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
FP64_TFLOPS_MEASURED = 34.0       # tools/microbench.cu DFMA loop on this pool (profiles/round1_microbench.json)
PHILOX_GWORDS_MEASURED = 411.16   # same microbenchmark: Philox4x64-10 words/s (the CS integer roof)
HEADLINE = dict(nu=2.5, L=4, m=4096)
HEADLINE_NAME = "cfg5: predict (K1 + apply), n=50000 U[0,1]^2, 4096x4096, L=4, nu=2.5, range 0.05 (configs[4] largest cell)"


def headline_config(world, embed, padded):
    """The headline line's `config`, identical for both arms (`--impl reference` prints it too)."""
    return {"workload": HEADLINE_NAME, "step": "K1 (weights kernel) + predict_rapid (T_predict, SURVEY 8(d))",
            "embed": [int(v) for v in embed], "padded": [int(v) for v in padded],
            "l2": "flushed (256 MB write) before every timed step", "parallelism": f"replicas x{world}"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout=5.0):
        t0 = time.perf_counter()
        while self.proc and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if "Active" in v and "Not" not in v:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def relaunch_under_torchrun(n):
    """--gpus N without a torchrun environment: re-exec as N processes (one per GPU)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execvp(cmd[0], cmd)


class L2Flush:
    def __init__(self):
        import torch
        self.buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MB > L2

    def __call__(self):
        self.buf.zero_()


def fft_flops(n):
    """Real fp64 flops of one complex length-n transform in our radix-9/6/8/4/2 schedule."""
    per_pt = {9: 16.0, 6: 12.7, 8: 10.5, 4: 8.5, 3: 12.0, 2: 6.0}   # codelet + twiddle flops per point
    rad, a, b, m = [], 0, 0, n
    while m % 2 == 0:
        m //= 2
        a += 1
    while m % 3 == 0:
        m //= 3
        b += 1
    rad += [9] * (b // 2)
    b -= 2 * (b // 2)
    if b:
        if a:
            rad.append(6)
            a -= 1
        else:
            rad.append(3)
    rad += [8] * (a // 3)
    a -= 3 * (a // 3)
    if a:
        rad.append(4 if a == 2 else 2)
    return n * sum(per_pt[r] for r in rad)


def _ncu(cfg, kernel, key):
    """A per-launch number of `kernel` from the committed ncu --set full capture."""
    for name in ("round2_traffic.json", "round1_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return json.load(f)["kernels"][cfg][kernel][key], f"profiles/{name}"
        except (OSError, KeyError, ValueError):
            continue
    return None, None


# ------------------------------------------------------------------ predict headline
def build_predict_case(pk, wl, world, rank, c_variants=4):
    """Inputs of one predict workload, resident in HBM: fit (rank 0; broadcast to the other
    ranks), setup (rank 0; broadcast), c variants, beta, grid covariates."""
    import torch
    from paper_2605_29284_b200 import workloads
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    t0 = time.perf_counter()
    f = pk.fit(model, wl.obs, wl.z, wl.X) if rank == 0 else None
    torch.cuda.synchronize()
    t_fit = time.perf_counter() - t0
    t0 = time.perf_counter()
    grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
    st = pk.build_setup(model, grid, wl.L, wl.obs) if rank == 0 else None
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    t_bcast = 0.0
    if world > 1:
        from paper_2605_29284_b200.distributed import broadcast_fit, broadcast_setup
        t0 = time.perf_counter()
        f = broadcast_fit(f)
        st = broadcast_setup(st)
        torch.cuda.synchronize()
        t_bcast = time.perf_counter() - t0
    xg = workloads.grid_covariates_for(grid.interior_nodes(), wl.grid_covariates)
    rng = np.random.default_rng(123)
    c0 = np.asarray(f.c)
    cs = [c0 * (1.0 + 1e-3 * k) + (0 if k == 0 else 1e-3 * rng.normal(size=c0.shape)) for k in range(c_variants)]
    return dict(model=model, fit=f, grid=grid, setup=st, xg=xg, cs=cs, beta=np.asarray(f.beta_hat),
                t_fit=t_fit, t_setup=t_setup, t_bcast=t_bcast)


class K1Buffers:
    """Device buffers the per-step weights kernel (K1) writes into."""

    def __init__(self, st):
        import torch
        n, M = st.n_obs, st.block_size
        self.base = torch.empty(n, dtype=torch.int32, device="cuda")
        self.w = torch.empty((n, M), dtype=torch.float64, device="cuda")
        self.cv = torch.empty(n, dtype=torch.float64, device="cuda")
        self.err = torch.tensor([2 ** 31 - 1, 2 ** 31 - 1, 0, 0], dtype=torch.int32, device="cuda")

    def launch(self, st, stream=None):
        from paper_2605_29284_b200 import _native as N
        N.call("rk_setup_weights_into", st.handle, N.ptr(self.base), N.ptr(self.w), N.ptr(self.cv),
               N.ptr(self.err), N.stream_ptr(stream))


def time_predict_device(pk, case, steps, warmup, flush, with_k1=True, soak_s=0.0):
    """Device-resident step (K1 + predict, or predict alone): per-step CUDA-event time on the
    launching stream, L2 flushed before each step."""
    import torch
    from paper_2605_29284_b200 import _native as N
    st = case["setup"]
    k1 = K1Buffers(st)
    cds = [torch.as_tensor(c, device="cuda") for c in case["cs"]]
    bd = torch.as_tensor(case["beta"], device="cuda")
    xd = None if case["xg"] is None else torch.as_tensor(case["xg"], device="cuda").contiguous()
    m1, m2 = st.grid.interior_dims
    out = torch.empty((m2, m1), dtype=torch.float64, device="cuda")

    def step(k):
        if with_k1:
            k1.launch(st)
        pk.predict_rapid(st, cds[k % len(cds)], bd, xd, out=out)

    for k in range(warmup):
        step(k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < soak_s:
        for k in range(10):
            flush()
            step(k)
        torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    l0 = N.launch_count()
    for k in range(steps):
        flush()
        ev[k][0].record()
        step(k)
        ev[k][1].record()
    torch.cuda.synchronize()
    launches = N.launch_count() - l0
    assert int(k1.err[2].item()) == 0
    return [a.elapsed_time(b) for a, b in ev], launches, out


def time_predict_e2e(pk, case, steps, warmup, flush):
    """Public API on pinned HOST buffers: K1 + predict_rapid(host c, beta) -> host field
    (H2D of c / beta and D2H of the field inside the timed region)."""
    import torch
    st = case["setup"]
    m1, m2 = st.grid.interior_dims
    k1 = K1Buffers(st)
    ch = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory().numpy() for c in case["cs"]]
    xg = None if case["xg"] is None else torch.from_numpy(np.ascontiguousarray(case["xg"])).pin_memory().numpy()
    beta = np.ascontiguousarray(case["beta"])
    out = torch.empty((m2, m1), dtype=torch.float64).pin_memory().numpy()
    t_w = time.perf_counter()
    k = 0
    while k < max(warmup, 2 * len(ch) + 1) or time.perf_counter() - t_w < 0.5:
        k1.launch(st)
        pk.predict_rapid(st, ch[k % len(ch)], beta, xg, out=out)
        k += 1
    ms = []
    gc.disable()
    try:
        for k in range(steps):
            flush()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            k1.launch(st)
            pk.predict_rapid(st, ch[k % len(ch)], beta, xg, out=out)
            ms.append((time.perf_counter() - t0) * 1e3)
    finally:
        gc.enable()
    h2d = 8 * (ch[0].size + beta.size + (0 if xg is None else xg.size))
    return ms, h2d, 8 * m1 * m2


def profile_passes(pk, case, reps, flush):
    """Per-pass kernel times (CUDA events on the launching stream) and algorithmic bytes."""
    import ctypes as C
    import torch
    from paper_2605_29284_b200 import _native as N
    st = case["setup"]
    cd = torch.as_tensor(case["cs"][0], device="cuda")
    bd = torch.as_tensor(case["beta"], device="cuda")
    xd = None if case["xg"] is None else torch.as_tensor(case["xg"], device="cuda").contiguous()
    p = int(bd.numel())
    m1, m2 = st.grid.interior_dims
    out = torch.empty((m2, m1), dtype=torch.float64, device="cuda")
    acc = np.zeros(4)
    for r in range(reps + 1):
        flush()
        ms = (C.c_float * 4)()
        N.call("rk_predict_profile", st.handle, N.ptr(cd), N.ptr(bd), p, N.ptr(xd), N.ptr(out),
               N.stream_ptr(), C.byref(ms))
        if r:
            acc += np.array(list(ms))
    b = (C.c_double * 4)()
    N.call("rk_predict_traffic", st.handle, p if xd is not None else 0, C.byref(b))
    return acc / reps, np.array(list(b))


def weights_k1(case, reps=20):
    """K1 alone: the per-observation weights kernel (back-to-back launches), with its FP64 rate
    against F_w = n (2 M^2 + 20 M)."""
    import ctypes as C
    from paper_2605_29284_b200 import _native as N
    st = case["setup"]
    ms = C.c_float(0.0)
    N.call("rk_setup_time_weights", st.handle, N.stream_ptr(), reps, C.byref(ms))
    n, M = st.n_obs, st.block_size
    flops = n * (2 * M * M + 20 * M)
    tf = flops / (ms.value * 1e-3) / 1e12
    return {"ms": round(ms.value, 5), "n": n, "M": M, "flops": flops, "fp64_tflops": round(tf, 3),
            "fp64_peak_tflops": FP64_TFLOPS_MEASURED, "fp64_frac": round(tf / FP64_TFLOPS_MEASURED, 4),
            "what": "weights kernel alone (rapid.py:202-225), back-to-back launches; F_w = n(2M^2+20M)"}


def cufft_reference(pk, case, reps, flush):
    """Reference point only (north_star): the same convolution + crop + fixed part with fp64
    cuFFT (torch.fft rfft2 / irfft2) on c* from our scatter, L2 flushed; (ms, max rel diff)."""
    import torch
    st = case["setup"]
    g = st.grid
    cd = torch.as_tensor(case["cs"][0], device="cuda")
    bd = torch.as_tensor(case["beta"], device="cuda")
    xd = None if case["xg"] is None else torch.as_tensor(case["xg"], device="cuda").contiguous()
    p1, p2 = st.embed_dims
    M1, M2 = g.total_dims
    m1, m2 = g.interior_dims
    l, _, b, _ = g.pad
    spec = torch.as_tensor(np.ascontiguousarray(np.asarray(st.filter_spectrum).real[:, : p1 // 2 + 1]),
                           device="cuda")
    cstar = st.coefficients_to_grid(cd)
    xpad = torch.zeros((p2, p1), dtype=torch.float64, device="cuda")

    def conv():
        xpad[:M2, :M1].copy_(cstar)
        y = torch.fft.irfft2(torch.fft.rfft2(xpad) * spec, s=(p2, p1))
        f = y[b:b + m2, l:l + m1]
        if xd is not None:
            return f + (xd @ bd).reshape(m2, m1)
        return f + bd[0]

    for _ in range(2):
        conv()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for k in range(reps):
        flush()
        ev[k][0].record()
        conv()
        ev[k][1].record()
    torch.cuda.synchronize()
    ours = pk.predict_rapid(st, cd, bd, xd)
    ref = conv()
    diff = float((ours - ref).abs().max() / ref.abs().max())
    del spec, xpad
    torch.cuda.empty_cache()
    return statistics.median(a.elapsed_time(b) for a, b in ev), diff


def predict_roofline(case, pass_ms, pass_bytes, k1, step_ms, peaks, peaks_kind, cfg):
    """Dominant kernel of the step (algorithmic bytes / its event time vs the HBM peak), plus the
    whole step against both roofs: HBM (B_apply + K1 bytes) and FP64 (FFT + K1 flops)."""
    st = case["setup"]
    p1, p2 = st.exec_dims   # the torus the passes run on (the reference's, or shorter along y)
    H1 = p1 // 2 + 1
    m1, m2 = st.grid.interior_dims
    M1, M2 = st.grid.total_dims
    n, M = st.n_obs, st.block_size
    flops = [0.0, (M2 + 1) // 2 * fft_flops(p1), H1 * 2 * fft_flops(p2), (m2 + 1) // 2 * fft_flops(p1)]
    names = ["gather_cstar", "pass1_gather_rowfft", "pass2_column_filter", "pass3_rowifft_epilogue"]
    dom = int(np.argmax(pass_ms))
    ach = pass_bytes[dom] / (pass_ms[dom] * 1e-3) / 1e9
    peak = float(peaks.get("hbm_gbs", 6650.0))
    fl = flops[dom] / (pass_ms[dom] * 1e-3) / 1e12
    b_k1 = n * (16 + 8 * M + 8 + 4)   # obs in; weights, cond_var, base out
    b_step = float(sum(pass_bytes)) + b_k1
    f_step = float(sum(flops)) + k1["flops"]
    t_hbm = b_step / (peak * 1e9) * 1e3
    t_fp64 = f_step / (FP64_TFLOPS_MEASURED * 1e12) * 1e3
    traffic, tsrc = _ncu(cfg, names[dom], "dram_bytes")
    smem, _ = _ncu(cfg, names[dom], "smem_busy_frac")
    return {
        "bound": "hbm", "kernel": names[dom], "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
        "frac": round(ach / peak, 4), "traffic": traffic, "peak_source": peaks_kind,
        "traffic_source": tsrc and f"{tsrc} (ncu --set full, dram bytes per launch)",
        "algorithmic_bytes": float(pass_bytes[dom]), "kernel_ms": round(float(pass_ms[dom]), 5),
        "fp64_tflops": round(fl, 3), "fp64_peak_tflops": FP64_TFLOPS_MEASURED,
        "fp64_frac": round(fl / FP64_TFLOPS_MEASURED, 4), "smem_busy_frac": smem,
        "step": {"ms": round(step_ms, 5), "bytes": b_step, "flops": f_step,
                 "hbm_roof_ms": round(t_hbm, 5), "fp64_roof_ms": round(t_fp64, 5),
                 "binding": "fp64" if t_fp64 > t_hbm else "hbm",
                 "frac_of_binding_roof": round(max(t_hbm, t_fp64) / step_ms, 4),
                 "hbm_frac": round(t_hbm / step_ms, 4), "fp64_frac": round(t_fp64 / step_ms, 4),
                 "what": "whole step (K1 + 3 predict passes): algorithmic bytes / HBM peak and FFT + "
                         "weights flops / measured DFMA peak vs the measured step time"},
        "passes": {names[i]: {"ms": round(float(pass_ms[i]), 5),
                              "GB/s": round(pass_bytes[i] / (pass_ms[i] * 1e-3) / 1e9, 1),
                              "fp64_TF/s": round(flops[i] / (pass_ms[i] * 1e-3) / 1e12, 3)}
                   for i in range(4) if pass_bytes[i] > 0},
    }


# ------------------------------------------------------------------ CS
def cs_roofline(setup, f_n, p, S, ms_per_real, peaks):
    """Per realization: bytes, FP64 flops and Philox words of the CS pipeline against the HBM,
    FP64 and integer (Philox) roofs; the largest roof time binds."""
    from paper_2605_29284_b200.simulate import embedding_dims
    ps1, ps2, _ = embedding_dims(setup.model, setup)
    M1, M2 = setup.grid.total_dims
    m1, m2 = setup.grid.interior_dims
    n, M = setup.n_obs, setup.block_size
    p1, p2 = setup.exec_dims
    H1, G, Npix, Ps = p1 // 2 + 1, M1 * M2, m1 * m2, ps1 * ps2
    b_apply = n * (8 * M + 16) + 16 * H1 * M2 + 8 * H1 * (p2 // 2 + 1) + 16 * H1 * m2 + 16 * H1 * m2 + 8 * Npix
    b = (32 * M1 * ps2 + 8 * G            # row generator writes V, column pass reads V, writes g
         + 16 * n * M + 24 * n            # local observations
         + 8 * n * n / S + 32 * n         # refit: the inverse factor read twice per super-batch, panels
         + b_apply + 24 * Npix)           # predict with the draw epilogue, moments
    fl = (ps2 * fft_flops(ps1) + (M1 + 1) // 2 * fft_flops(ps2)     # unconditional field
          + 40.0 * 2 * Ps                                          # inverse normals
          + 2.0 * n * n                                            # refit (two triangular products)
          + (M2 + 1) // 2 * fft_flops(p1) + H1 * 2 * fft_flops(p2) + (m2 + 1) // 2 * fft_flops(p1))
    words = 2.0 * Ps
    peak = float(peaks.get("hbm_gbs", 6650.0))
    t = {"hbm": b / (peak * 1e9), "fp64": fl / (FP64_TFLOPS_MEASURED * 1e12), "int_philox": words / (PHILOX_GWORDS_MEASURED * 1e9)}
    bind = max(t, key=t.get)
    meas = ms_per_real * 1e-3
    return {"bound": bind, "achieved": round(t[bind] / meas, 4), "peak": 1.0, "unit": "fraction of the binding roof",
            "frac": round(t[bind] / meas, 4), "traffic": None,
            "roof_us": {k: round(v * 1e6, 2) for k, v in t.items()}, "measured_us": round(meas * 1e6, 2),
            "bytes": b, "fp64_flops": fl, "philox_words": words,
            "peaks": {"hbm_gbs": peak, "fp64_tflops": FP64_TFLOPS_MEASURED, "philox_gwords_s": PHILOX_GWORDS_MEASURED},
            "what": "per realization: B_cs / HBM, F_cs / FP64 (FFTs, inverse normals, 2n^2 refit), "
                    "2 Ps Philox words / measured Philox rate; frac = binding roof time / measured time"}


def refit_roofline(fit, S, reps=3):
    import ctypes as C
    from paper_2605_29284_b200 import _native as N
    ms = (C.c_float * 2)()
    N.call("rk_refit_profile", fit.handle, int(S), reps, N.stream_ptr(), C.byref(ms))
    n = fit.n_obs
    fl = float(n) * n * S   # n(n+1)/2 multiply-adds per column and product
    return {"S": int(S), "ms": [round(ms[0], 4), round(ms[1], 4)],
            "fp64_tflops": [round(fl / (m * 1e-3) / 1e12, 2) for m in ms], "fp64_peak_tflops": FP64_TFLOPS_MEASURED,
            "what": "refit's two triangular panel products (L^-1 Z, L^-T H) on FP64 tensor cores (DMMA), "
                    "S right-hand sides; flops = n^2 S each"}


def bench_cs(pk, wl, R, steps, warmup, rank, world, label, batch=64):
    import torch
    from paper_2605_29284_b200 import _native as N
    from paper_2605_29284_b200.distributed import broadcast_fit, broadcast_setup, generate_ensemble_sharded
    from paper_2605_29284_b200.simulate import embedding_dims
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    t0 = time.perf_counter()
    f = pk.fit(model, wl.obs, wl.z) if rank == 0 else None
    grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
    st = pk.build_setup(model, grid, wl.L, wl.obs) if rank == 0 else None
    if rank == 0:
        emb = embedding_dims(model, st)
        f.prepare_refit()
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    t_b = 0.0
    if world > 1:
        t0 = time.perf_counter()
        f = broadcast_fit(f)
        st = broadcast_setup(st)
        torch.cuda.synchronize()
        t_b = time.perf_counter() - t0
    emb = embedding_dims(model, st)
    seed = wl.extra["ens_seed"]
    for _ in range(max(1, warmup)):
        generate_ensemble_sharded(f, st, R, seed, batch=batch)
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = N.launch_count()
    ev0.record()
    for _ in range(steps):
        generate_ensemble_sharded(f, st, R, seed, batch=batch)
    ev1.record()
    torch.cuda.synchronize()
    launches = N.launch_count() - l0
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    barrier(world)
    t0 = time.perf_counter()   # e2e: public API, mean / SE copied to the host inside the timed region
    for _ in range(steps):
        ens_h = generate_ensemble_sharded(f, st, R, seed, batch=batch, host=True)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3, world)
    m1, m2 = grid.interior_dims
    ms_real = ms / steps / R
    S = min(-(-R // world), max(batch, int(16e9 / (8.0 * grid.total_dims[0] * grid.total_dims[1]))))
    out = {
        "metric": "CS realizations/s", "value": round(R * steps / (ms * 1e-3), 2), "unit": "realizations/s",
        "config": {"workload": label, "cs_torus": list(emb[:2]), "doubled": bool(emb[2]), "batch": batch,
                   "sharding": f"contiguous realization blocks over {world} rank(s), 1 int64 all-reduce",
                   "parallelism": f"cs x{world}"},
        "n_gpus": world, "steps": steps, "ms_per_ensemble": round(ms / steps, 3),
        "ms_per_realization": round(ms_real, 5), "setup_s": round(t_setup, 3), "broadcast_s": round(t_b, 3),
        "gpu_launches": int(launches),
        "e2e": {"value": round(R * steps / (e2e_ms * 1e-3), 2), "unit": "realizations/s",
                "h2d_bytes_per_step": 8, "d2h_bytes_per_step": 16 * m1 * m2},
        "se_mean": float(np.mean(ens_h.empirical_se)),
        "roofline": cs_roofline(st, st.n_obs, 1, S, ms_real * world, _peaks()[0]),
        "refit": refit_roofline(f, S),
    }
    return out


# ------------------------------------------------------------------ CPU legs (oracle port)
def _cpu_predict_leg(q, nu, L, m, n_predicts):
    """Oracle port (numpy/pocketfft, one core) of the headline step: K1 (rapid.py:200-225) +
    predict_rapid, on the same seeded inputs; bounded sample of n_predicts steps."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, ROOT)
    from oracle import rk_oracle as ro
    from paper_2605_29284_b200 import workloads
    wl = workloads.cfg5(nu=nu, L=L, m=m)
    model = ro.Model(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    og = ro.make_grid(wl.domain, wl.dims, wl.L, wl.obs)
    ost = ro.rapid_setup(model, og, wl.L, wl.obs)
    c = np.random.default_rng(123).normal(size=wl.obs.shape[0])
    times = []
    for _ in range(n_predicts):
        t0 = time.perf_counter()
        ro.rapid_weights(model, og, wl.L, wl.obs, ost.chol)
        ro.predict(ost, c, np.array([1.0]))
        times.append(time.perf_counter() - t0)
    q.put(("predict", times))


def _cs_worker(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    name, j = args
    from oracle import rk_oracle as ro
    t0 = time.perf_counter()
    W = _CSW[name]
    ro.cond_draw(W["fit"], W["setup"], ro.sub_seed(0, j), None, W["dp"], W["root"])
    return time.perf_counter() - t0


_CSW = {}


def _cpu_cs_leg(q, name, draws, procs):
    """Oracle port of generate_ensemble (simulate.py:174-192) on `draws` realizations with a pool
    of `procs` single-threaded processes (OPENBLAS_NUM_THREADS=1).  cfg4: the oracle's own fit;
    cfg5 (n = 50000): a synthetic diagonal factor of the right size stands in for chol_M (the
    reference fit needs > 62 GB and minutes; it is setup, and the per-draw solves cost the same
    for any factor)."""
    import multiprocessing as mp
    os.environ["OPENBLAS_NUM_THREADS"] = str(os.cpu_count() or 1)
    sys.path.insert(0, ROOT)
    from oracle import rk_oracle as ro
    from paper_2605_29284_b200 import workloads
    wl = workloads.cfg4() if name == "cfg4" else workloads.cfg5(nu=1.5, L=4, m=4096)
    om = ro.Model(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    t0 = time.perf_counter()
    if name == "cfg4":
        fit = ro.exact_fit(om, wl.obs, wl.z)
    else:   # timing sample only: the per-draw refit cost (3 triangular solves) does not depend
        n = wl.obs.shape[0]   # on the factor's values; the n = 50000 fit itself is setup
        fit = ro.Fit(om, wl.obs, np.ones((n, 1)), 2.0 * np.eye(n), np.array([1.0]), np.zeros(n))
    og = ro.make_grid(wl.domain, wl.dims, wl.L, wl.obs)
    st = ro.rapid_setup(om, og, wl.L, wl.obs)
    root = ro.embedding_root(om, og)
    dp = ro.predict(st, fit.c, fit.beta)
    t_setup = time.perf_counter() - t0
    _CSW[name] = dict(fit=fit, setup=st, root=root, dp=dp)
    with mp.get_context("fork").Pool(procs) as pool:
        t0 = time.perf_counter()
        per = pool.map(_cs_worker, [(name, j) for j in range(draws)], chunksize=1)
        wall = time.perf_counter() - t0
    q.put((f"cs_{name}", {"wall_s": wall, "draws": draws, "procs": procs, "per_draw_s": per, "setup_s": t_setup}))


def start_cpu_legs(quick):
    """CPU baselines in separate processes (started after the GPU measurements)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    cores = os.cpu_count() or 1
    legs = [ctx.Process(target=_cpu_predict_leg, args=(q, HEADLINE["nu"], HEADLINE["L"], HEADLINE["m"], 1))]
    legs.append(ctx.Process(target=_cpu_cs_leg, args=(q, "cfg4", 16, min(16, max(1, cores - 2)))))
    if not quick:
        legs.append(ctx.Process(target=_cpu_cs_leg, args=(q, "cfg5", 1, 1)))
    for p in legs:
        p.start()
    return q, legs


def collect_cpu_legs(q, legs, timeout=900):
    res = {}
    t0 = time.perf_counter()
    while len(res) < len(legs) and time.perf_counter() - t0 < timeout:
        try:
            k, v = q.get(timeout=5)
            res[k] = v
        except Exception:
            if not any(p.is_alive() for p in legs):
                break
    for p in legs:
        p.join(timeout=5)
        if p.is_alive():
            p.terminate()
    return res


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------ reference arm
_W = {}


def _ref_worker_init():
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"


def _ref_step(_):
    ro = _W["ro"]
    t0 = time.perf_counter()
    ro.rapid_weights(_W["model"], _W["grid"], _W["L"], _W["obs"], _W["st"].chol)
    ro.predict(_W["st"], _W["c"], _W["beta"])
    return time.perf_counter() - t0


def run_reference(args):
    """The reference algorithm's CPU implementation (numpy oracle port) of the headline step on
    all host cores: the setup (incl. the 8748^2 filter spectrum) is built once in the parent and
    shared copy-on-write with one worker process per core; a step = one K1 + predict in every
    worker at once.  Steps are a bounded sample: after one warm-up round, rounds run until
    args.steps or ~150 s."""
    import multiprocessing as mp
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import rk_oracle as ro
    from paper_2605_29284_b200 import workloads
    wl = workloads.cfg5(**HEADLINE)
    model = ro.Model(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    og = ro.make_grid(wl.domain, wl.dims, wl.L, wl.obs)
    t0 = time.perf_counter()
    st = ro.rapid_setup(model, og, wl.L, wl.obs)
    t_setup = time.perf_counter() - t0
    _W.update(ro=ro, model=model, grid=og, L=wl.L, obs=wl.obs, st=st,
              c=np.random.default_rng(123).normal(size=wl.obs.shape[0]), beta=np.array([1.0]))
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, int(os.environ.get("RK_REF_PROCS", cores))))
    N = wl.dims[0] * wl.dims[1]
    with mp.get_context("fork").Pool(procs, initializer=_ref_worker_init) as pool:
        pool.map(_ref_step, range(procs), chunksize=1)   # warm-up round
        step_s = []
        t_all = time.perf_counter()
        while len(step_s) < max(1, args.steps) and (not step_s or time.perf_counter() - t_all < 150.0):
            t0 = time.perf_counter()
            pool.map(_ref_step, range(procs), chunksize=1)
            step_s.append(time.perf_counter() - t0)
    tot = sum(step_s)
    value = N * procs * len(step_s) / tot
    line = {
        "impl": "reference", "metric": "predicted grid points/s (fp64)", "value": round(value, 1),
        "unit": "points/s", "n_gpus": world, "steps": len(step_s), "warmup": 1,
        "ms_per_step": round(1e3 * tot / len(step_s), 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; BASELINE configs[4] shapes)",
        "config": headline_config(world, st.embed_dims, og.total_dims),
        "cpu_baseline": {"value": round(value, 1), "unit": "points/s", "cores": procs, "kind": "port",
                         "sample": f"{len(step_s)} rounds x {procs} concurrent K1 + predict steps (one process per "
                                   f"core; numpy/pocketfft oracle port of rapid.py:200-261; steps capped at ~150 s "
                                   f"of rounds); setup {t_setup:.1f} s untimed",
                         "cpu": cpu_model(), "openblas_threads": 1},
        "e2e": {"value": round(value, 1), "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip the CS / smaller-config extras")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline legs")
    ap.add_argument("--quick", action="store_true", help="skip the slowest legs (CS cfg5 and its CPU sample)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args)
        return
    if world == 1 and args.gpus > 1:
        relaunch_under_torchrun(args.gpus)
    if world > 1 and args.gpus not in (1, world):
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    args.warmup = max(3, args.warmup)
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        print(f"[bench] rank {rank}/{world}: backend {dist.get_backend()}, cuda:{local} "
              f"({torch.cuda.get_device_name(local)}), NCCL {torch.cuda.nccl.version()}", file=sys.stderr, flush=True)
    cpu = None
    import paper_2605_29284_b200 as pk
    from paper_2605_29284_b200 import workloads
    peaks, peaks_kind = _peaks()
    flush = L2Flush()

    wl = workloads.cfg5(**HEADLINE)
    case = build_predict_case(pk, wl, world, rank)
    barrier(world)
    with ClockSampler(local) as clk:
        clk.wait_first()
        ms, launches, out = time_predict_device(pk, case, args.steps, args.warmup, flush, with_k1=True, soak_s=0.5)
    tot_ms = max_over_ranks(sum(ms), world)
    N = wl.dims[0] * wl.dims[1]
    value = N * args.steps * world / (tot_ms * 1e-3)
    ms_a, _, _ = time_predict_device(pk, case, args.steps, 2, flush, with_k1=False)
    tot_a = max_over_ranks(sum(ms_a), world)
    pass_ms, pass_bytes = profile_passes(pk, case, 5, flush)
    k1 = weights_k1(case, reps=10)
    e2e_ms, h2d, d2h = time_predict_e2e(pk, case, max(args.steps, 20), args.warmup, flush)
    e2e_tot = max_over_ranks(sum(e2e_ms), world)
    cu_ms, cu_diff = cufft_reference(pk, case, 5, flush)
    st = case["setup"]
    line = {
        "metric": "predicted grid points/s (fp64)", "value": round(value, 1), "unit": "points/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_ms / args.steps, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; BASELINE configs[4] shapes: U[0,1]^2 obs, sinusoid-sum z)",
        "config": headline_config(world, st.embed_dims, st.grid.total_dims),
        "setup": {"setup_s": round(case["t_setup"], 3), "fit_s": round(case["t_fit"], 3),
                  "broadcast_s": round(case["t_bcast"], 3), "what": "untimed: fit (rank 0), build_setup (rank 0), "
                                                                   "NCCL broadcast to the other ranks"},
        "e2e": {"value": round(N * len(e2e_ms) * world / (e2e_tot * 1e-3), 1), "unit": "points/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "roofline": predict_roofline(case, pass_ms, pass_bytes, k1, tot_ms / args.steps, peaks, peaks_kind, "cfg5"),
        "gpu_launches": int(launches),
        "apply_only": {"value": round(N * args.steps * world / (tot_a * 1e-3), 1), "unit": "points/s",
                       "ms": round(tot_a / args.steps, 5), "what": "N / T_apply (predict_rapid alone, no K1)"},
        "weights_k1": k1,
        "cufft_reference": {"ms": round(cu_ms, 4), "ours_apply_ms": round(tot_a / args.steps, 4),
                            "max_rel_diff": cu_diff,
                            "what": "reference point only: c* (ours) -> torch.fft rfft2 x spectrum -> irfft2 -> "
                                    "crop + fixed part, fp64 cuFFT, L2 flushed"},
        "clocks": {**clk.summary(), "window": "0.5 s soak of the same flushed steps + the timed steps"},
    }
    del case
    torch.cuda.empty_cache()
    extra = {}
    if not args.no_extra:
        extra["cs_cfg4"] = bench_cs(pk, workloads.cfg4(), 1024, 2, 1, rank, world,
                                    "cfg4: n=5000, 512x512, L=3, nu=1.5, R=1024, seed 0 (configs[3])")
        torch.cuda.empty_cache()
        if not args.quick:
            extra["cs_cfg5"] = bench_cs(pk, workloads.cfg5(nu=1.5, L=4, m=4096), 256, 1, 1, rank, world,
                                        "cfg5: n=50000, 4096x4096, L=4, nu=1.5, R=256, seed 0 (configs[4] CS)",
                                        batch=16)
            torch.cuda.empty_cache()
        for name, fn in (("predict_cfg2", workloads.cfg2), ("predict_cfg3", workloads.cfg3)):
            w = fn()
            c2 = build_predict_case(pk, w, world, rank, c_variants=2)
            m2s, _, _ = time_predict_device(pk, c2, max(5, args.steps // 2), 3, flush, with_k1=True)
            t2 = max_over_ranks(sum(m2s), world)
            k12 = weights_k1(c2, reps=10)
            pm2, pb2 = profile_passes(pk, c2, 5, flush)
            N2 = w.dims[0] * w.dims[1]
            extra[name] = {"value": round(N2 * len(m2s) * world / (t2 * 1e-3), 1), "unit": "points/s",
                           "ms_per_step": round(t2 / len(m2s), 5), "workload": w.name,
                           "embed": list(c2["setup"].embed_dims), "weights_k1_ms": k12["ms"],
                           "roofline": predict_roofline(c2, pm2, pb2, k12, t2 / len(m2s), peaks, peaks_kind, w.name)}
            del c2
            torch.cuda.empty_cache()
    # the CPU baselines run after every GPU measurement: concurrently, their numpy FFTs on all
    # host cores compete with the e2e leg's host work and DMA for host memory bandwidth (measured:
    # the cfg5 e2e step 3.5 -> 7.5 ms)
    if rank == 0 and not args.no_cpu:
        cpu = start_cpu_legs(args.quick)
    if cpu is not None:
        res = collect_cpu_legs(*cpu)
        cores = os.cpu_count() or 1
        if "predict" in res:
            t = res["predict"]
            line["cpu_baseline"] = {
                "value": round(N / statistics.median(t), 1), "unit": "points/s", "cores": 1, "kind": "port",
                "sample": f"{len(t)} step(s) of K1 + predict_rapid on the headline workload with the numpy oracle "
                          "port, one process, one core (pocketfft is single-threaded)", "cpu": cpu_model()}
        for name in ("cfg4", "cfg5"):
            r = res.get(f"cs_{name}")
            if r and f"cs_{name}" in extra:
                extra[f"cs_{name}"]["cpu_baseline"] = {
                    "value": round(r["draws"] / r["wall_s"], 3), "unit": "realizations/s", "cores": r["procs"],
                    "kind": "port",
                    "sample": f"{r['draws']} conditional draws of generate_ensemble (oracle port of simulate.py:146-192) "
                              f"over {r['procs']} single-threaded processes (OPENBLAS_NUM_THREADS=1), extrapolated as "
                              f"draws / wall time; setup {r['setup_s']:.1f} s untimed",
                    "cpu": cpu_model(), "nproc": cores}
    if extra:
        line["extra"] = extra
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
