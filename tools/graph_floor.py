"""Floor of an event-timed CUDA-graph replay after an L2 flush: graphs of k tiny kernels.

python tools/graph_floor.py  -> median event time (us) for k = 1, 2, 3, 4 trivial kernels."""
import statistics

import torch

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
x = torch.zeros(1, device="cuda")
s = torch.cuda.Stream()
for k in (1, 2, 3, 4):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for _ in range(3):
            for _ in range(k):
                x.add_(1)
        with torch.cuda.graph(g, stream=s):
            for _ in range(k):
                x.add_(1)
    torch.cuda.synchronize()
    for mode in ("flushed", "warm"):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
        for a, b in ev:
            if mode == "flushed":
                flush.zero_()
            a.record()
            g.replay()
            b.record()
        torch.cuda.synchronize()
        ms = [a.elapsed_time(b) * 1000 for a, b in ev]
        print(f"graph of {k} tiny kernels, {mode}: median {statistics.median(ms):.2f} us, min {min(ms):.2f}")
