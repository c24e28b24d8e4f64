"""H2D / D2H timing of the e2e-sized copies over time (PCIe link state), with nvidia-smi link gen."""
import subprocess
import time

import torch

h = torch.empty(2940000 // 8, dtype=torch.float64).pin_memory()
d = torch.empty_like(h, device="cuda")
o = torch.empty(980000 // 8, dtype=torch.float64).pin_memory()
do = torch.empty_like(o, device="cuda")


def link():
    return subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,clocks.sm",
                           "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()


print("idle link:", link())
for phase in range(3):
    ts = []
    for k in range(60):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(h, non_blocking=True)
        o.copy_(do, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(round((time.perf_counter() - t0) * 1e6))
    print(f"phase {phase}: {ts[:10]} ... {ts[-10:]}  link {link()}")
    time.sleep(0.5)
