"""A/B of flushed device-path predict times across environment switches.

python tools/ab.py cfg2,cfg1 RK_C_SMEM=0 RK_C_SMEM=1 ...
Each variant runs in its own process (the switches are read once per process); prints the
median / p10 / p90 per-step CUDA-event time of predict_rapid with L2 flushed before each step."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfgs):
    sys.path.insert(0, ROOT)
    import bench
    import paper_2605_29284_b200 as pk
    from paper_2605_29284_b200 import workloads
    flush = (lambda: None) if os.environ.get("AB_NOFLUSH") == "1" else bench.L2Flush()
    res = {}
    for name in cfgs:
        case = bench.build_predict_case(pk, workloads.CONFIGS[name](), c_variants=2)
        ms, _, _ = bench.time_predict_device(pk, case, 200, 10, flush)
        ms = sorted(m * 1000 for m in ms)
        res[name] = (statistics.median(ms), ms[len(ms) // 10], ms[9 * len(ms) // 10])
    print(json.dumps(res))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2].split(","))
        sys.exit(0)
    cfgs = sys.argv[1]
    for variant in sys.argv[2:] or ["-"]:
        env = dict(os.environ)
        if variant != "-":
            for kv in variant.split(";"):
                k, v = kv.split("=")
                env[k] = v
        out = subprocess.run([sys.executable, __file__, "--child", cfgs], env=env, capture_output=True, text=True)
        try:
            res = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            print(variant, "FAILED", out.stderr[-2000:])
            continue
        print(variant, " ".join(f"{k}: {v[0]:.2f} us (p10 {v[1]:.2f}, p90 {v[2]:.2f})" for k, v in res.items()),
              flush=True)
