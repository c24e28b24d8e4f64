"""Turn one round's raw GPU evidence in gpurun_out/ into the committed profiles/ files.

python tools/summarize_profiles.py v5      (expects gpurun_out/bench_v5.json, bench_ref_v5.json,
                                            launches_bench_v5.csv, prof_cfg2_v5.ncu-rep,
                                            prof_cfg3_v5.ncu-rep)
writes profiles/round1_bench_<tag>.json, round1_bench_ref_<tag>.json,
round1_launches_bench_<tag>.csv + _summary.txt, round1_ncu_full_<tag>_summary.txt and
round1_traffic.json (the dram bytes bench.py reports as roofline.traffic)."""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")
NAMES = {"row_fwd": "pass1_gather_rowfft", "col_kernel": "pass2_column_filter", "row_inv": "pass3_rowifft_epilogue"}
FULL_METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
                "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
                "sm__warps_active.avg.pct_of_peak_sustained_active",
                "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
                "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu_raw(rep, metrics):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    return r[0], r[1], [dict(zip(r[0], row)) for row in r[2:]]


def main(tag):
    for src, dst in ((f"bench_{tag}.json", f"round1_bench_{tag}.json"),
                     (f"bench_ref_{tag}.json", f"round1_bench_ref_{tag}.json"),
                     (f"launches_bench_{tag}.csv", f"round1_launches_bench_{tag}.csv")):
        shutil.copy(os.path.join(RAW, src), os.path.join(OUT, dst))
    # launch list summary (cold-cache, serialized durations)
    rows = list(csv.reader(open(os.path.join(RAW, f"launches_bench_{tag}.csv"))))
    h, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            data.append(dict(zip(h, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v = v / 1000 if d["Metric Unit"] in ("ns", "nsecond") else (v * 1000 if d["Metric Unit"] in ("ms", "msecond") else v)
        k = re.sub(r"\(.*", "", d["Kernel Name"])[:60]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v for _, v in agg.values())
    lines = ["ncu --metrics gpu__time_duration.sum --clock-control none -c 600 (bench.py --steps 5 --warmup 3 "
             "--no-extra); cold-cache serialized durations (setup kernels run once, predict kernels x steps)"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:24]:
        lines.append(f"{v:10.1f} us {100 * v / tot:5.1f}% x{n:4d}  avg {v / n:8.2f} us  {k}")
    pk = {k: (n, v) for k, (n, v) in agg.items() if re.search(r"rk::(row_fwd_kernel<3|col_kernel<0|row_inv)", k)}
    ps = sum(v for _, v in pk.values())
    lines.append("predict kernels: " + ", ".join(f"{k}: {v / n:.2f} us avg ({100 * v / ps:.0f}%)"
                                                 for k, (n, v) in pk.items()))
    open(os.path.join(OUT, f"round1_launches_bench_{tag}_summary.txt"), "w").write("\n".join(lines) + "\n")
    # full captures: summary + traffic
    traffic = {"source": f"ncu --set full --clock-control none (tools/profile_predict.py <cfg> 3), {tag}: "
                         "dram__bytes_read.sum + dram__bytes_write.sum per launch", "kernels": {}}
    out = []
    for cfg in ("cfg2", "cfg3"):
        rep = os.path.join(RAW, f"prof_{cfg}_{tag}.ncu-rep")
        h, units, recs = ncu_raw(rep, FULL_METRICS)
        out.append(f"== {cfg}: ncu --set full --clock-control none --import-source on "
                   f"-k regex:row_fwd|col_kernel|row_inv (tools/profile_predict.py {cfg} 3)")
        for d in recs:
            name = next(v for kk, v in NAMES.items() if kk in d["Kernel Name"])
            out.append(f"  {d['Kernel Name'][:60]}  [{name}]")
            for k, u in zip(h, units):
                if "__" in k:
                    out.append(f"     {k:90s} {d[k]} {u}")
            rd = float(d["dram__bytes_read.sum"]) * SCALE[units[h.index("dram__bytes_read.sum")]]
            wr = float(d["dram__bytes_write.sum"]) * SCALE[units[h.index("dram__bytes_write.sum")]]
            # shared-memory data pipe: one 128-byte wavefront per SM cycle at most
            wf = float(d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"])
            cyc = float(d["sm__cycles_elapsed.avg"])
            traffic["kernels"].setdefault(cfg, {})[name] = {"dram_bytes": rd + wr, "read": rd, "write": wr,
                                                             "ncu_us": float(d["gpu__time_duration.sum"]),
                                                             "smem_wavefronts": wf,
                                                             "smem_busy_frac": round(wf / (148 * cyc), 4)}
    # optional captures: the weights kernel (K1) per config and the CS ensemble kernels
    extra_metrics = FULL_METRICS + ["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                                    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                                    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
    for label, fname in [("weights kernel (K1), cfg2", f"prof_weights_cfg2_{tag}.ncu-rep"),
                         ("weights kernel (K1), cfg3", f"prof_weights_cfg3_{tag}.ncu-rep"),
                         ("CS ensemble kernels, cfg4 (tools/cs_probe.py 64 32)", f"prof_cs_{tag}.ncu-rep")]:
        rep = os.path.join(RAW, fname)
        if not os.path.exists(rep):
            continue
        h, units, recs = ncu_raw(rep, extra_metrics)
        out.append(f"== {label}: ncu --set full --clock-control none --import-source on ({fname})")
        for d in recs:
            out.append(f"  {d['Kernel Name'][:70]}")
            for k, u in zip(h, units):
                if "__" in k:
                    out.append(f"     {k:90s} {d[k]} {u}")
    open(os.path.join(OUT, f"round1_ncu_full_{tag}_summary.txt"), "w").write("\n".join(out) + "\n")
    json.dump(traffic, open(os.path.join(OUT, "round1_traffic.json"), "w"), indent=1)
    print("\n".join(lines[:12]))
    print(json.dumps(traffic["kernels"], indent=1)[:800])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "v5")
