"""Key ncu metrics per kernel from a .ncu-rep (ncu --page raw --csv): time, DRAM bytes, pipe /
issue utilisation, occupancy, stall reasons.  Usage: python tools/ncu_summary.py REPORT [regex]"""
import csv
import io
import re
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__occupancy_limit_shared_mem", "occ_limit_smem"),
    ("launch__occupancy_limit_registers", "occ_limit_regs"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "smem_dyn"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("sm__cycles_elapsed.avg", "sm_cycles"),
    ("smsp__inst_executed.sum", "inst"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_barrier"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall_mio"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall_short_sb"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall_math"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "stall_membar"),
]

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
ix = {k: hdr.index(k) for k, _ in WANT if k in hdr}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if pat and not pat.search(name):
        continue
    print(name)
    for k, short in WANT:
        if k in ix:
            print(f"   {short:22s} {r[ix[k]]:>16s} {units[ix[k]]}")
    if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in ix and "sm__cycles_elapsed.avg" in ix:
        try:
            wf = float(r[ix["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]].replace(",", ""))
            cyc = float(r[ix["sm__cycles_elapsed.avg"]].replace(",", ""))
            print(f"   {'smem_busy_frac':22s} {wf / (148 * cyc):16.3f}")
        except ValueError:
            pass
