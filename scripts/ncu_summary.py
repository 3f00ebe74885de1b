"""Summarise one kernel of an `ncu --set full` report (.ncu-rep) into the key metrics this repo
judges kernels by: duration, instructions, issue and pipe utilisation, shared-memory wavefronts
and bank conflicts, DRAM/L2 traffic, occupancy limits and the top warp-stall reasons.
Usage: python scripts/ncu_summary.py REPORT.ncu-rep "header line" [kernel-substring] > profiles/....txt
(with several kernels in the report, the first whose name contains kernel-substring)"""
import csv, io, re, subprocess, sys

rep, header = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
want = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
v = next(r for r in rows[2:] if want in r[h.index("Kernel Name")])
KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_src_tf32_dst_fp32.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum",
]
if header:
    print(header)
for k in KEYS:
    if k in h:
        i = h.index(k)
        print(f"{k:70s} {v[i]} {units[i] if k != 'Kernel Name' else ''}".rstrip())
stalls = []
for i, n in enumerate(h):
    m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", n)
    if m and not n.endswith("not_issued"):
        try:
            stalls.append((float(v[i].replace(",", "")), m.group(1)))
        except ValueError:
            pass
tot = sum(s for s, _ in stalls) or 1.0
print("warp-stall samples (share):", ", ".join(f"{n} {100 * s / tot:.1f}%" for s, n in sorted(stalls, reverse=True)[:8]))
