"""Summarise an ncu --set full report (one kernel launch) into a text file for profiles/."""
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
algo_bytes = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {k: (u, v) for k, u, v in zip(hdr, units, vals)}
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
        "gpc__cycles_elapsed.avg.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
lines = [f"ncu --set full summary of {rep}", ""]
for k in keys:
    if k in d:
        lines.append(f"{k:60s} {d[k][1]:>20s} {d[k][0]}")
stalls = []
for k, (u, v) in d.items():
    if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
        try:
            stalls.append((float(v), k))
        except ValueError:
            pass
lines.append("")
lines.append("warp stall reasons (warps per issue, top 8):")
for v, k in sorted(stalls, reverse=True)[:8]:
    lines.append(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v:.3f}")
if algo_bytes:
    rd = float(d["dram__bytes_read.sum"][1]); wr = float(d["dram__bytes_write.sum"][1])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tb = rd * scale[d["dram__bytes_read.sum"][0]] + wr * scale[d["dram__bytes_write.sum"][0]]
    lines.append("")
    lines.append(f"traffic (dram read+write) = {tb:.4e} B; algorithmic = {algo_bytes:.4e} B; ratio = {tb / algo_bytes:.4f}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
