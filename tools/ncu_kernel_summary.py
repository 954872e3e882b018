"""One-kernel ncu summary for profiles/: key raw metrics + stall breakdown + hottest SASS lines.
    python tools/ncu_kernel_summary.py <rep.ncu-rep> <out.txt> "<title / command line>"
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
lines = [f"# {title}", "# ncu --set full --clock-control none --import-source on (one launch, cold-cache, serialised)"]
for k in want:
    if k in h:
        i = h.index(k)
        unit = rows[1][i] if len(rows) > 2 else ""
        lines.append(f"{k:70s} {v[i]} {unit}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
starts = [i for i, r in enumerate(srows) if r and r[0] == "Kernel Name"]
if starts:
    hh = srows[starts[0] + 1]
    idx = {k: i for i, k in enumerate(hh)}
    data = [r for r in srows[starts[0] + 2:(starts[1] if len(starts) > 1 else len(srows))] if len(r) == len(hh)]
    S = lambda r: int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    tot = sum(S(r) for r in data)
    agg = Counter()
    for r in data:
        for k in hh:
            if k.startswith("stall_") and "Not Issued" not in k and r[idx[k]]:
                agg[k] += int(r[idx[k]])
    lines.append(f"stall samples {tot}: " + ", ".join(f"{k[6:]} {100 * c / max(tot, 1):.0f}%" for k, c in agg.most_common(8)))
    lines.append("hottest SASS lines (samples, executions, instruction):")
    for r in sorted(data, key=lambda r: -S(r))[:12]:
        lines.append(f"  {S(r):6d} {r[idx['Instructions Executed']]:>10}  {r[idx['Source']][:80]}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
