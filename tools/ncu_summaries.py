"""Write the profiles/ summaries from gpurun_out/ captures:
    python tools/ncu_summaries.py <round-tag>
  launches.csv  -> profiles/<tag>_launches.txt (+ .csv copy)
  k1_c3.ncu-rep -> profiles/<tag>_k1_c3_ncu_summary.txt and profiles/k1_traffic.json
  k1sym_c3.ncu-rep -> profiles/<tag>_k1sym_c3_ncu_summary.txt"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")

rows = list(csv.reader(open(os.path.join(G, "launches.csv"))))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = defaultdict(lambda: [0, 0.0])
for d in data:
    k = d["Kernel Name"].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
out = [f"# {tag} launch list: ncu --metrics gpu__time_duration.sum --clock-control none",
       "# command: python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 (configs[3], oqr_normal; warm-up launches included)",
       "# per-launch times are cold-cache and serialised: compare SHARES, not absolutes",
       f"# {'launches':>8} {'total_ms':>10} {'mean_ms':>9} {'share':>7}  kernel"]
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(f"  {c:8d} {v / 1e6:10.3f} {v / 1e6 / c:9.4f} {100 * v / tot:6.2f}%  {k}")
open(os.path.join(P, f"{tag}_launches.txt"), "w").write("\n".join(out) + "\n")
shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"{tag}_launches.csv"))
print("\n".join(out))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_active.avg",
        "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_short_scoreboard"]
MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summary(rep, name, title):
    r = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                       text=True).stdout.splitlines()))
    d = {a: (c, b) for a, b, c in zip(r[0], r[1], r[2])}
    lines = [title]
    for k in KEYS:
        if k in d:
            lines.append(f"{k:85s} {d[k][0]} {d[k][1]}")
    open(os.path.join(P, name), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return d


d = summary(os.path.join(G, "k1_c3.ncu-rep"), f"{tag}_k1_c3_ncu_summary.txt",
            f"# {tag} K1 gram_fused_kernel<25, dense> (ncu --set full --clock-control none), m=40000 n=200; "
            "command: python tools/prof_k1.py 40000 200 2 (-k regex:gram_fused -s 1 -c 1)")


def dram_bytes(d):
    return sum(float(d[k][0]) * MULT[d[k][1]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))


tp = os.path.join(P, "k1_traffic.json")
prev = json.load(open(tp)) if os.path.exists(tp) else {}
traffic = {"m": 40000, "n": 200,
           "dense": {"kernel": "gram_fused_kernel<25, dense>", "dram_bytes_per_launch": dram_bytes(d),
                     "algorithmic_bytes_per_launch": 8 * 40000 ** 2,
                     "source": f"profiles/{tag}_k1_c3_ncu_summary.txt (ncu --set full)"}}
if os.path.exists(os.path.join(G, "k1sym_c3.ncu-rep")):
    ds = summary(os.path.join(G, "k1sym_c3.ncu-rep"), f"{tag}_k1sym_c3_ncu_summary.txt",
                 f"# {tag} K1 gram_fused_kernel<25, sym> (block-lower triangle), m=40000 n=200; "
                 "command: python tools/time_k1.py 40000 200 1 sym (-k regex:gram_fused -s 1 -c 1)")
    P64 = 40000 // 64
    traffic["sym"] = {"kernel": "gram_fused_kernel<25, sym> (block-lower triangle of A)",
                      "dram_bytes_per_launch": dram_bytes(ds),
                      "algorithmic_bytes_per_launch": 8 * 64 * 64 * P64 * (P64 + 1) // 2,
                      "source": f"profiles/{tag}_k1sym_c3_ncu_summary.txt (ncu --set full)"}
elif "sym" in prev:  # keep the last symmetric-schedule capture
    traffic["sym"] = prev["sym"]
json.dump(traffic, open(tp, "w"), indent=1)
