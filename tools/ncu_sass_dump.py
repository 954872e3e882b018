"""Per-SASS-line stall samples of one captured kernel, in program order (for reading a hot loop).
    python tools/ncu_sass_dump.py <rep.ncu-rep> <out.txt>
"""
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
hh = rows[starts[0] + 1]
idx = {k: i for i, k in enumerate(hh)}
data = [r for r in rows[starts[0] + 2:(starts[1] if len(starts) > 1 else len(rows))] if len(r) == len(hh)]
stalls = [k for k in hh if k.startswith("stall_") and "Not Issued" not in k]
with open(out, "w") as f:
    for r in data:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        top = sorted(((int(r[idx[k]] or 0), k[6:]) for k in stalls), reverse=True)[:2]
        tops = " ".join(f"{k}:{v}" for v, k in top if v)
        f.write(f"{s:6d} {r[idx['Instructions Executed']]:>9} {tops:34s} {r[idx['Source']][:90]}\n")
