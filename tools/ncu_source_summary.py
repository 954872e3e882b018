"""Summarise an ncu --page source --csv --print-source sass dump (first kernel in the file):
stall reasons overall and the top instructions by sampled stalls.
    ncu -i rep --page source --csv --print-source sass > x.csv; python tools/ncu_source_summary.py x.csv [ntop]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 15
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
a = starts[0]
b = starts[1] if len(starts) > 1 else len(rows)
print(rows[a][1][:100])
h = rows[a + 1]
idx = {k: i for i, k in enumerate(h)}
data = [r for r in rows[a + 2:b] if len(r) == len(h)]
S = lambda r: int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
print("total samples", sum(S(r) for r in data))
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = Counter()
for r in data:
    for k in reasons:
        if r[idx[k]]:
            agg[k] += int(r[idx[k]])
print(agg.most_common(8))
for i in sorted(range(len(data)), key=lambda i: -S(data[i]))[:ntop]:
    r = data[i]
    print(f"{i:5d} {S(r):7d} {r[idx['Instructions Executed']]:>10} {r[idx['Source']][:90]}")
