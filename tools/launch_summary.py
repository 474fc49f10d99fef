#!/usr/bin/env python3
"""Per-kernel summary of the LAST matvec in an ncu launch list (--metrics gpu__time_duration.sum
--csv): serialised, cold-cache durations; each matvec starts at permute_kernel and ends at
combine_kernel.   launch_summary.py <launches.csv>"""
import collections
import csv
import io
import sys

text = open(sys.argv[1]).read()
text = text[text.index('"ID"'):]            # skip ncu's preamble lines
rows = [r for r in csv.DictReader(io.StringIO(text)) if r.get("Metric Name") == "gpu__time_duration.sum"]
starts = [i for i, r in enumerate(rows) if "permute_kernel" in r["Kernel Name"]]
last = rows[starts[-1]:] if starts else rows
end = next((i for i, r in enumerate(last) if "combine_kernel" in r["Kernel Name"]), len(last) - 1)
mv = last[:end + 1]
tot = sum(float(r["Metric Value"]) for r in mv) / 1e6
agg = collections.OrderedDict()
for r in mv:
    k = r["Kernel Name"].split("(")[0].replace("void ", "")[:70]
    agg.setdefault(k, [0.0, 0])
    agg[k][0] += float(r["Metric Value"]) / 1e6
    agg[k][1] += 1
print(f"{sys.argv[1]}: {len(starts)} matvecs; last matvec {len(mv)} launches, serialised sum {tot:.3f} ms")
for k, (t, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"  {t:9.3f} ms {100 * t / tot:5.1f}%  x{n:<3d} {k}")
