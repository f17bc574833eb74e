"""Aggregate ncu --page source --print-source cuda,sass CSV by CUDA source
line: stall samples and executed instructions."""
import collections
import csv
import sys

cur_file = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
tot = 0
for row in csv.reader(open(sys.argv[1])):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        hdr = None
        continue
    if row[0] == "Function Name":
        continue
    if row[0] == "Line No":
        hdr = row
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(row) <= si or not row[0]:
        continue
    try:
        s = int(row[si] or 0)
        n = int(row[ii] or 0)
    except ValueError:
        continue
    key = (cur_file, row[0])
    agg[key][0] += s
    agg[key][1] += n
    if not agg[key][2]:
        agg[key][2] = row[1][:90]
    tot += s
top = sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for (f, ln), (s, n, src) in top:
    print(f"{100.0 * s / max(tot, 1):5.1f}% {n:10d} {f}:{ln:5s} {src}")
