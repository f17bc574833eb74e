"""Analyse an HGPU_TIMELINE file (last factorisation in it): per-kind busy
time and the per-stage critical chain."""
import collections
import sys

KIND = {0: "col(pivot)", 1: "extract(pivot)", 2: "recip", 3: "col(rest)", 4: "extract(rest)",
        5: "divide", 6: "col(all)", 7: "extract(all)", 8: "update(next)", 9: "update(rest)",
        10: "col(far)", 11: "extract(far)", 12: "divide(far)",
        13: "update(catch-up)", 14: "update(far sub-panel)", 15: "update(next band, lookahead)",
        16: "pivot entry (early stages)", 17: "next row (sn)"}
blocks, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = {"hdr": line.strip(), "recs": []}
        blocks.append(cur)
        continue
    k, p, a, b = line.strip().split(",")
    cur["recs"].append((int(k), int(p), float(a), float(b)))
blk = blocks[-1]
print(blk["hdr"])
recs = blk["recs"]
busy = collections.defaultdict(float)
cnt = collections.Counter()
for k, p, a, b in recs:
    busy[k] += b - a
    cnt[k] += 1
for k in sorted(busy):
    print(f"{KIND[k]:16s} n={cnt[k]:5d} total {busy[k]:8.2f} ms  avg {1e3 * busy[k] / cnt[k]:8.1f} us")
by = collections.defaultdict(dict)
for k, p, a, b in recs:
    if k <= 7:
        by[p][k] = (a, b)
ps = sorted(by)
seg = collections.defaultdict(list)
for i, p in enumerate(ps):
    d = by[p]
    if 5 in d and i > 0 and 5 in by[ps[i - 1]]:
        seg["stage (divide end to divide end)"].append(d[5][1] - by[ps[i - 1]][5][1])
    if 2 in d and 5 in d:
        seg["recip end -> divide start"].append(d[5][0] - d[2][1])
    if 4 in d and 5 in d:
        seg["extract(rest) end -> divide start"].append(d[5][0] - d[4][1])
    if 2 in d and 1 in d:
        seg["extract(pivot) end -> recip start"].append(d[2][0] - d[1][1])
    if 0 in d and 1 in d:
        seg["col(pivot) end -> extract(pivot) start"].append(d[1][0] - d[0][1])
    if 5 in d and i > 0 and 0 in d and 5 in by[ps[i - 1]]:
        seg["prev divide end -> col(pivot) start"].append(d[0][0] - by[ps[i - 1]][5][1])
for k, v in seg.items():
    v = sorted(v)
    print(f"{k:40s} mean {1e3 * sum(v) / len(v):8.1f} us  median {1e3 * v[len(v) // 2]:8.1f} us")
for k in (0, 1, 2, 3, 4, 5):
    d = sorted(1e3 * (b - a) for kk, p, a, b in recs if kk == k)
    if d:
        print(f"{KIND[k]:16s} median {d[len(d) // 2]:8.1f} us  p90 {d[int(len(d) * 0.9)]:8.1f} us")
