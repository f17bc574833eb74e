"""Per-stage analysis of an HGPU_TIMELINE capture (fused chain, default
schedule): what k_pivot(p) waited for and how long each path took.
Kinds: 2 k_pivot, 3 near col update, 4 near extract, 5 divide (near, or the
chain's own at the panel end), 16 pivot-entry early stages, 10-12 far rows."""
import collections
import statistics
import sys

blocks, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = []
        blocks.append(cur)
        continue
    k, p, a, b = line.strip().split(",")
    cur.append((int(k), int(p), float(a) * 1e3, float(b) * 1e3))  # us
recs = blocks[-1]
by = collections.defaultdict(lambda: collections.defaultdict(list))
for k, p, a, b in recs:
    by[p][k].append((a, b))
n = 1 + max(by)
last = collections.Counter()
rows = []
for p in range(2, n - 1):
    if 2 not in by[p] or 2 not in by[p - 1]:
        continue
    s, e = by[p][2][0]
    deps = {"k_pivot(p-1)": by[p - 1][2][0][1]}
    if 4 in by[p - 1]:
        deps["near extract(p-1)"] = max(x[1] for x in by[p - 1][4])
    if 5 in by[p - 2] if p - 2 in by else False:
        deps["near divide(p-2)"] = max(x[1] for x in by[p - 2][5])
    if 16 in by[p]:
        deps["entry pre(p)"] = by[p][16][0][1]
    d = max(deps, key=deps.get)
    last[d] += 1
    near = by[p - 1]
    ncol = sum(b - a for a, b in near.get(3, []))
    next_ = sum(b - a for a, b in near.get(4, []))
    ndiv = sum(b - a for a, b in near.get(5, []))
    rows.append((p, e - s, s - deps[d], d, ncol, next_, ndiv, s - by[p - 1][2][0][1]))
print("k_pivot released by:", dict(last))
for lo, hi in ((2, 200), (200, 500), (500, 800), (800, 1000)):
    sel = [r for r in rows if lo <= r[0] < hi]
    if not sel:
        continue
    med = lambda i: statistics.median(x[i] for x in sel)
    print(f"p in [{lo},{hi}): k_pivot {med(1):6.1f} us, launch gap after last dep {med(2):5.1f} us, "
          f"start after prev k_pivot end {med(7):6.1f} us; near path of p-1: col {med(4):5.1f} "
          f"extract {med(5):5.1f} divide {med(6):5.1f} us")
tot = sum(r[1] for r in rows)
print(f"k_pivot busy {tot/1e3:.1f} ms of the factorisation; stage period median "
      f"{statistics.median(by[p][2][0][0]-by[p-1][2][0][0] for p in range(2, n-1) if 2 in by[p] and 2 in by[p-1]):.1f} us")
