"""Which dependency releases each k_pivot (HGPU_TIMELINE, fused chain): the
previous k_pivot, the near extraction of the previous stage (kind 4), the
early-stage pivot-entry update (kind 16), or none (launch latency)."""
import collections
import statistics
import sys

blocks, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith('#'):
        cur = []
        blocks.append(cur)
        continue
    k, p, a, b = line.strip().split(',')
    cur.append((int(k), int(p), float(a), float(b)))
by = collections.defaultdict(lambda: collections.defaultdict(list))
for k, p, a, b in blocks[-1]:
    by[p][k].append((a, b))
n = 1 + max(by)
cnt = collections.Counter()
gaps = collections.defaultdict(list)
for p in range(2, n - 1):
    if 2 not in by[p] or 2 not in by[p - 1]:
        continue
    start = by[p][2][0][0]
    deps = {"prev k_pivot": by[p - 1][2][0][1]}
    if 4 in by[p - 1]:
        deps["near extract p-1"] = by[p - 1][4][0][1]
    if 16 in by[p]:
        deps["entry pre-update"] = by[p][16][0][1]
    if 5 in by[p - 1]:
        deps["chain divide p-1"] = max(x[1] for x in by[p - 1][5])
    last = max(deps, key=deps.get)
    cnt[last] += 1
    gaps[last].append(1e3 * (start - deps[last]))
    for d, t in deps.items():
        gaps["slack " + d].append(1e3 * (start - t))
print("releasing dependency counts:", dict(cnt))
for k, v in sorted(gaps.items()):
    print(f"{k:32s} median {statistics.median(v):8.1f} us  mean {statistics.mean(v):8.1f} us")
