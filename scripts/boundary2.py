"""Pivot-chain time and panel-boundary gaps per panel from an HGPU_TIMELINE
file with the fused chain (k_pivot = kind 2)."""
import collections
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
kb = 32
n = 1 + max(by)
tc = tb = 0
for b in range((n + kb - 1) // kb - 1):
    p0, pl = b * kb, min(n - 2, b * kb + kb - 1)
    st = by[p0][2][0][0]
    en = by[pl][2][0][1]
    if 5 in by[pl]:
        en = max(en, max(x[1] for x in by[pl][5]))
    far = max((x[1] for x in by[pl][12]), default=en)
    nxt = by[(b + 1) * kb][2][0][0] if (b + 1) * kb < n - 1 else en
    tc += en - st
    tb += nxt - en
    print(f"{b:2d} chain {en - st:6.2f} ms  far lag {far - en:6.2f}  boundary {nxt - en:6.2f} ms")
print(f"chain total {tc:.1f} ms, boundary total {tb:.1f} ms")
