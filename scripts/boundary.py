"""Per-panel pivot-chain time and panel-boundary gap from an HGPU_TIMELINE
file (last factorisation in it)."""
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
    st = by[p0][0][0][0]
    en = max(x[1] for x in by[pl][5])
    far = by[pl][12][0][1] if 12 in by[pl] else en
    nxt = by[(b + 1) * kb][0][0][0] if (b + 1) * kb < n - 1 else en
    un = by[b][8][0] if 8 in by[b] else (0, 0)
    tc += en - st
    tb += nxt - en
    print(f"{b:2d} chain {en - st:6.2f} ms  far lag {far - en:6.2f}  next-band update {un[0] - en:6.2f}..{un[1] - en:6.2f}  boundary {nxt - en:6.2f} ms")
print(f"chain total {tc:.1f} ms, boundary total {tb:.1f} ms")
