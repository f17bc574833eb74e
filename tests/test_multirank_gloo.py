"""CPU, world_size 2 and 3 over gloo: the multi-GPU schedule of
paper_0902_0852_b200/csrc/engine.cpp (Matrix::run) with exact oracle
arithmetic in place of the kernels.

Each rank owns the column blocks hgpu_block_owner assigns it (the library's
own ownership function, assignment.hpp:15-23 over blocks); the owner of a
panel factors it left-looking, broadcasts (V_p, R_p, pivots) exactly like
panel_broadcast does over NCCL, and every rank applies the rank-kb trailing
update to its own columns.  The result must be bit-identical to the serial
reference for every world size (tests/test_parallel.cpp:42-55)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import random_pd_hankel
import pyoracle as po


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def schedule_rank(rank, world, strip, x, k, kb):
    from paper_0902_0852_b200 import hgpu
    n = (len(strip) + 1) // 2
    k2 = k // 2
    nblocks = (n + kb - 1) // kb
    owned = [b for b in range(nblocks) if hgpu.block_owner(b, world) == rank]
    cols = [c for b in owned for c in range(b * kb, min(n, (b + 1) * kb))]
    W = {c: [strip[r + c] - (x if r == c else 0) for r in range(c, n)] for c in cols}
    pivots = [None] * n
    zero = None
    for b in range(nblocks):
        p0, p1 = b * kb, min(n, (b + 1) * kb)
        owner = hgpu.block_owner(b, world)
        payload = [None]
        if owner == rank:
            V, R, piv, zp = {}, {}, {}, None
            for p in range(p0, p1):
                col = W[p]
                for s in range(p0, p):  # left-looking inside the panel
                    for r in range(p, n):
                        col[r - p] -= V[s][p] * R[s][r]
                if col[0] == 0:
                    zp = p
                    break
                piv[p] = col[0]
                if p == n - 1:
                    break
                V[p] = {r: po.tdiv_q_2exp(col[r - p], k2) for r in range(p, n)}
                if V[p][p] == 0:
                    zp = p
                    break
                R[p] = {r: po.tdiv_q(V[p][r] << k2, V[p][p]) for r in range(p + 1, n)}
            payload = [(V, R, piv, zp)]
        dist.broadcast_object_list(payload, src=owner)
        V, R, piv, zp = payload[0]
        for p, v in piv.items():
            pivots[p] = v
        if zp is not None:
            zero = zp
            break
        for c in cols:  # trailing rank-kb update of owned columns
            if c < p1:
                continue
            colc = W[c]
            for s in range(p0, p1):
                if s not in R:
                    continue
                vc = V[s][c]
                for r in range(c, n):
                    colc[r - c] -= vc * R[s][r]
    return pivots, zero


def _worker(rank, world, port, strip, x, k, kb, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = schedule_rank(rank, world, strip, x, k, kb)
    finally:
        dist.destroy_process_group()


def run_world(world, strip, x, k, kb):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), strip, x, k, kb, out), nprocs=world, join=True)
    return [out[r] for r in range(world)]


@pytest.mark.parametrize("world", [2, 3])
def test_column_block_cyclic_bit_identical(world):
    n, k, kb = 21, 128, 4
    strip = random_pd_hankel(73, n, k)
    x = 1 << 100
    want = po.ldlt_py(strip, x, k, capture=False).pivots
    results = run_world(world, strip, x, k, kb)
    for pivots, zero in results:
        assert zero is None
        assert pivots == want


def test_zero_pivot_propagates_to_every_rank():
    # all-ones 3x3 (tests/test_parallel.cpp:90-97): every rank learns index 1
    strip = [1 << 64] * 5
    results = run_world(2, strip, 0, 64, 1)
    assert [z for _, z in results] == [1, 1]
