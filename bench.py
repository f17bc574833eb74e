#!/usr/bin/env python
"""Benchmark: the LDL^T (square-root-free Cholesky) factorisation of the
Hankel moment matrix at BASELINE config 3 (N=1000, beta=1, P=24576 bits).

One step = one full factorisation of M - xI on the device (every stage:
extraction, pivot reciprocal, ratios, transforms, rank-kb trailing update)
with x = x1 = -2^-16 * min(1, M00), the secant's first probe
(secant.cpp:7-16), so ratios are truncated (not the exact x=0 closed form).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line on rank 0 (see DESIGN.md §6 for every key).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = {"workload": "LDL^T factorisation of M - x1*I, N=1000, beta=1, P=24576",
          "n": 1000, "beta": "1", "precision_bits": 24576, "shift": "x1=-2^-16",
          "l2": "workspace (plan.workspace_bytes, GBs) >> 126 MB L2: inputs larger than L2"}
METRIC = "Cholesky MP-MAC/s (N=1000, beta=1, P=24576)"
UNIT = "MP-MAC/s"


def mp_macs(n: int) -> float:
    """(N^3 - N)/6 MP multiply-adds per factorisation (ldlt.cpp:65-71)."""
    return (n ** 3 - n) / 6.0


def schoolbook_limb_products(n: int, k: int) -> float:
    """Sum over the trailing updates of ceil(bits(V)/32)*ceil(bits(R)/32) for
    beta=1, x=0 (closed form): the schoolbook-equivalent work,
    independent of the algorithm actually used."""
    import numpy as np
    k2 = k // 2
    lf = np.zeros(n + 1)
    for i in range(2, n + 1):
        lf[i] = lf[i - 1] + math.log2(i)
    total = 0.0
    for p in range(n - 1):
        c = np.arange(p + 1, n)
        vbits = 2 * lf[c] - lf[c - p] + k2 + 1       # (c!)^2/(c-p)! 2^k2
        rbits = 2 * lf[c] - 2 * lf[p] - lf[c - p] + k2 + 1  # C(r,p) r!/p! 2^k2
        vl = np.ceil(vbits / 32.0)
        rl = np.ceil(rbits / 32.0)
        # sum_{c<=r} vl[c]*rl[r] = sum_c vl[c] * suffix(rl)[c]
        suffix = np.cumsum(rl[::-1])[::-1]
        total += float(np.dot(vl, suffix))
    return total


# --------------------------------------------------------------- clocks ----

class ClockSampler:
    """Samples nvidia-smi SM clocks + throttle reasons while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def loop():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                    if out.returncode == 0 and out.stdout.strip():
                        self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        return self

    def stop(self) -> dict:
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- inputs ---

def config_strip(n: int, k: int) -> list[int]:
    """beta=1 moments M_ij = Gamma(1+i+j) = (i+j)!, exact at K bits: the
    reference's build_matrix is exact for integer Gamma arguments
    (hankel_matrix.cpp:13-31, gamma.cpp:193-197)."""
    strip, f = [], 1
    for s in range(2 * n - 1):
        if s > 0:
            f *= s
        strip.append(f << k)
    return strip


def x1_shift(strip: list[int], k: int) -> int:
    """initial_points (secant.cpp:7-16): x1 = -trunc(min(1, M00) / 2^16)."""
    one = 1 << k
    smaller = strip[0] if strip[0] < one else one
    mant = smaller >> 16
    return -(mant if mant else 1)


# ------------------------------------------------------------- GPU arm -----

def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_gpu(args) -> None:
    """N GPUs: by default one process drives all N as an in-process rank
    group (hgpu_matrix_new_group: panels published with CUDA events, pulled
    over NVLink peer memory) while the other torchrun ranks wait for it;
    --transport nccl runs one rank per process with the NCCL panel
    broadcast instead."""
    import torch
    world_env, rank, local = _dist_env()
    if world_env > 1 and args.transport == "group":
        import torch.distributed as dist
        dist.init_process_group("gloo")  # rendezvous only; no device traffic
        try:
            if rank == 0:
                _run_gpu_body(args, hgpu_devices=list(range(world_env)), nccl=False, rank=0, local=0)
        finally:
            dist.barrier()
            dist.destroy_process_group()
        return
    if world_env <= 1 and os.environ.get("BENCH_RANK_DEVICES"):
        # the rank-group path on explicit devices (a device may repeat: the
        # multi-rank schedule on a one-GPU lease)
        devs = [int(d) for d in os.environ["BENCH_RANK_DEVICES"].split(",")]
        _run_gpu_body(args, hgpu_devices=devs, nccl=False, rank=0, local=devs[0])
        return
    if world_env > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _run_gpu_body(args, hgpu_devices=[local], nccl=world_env > 1, rank=rank, local=local)


def _run_gpu_body(args, hgpu_devices, nccl, rank, local) -> None:
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1")) if nccl else 1
    ndev = world if nccl else len(hgpu_devices)
    torch.cuda.set_device(local)
    from paper_0902_0852_b200 import hgpu
    n, k = CONFIG["n"], CONFIG["precision_bits"]
    strip = config_strip(n, k)
    x = x1_shift(strip, k)

    def new_matrix():
        mm = hgpu.HankelMatrixGPU(strip, k, device=local,
                                  devices=hgpu_devices if len(hgpu_devices) > 1 else None)
        if nccl:
            import torch.distributed as dist
            obj = [hgpu.HankelMatrixGPU.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            mm.set_comm(rank, world, obj[0])
        return mm

    m = new_matrix()
    plan = m.plan()

    def barrier():
        if nccl:
            import torch.distributed as dist
            dist.barrier()
        for d in sorted(set(hgpu_devices)):
            torch.cuda.synchronize(d)

    for _ in range(args.warmup):
        m.ldlt(x)
    barrier()
    clocks = ClockSampler(local).start()
    dev_ms, launches, upd_ms, upd_prod, upd_n = [], 0, 0.0, 0.0, 0
    for _ in range(args.steps):
        r = m.ldlt(x, profile=True)
        dev_ms.append(r.device_ms)
        launches += r.launches
        upd_ms += r.update_ms
        upd_prod += r.update_products
        upd_n += r.update_launches
    barrier()
    clk = clocks.stop()
    total_ms = sum(dev_ms)
    if nccl:
        import torch.distributed as dist
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = mp_macs(n) / (ms_per_step * 1e-3)

    # parity of the benched workload: one more factorisation of the same
    # matrix at the same shift, its leading block (pivots and every ratio
    # R_p[r], p < r < n') against the reference's ldlt_det_serial on that
    # block (tests/golden/leading_blocks.json, generated by oracle/_ref)
    parity = leading_block_parity(m, x, hgpu)

    # end to end through the public API with host buffers, every step: the
    # strip (the step's input) from host memory into the matrix handle
    # (hgpu_matrix_set_strip: copied and transformed on the device by the
    # factorisation), the factorisation, and every pivot back to the host as
    # Python integers (the step's result)
    e2e_ms, h2d, d2h = [], 0, 0
    sizes, limbs = hgpu.pack_ints(strip)
    h2d = sizes.nbytes + limbs.nbytes + 8
    for _ in range(max(1, min(args.steps, 3))):
        barrier()
        t0 = time.perf_counter()
        m.set_strip((sizes, limbs))
        rr = m.ldlt(x)
        barrier()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        d2h = sum((abs(v).bit_length() + 31) // 32 * 4 + 4 for v in rr.pivots)
    del m
    e2e_step = statistics.median(e2e_ms)

    # time to lambda_min (north-star): inverse iteration with Rayleigh-quotient
    # refactorisation from the seed-0 start vector, x = 0, to the 2^-(P/2)
    # rule, through the public API (single rank: the solve is not sharded)
    lam = None
    if not nccl and not args.no_lambda:
        barrier()
        t0 = time.perf_counter()
        mm = new_matrix()
        rq = hgpu.inverse_iteration(mm, hgpu.seeded_start_vector(n, k), 0, 40, digits=40)
        barrier()
        lam = {"seconds": time.perf_counter() - t0, "iterations": rq["iterations"],
               "lambda_min": rq["eigenvalue"], "digits": 40,
               "method": "shifted inverse iteration + RQI on the GPU LDL^T (hgpu_inverse_iteration)",
               "includes": "strip upload, every factorisation and triangular solve",
               "pool": "warm (the engine's device memory pool kept from the timed steps)"}
        # the same again on the same handle: solve buffers, the solve plan and
        # the L store are in place (the steady state of a sweep over matrices
        # of one shape); the strip is handed over again
        barrier()
        t0 = time.perf_counter()
        mm.set_strip((sizes, limbs))
        r2 = hgpu.inverse_iteration(mm, hgpu.seeded_start_vector(n, k), 0, 40, digits=40)
        barrier()
        lam["seconds_steady_state"] = time.perf_counter() - t0
        lam["steady_state_same_digits"] = r2["eigenvalue"] == rq["eigenvalue"]
        del mm
        # the same with the pool handed back to the driver first: the cold
        # start a fresh process pays (workspace and slot-set allocations)
        for d in sorted(set(hgpu_devices)):
            hgpu.trim_pool(d)
        barrier()
        t0 = time.perf_counter()
        mm = new_matrix()
        rc = hgpu.inverse_iteration(mm, hgpu.seeded_start_vector(n, k), 0, 40, digits=40)
        barrier()
        lam["seconds_cold_pool"] = time.perf_counter() - t0
        lam["cold_pool_same_digits"] = rc["eigenvalue"] == rq["eigenvalue"]
        del mm
        # certification of those digits (verify_eigenvalue on the GPU
        # interval LDL^T at Kv = 2P, row f1): two interval factorisations
        barrier()
        t0 = time.perf_counter()
        kv = 2 * k
        sv = config_strip(n, kv)
        im = hgpu.IntervalMatrixGPU(sv, sv, kv, device=local)
        vr = hgpu.verify_eigenvalue(im, rq["eigenvalue"], 40)
        barrier()
        lam["certification"] = {
            "seconds": time.perf_counter() - t0, "status": vr["status"], "digits": 40,
            "kv_bits": kv, "probe_low": vr["probe_low"], "probe_high": vr["probe_high"],
            "method": "verify_eigenvalue (verify.cpp:8-42) on the GPU interval LDL^T "
                      "(hgpu_verify_eigenvalue), strip upload included"}
        del im

    # BASELINE configs 4 and 5 (after everything config 3 measures, so the
    # device pool they grow does not shape the config-3 numbers)
    secondary = None
    if ndev == 1 and not args.no_secondary:
        secondary = secondary_configs(hgpu, args)

    # roofline of the dominant kernel (trailing update): modular products per
    # launch / average launch time, against the measured IMAD.WIDE rate
    probe = probe_imad()
    upd_avg_ms = upd_ms / max(upd_n, 1)
    prod_per_launch = upd_prod / max(upd_n, 1)
    achieved = prod_per_launch / (upd_avg_ms * 1e-3) / 1e12 if upd_n else None
    peak = probe.get("wide_ops_per_s", 0) / 1e12 or None

    out = {
        "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": ndev, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32 (exact mod-q residues, 32-bit limbs)",
        "data": "synthetic: exact factorial moments (the reference's beta=1 strip)",
        "config": dict(CONFIG, parallelism=f"column-block-cyclic x{ndev}",
                       transport=("nccl broadcast, one process per GPU" if nccl else
                                  "in-process rank group, NVLink peer reads" if ndev > 1
                                  else "single rank"),
                       plan=plan),
        "limb_products_per_s": schoolbook_limb_products(n, k) / (ms_per_step * 1e-3),
        "e2e": {"value": mp_macs(n) / (e2e_step * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_step},
        "gpu_launches": launches,
        "roofline": {"bound": "imad", "kernel": "k_update (trailing rank-kb update)",
                     "achieved": achieved, "peak": peak, "unit": "Tprod/s (IMAD.WIDE)",
                     "frac": (achieved / peak) if achieved and peak else None,
                     "traffic": None, "peak_source": "measured IMAD.WIDE probe (csrc/probe.cu)",
                     "update_share_of_step": (upd_ms / args.steps) / ms_per_step},
        "imad_probe": probe,
        "clocks": clk,
    }
    out["parity"] = parity
    if secondary:
        out["secondary_configs"] = secondary
    if lam:
        out["time_to_lambda_min"] = lam
    traffic = _profiled_traffic()
    if traffic:
        out["roofline"]["traffic"] = traffic["dram_bytes_per_launch"]
        out["roofline"]["traffic_source"] = traffic["source"]
        # the same kernel profiled alone: IMAD.WIDE (FMA-heavy) pipe busy %,
        # time-weighted over every launch of a factorisation, and on a full
        # band run; its HBM rate alone (GB/s)
        out["roofline"]["ncu_imad_pipe_frac_alone"] = (traffic.get("pipe_pct") or 0) / 100 or None
        if traffic.get("pipe_pct_full_band_run"):
            out["roofline"]["ncu_imad_pipe_frac_full_band_run"] = traffic["pipe_pct_full_band_run"] / 100
        if traffic.get("hbm_gbs_alone"):
            out["roofline"]["ncu_hbm_gbs_alone"] = traffic["hbm_gbs_alone"]
        if upd_n and traffic.get("dram_bytes_per_launch"):
            # profiled bytes per launch (the same su1 + su2 launches the engine
            # times) over the launch's average time in the step
            out["roofline"]["hbm_gbs_in_step"] = traffic["dram_bytes_per_launch"] / (upd_avg_ms * 1e-3) / 1e9
    if rank == 0 and ndev == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if nccl:
        import torch.distributed as dist
        dist.destroy_process_group()


SECONDARY = [
    # (config, N, beta_num, beta_den, P)
    (4, 1500, 1, 2, 65536),
    (5, 2000, 3, 2, 32768),
]


def secondary_configs(hgpu, args) -> list:
    """BASELINE configs 4 and 5 at full size on one GPU: one warm-up and
    one timed factorisation of M - x1 I each (device time, CUDA events), with
    the trailing update's share (HGPU_PROFILE) beside the panel side.  The
    config-5 moments come from the repo's threaded build_matrix (bit-identical
    to the reference's, tests/test_moments.py); its time is reported apart."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    out = []
    for cfg, n, bn, bd, k in SECONDARY:
        t0 = time.perf_counter()
        if (bn, bd) == (1, 2):
            strip = [2 * math.factorial(2 * (1 + s) - 1) << k for s in range(2 * n - 1)]
        else:
            strip = hgpu.build_moments(n, bn, bd, k)
        t_strip = time.perf_counter() - t0
        x = x1_shift(strip, k)
        mm = hgpu.HankelMatrixGPU(strip, k)
        mm.ldlt(x)
        r = mm.ldlt(x, profile=True)
        plan = mm.plan()
        mm.close()
        del mm
        out.append({"config": cfg, "n": n, "beta": f"{bn}/{bd}", "precision_bits": k,
                    "shift": "x1 (secant.cpp:7-16)", "ms_per_factorisation": r.device_ms,
                    "mp_macs_per_s": mp_macs(n) / (r.device_ms * 1e-3),
                    "update_ms": r.update_ms, "update_share": r.update_ms / r.device_ms,
                    "gpu_launches": r.launches, "plan": plan,
                    "moments_seconds": round(t_strip, 2),
                    "moments": "exact factorials" if (bn, bd) == (1, 2)
                    else "hgpu_build_moments (host threads)"})
    return out


def leading_block_parity(m, x, hgpu) -> dict:
    """Leading n' x n' block of this workload's factorisation against the
    reference's digests (made by tests/golden/make_leading_blocks.py)."""
    import hashlib
    path = os.path.join(ROOT, "tests", "golden", "leading_blocks.json")
    want = next((c for c in json.load(open(path))
                 if c["name"] == "config3" and c["shift"] == "x1"), None)
    if want is None:
        return {"checked": False, "why": "no config3/x1 fixture"}
    nb = want["n_prime"]
    r = m.ldlt(x, capture_rows=nb, ratio_digest=True)
    h = hashlib.sha256()
    for v in r.pivots[:nb]:
        h.update(hgpu._hex(v).encode() + b"\n")
    ok_p = h.hexdigest() == want["pivots_sha256"]
    ok_r = r.ratio_sha256 == want["ratios_sha256"]
    return {"checked": True, "bit_exact": ok_p and ok_r, "pivots": ok_p, "ratios": ok_r,
            "block": nb, "n_ratios": want["n_ratios"],
            "against": "reference ldlt_det_serial + LdltCapture on the leading block "
                       "(oracle/_ref, tests/golden/leading_blocks.json)"}


def _profiled_traffic():
    """DRAM bytes per k_update_tiled launch (average over every launch of one
    factorisation) and the kernel's IMAD.WIDE pipe utilisation alone, from the
    committed ncu summaries (profiles/*/k_update_all_launches.json, and the
    full band run of k_update_full.json), if present."""
    import glob
    out = {}
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "k_update_all_launches.json")))
    if files:
        with open(files[-1]) as f:
            d = json.load(f)
        out = {"dram_bytes_per_launch": d.get("dram_bytes_per_launch"),
               "pipe_pct": d.get("sm_pipe_fmaheavy_pct_time_weighted"),
               "hbm_gbs_alone": d.get("hbm_gbs_alone"),
               "source": os.path.relpath(files[-1], ROOT)}
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "k_update_full.json")))
    if files:
        with open(files[-1]) as f:
            d = json.load(f)
        out["pipe_pct_full_band_run"] = d.get("sm_pipe_fmaheavy_pct_of_peak_elapsed")
        if "dram_bytes_per_launch" not in out:
            out.update(dram_bytes_per_launch=d.get("dram_bytes_per_launch"),
                       pipe_pct=d.get("sm_pipe_fmaheavy_pct_of_peak_elapsed"),
                       source=os.path.relpath(files[-1], ROOT))
    return out or None


def probe_imad() -> dict:
    import ctypes
    path = os.path.join(ROOT, "paper_0902_0852_b200", "libhgpu_probe.so")
    if not os.path.exists(path):
        return {}
    lib = ctypes.CDLL(path)
    lib.hgpu_probe_imad.argtypes = [ctypes.c_int] + [ctypes.POINTER(ctypes.c_double)] * 3
    res = {}
    for kind, name in ((0, "imad"), (1, "wide")):
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        if lib.hgpu_probe_imad(kind, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)) == 0:
            res[f"{name}_ops_per_s"] = a.value
            res[f"{name}_sm_mhz"] = b.value
            res[f"{name}_per_clk_sm"] = c.value
    return res


# ------------------------------------------------------------ CPU legs -----

def cpu_sample(seconds_budget: float = 20.0):
    """Times the reference's own ldlt_det_parallel (oracle/_ref, all host
    threads) on the leading n' x n' block of the config-3 matrix at the same
    P and shift.  Returns (seconds, n', workers, limb-products of the sample)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    k = CONFIG["precision_bits"]
    workers = os.cpu_count() or 1
    ref = po.RefLib()
    nprime = 120
    while True:
        strip = config_strip(nprime, k)
        x = x1_shift(strip, k)
        _, secs = ref.ldlt_parallel(strip, x, k, workers)
        if secs * 2.2 ** 3 > seconds_budget or nprime >= 400:
            break
        nprime = int(nprime * 1.5)
    return secs, nprime, workers, schoolbook_limb_products(nprime, k)


def cpu_baseline(args) -> dict:
    secs, nprime, workers, lp = cpu_sample()
    full_lp = schoolbook_limb_products(CONFIG["n"], CONFIG["precision_bits"])
    est_full_s = secs * full_lp / lp
    return {"value": mp_macs(CONFIG["n"]) / est_full_s, "unit": UNIT, "cores": workers,
            "kind": "reference",
            "sample": f"ldlt_det_parallel (oracle/_ref, {workers} threads) on the leading "
                      f"{nprime}x{nprime} block at P=24576: {secs:.2f} s; scaled to N=1000 by "
                      f"schoolbook limb-products ({lp:.3e} -> {full_lp:.3e}): est {est_full_s:.0f} s "
                      f"per factorisation"}


def run_reference(args) -> None:
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    vals = []
    for _ in range(args.warmup):
        cpu_sample(seconds_budget=5.0)
    for _ in range(args.steps):
        secs, nprime, workers, lp = cpu_sample(seconds_budget=10.0)
        full_lp = schoolbook_limb_products(CONFIG["n"], CONFIG["precision_bits"])
        vals.append(mp_macs(CONFIG["n"]) / (secs * full_lp / lp))
    v = statistics.median(vals)
    sample = (f"ldlt_det_parallel (oracle/_ref, {workers} threads) on the leading {nprime}x{nprime} "
              f"block at P=24576, scaled to N=1000 by schoolbook limb-products")
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": mp_macs(CONFIG["n"]) / v * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "mpz (GMP 6.3.0)", "data": "synthetic: exact factorial moments",
           "config": dict(CONFIG, parallelism=f"{workers} host threads"), "impl": "reference",
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def _spawn_ranks(n: int) -> None:
    """--gpus N without a launcher: run this script under torch.distributed.run
    with N ranks on this node (one process per GPU, NCCL) and exit with its
    status; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="group", choices=["group", "nccl"],
                    help="N > 1: one process drives every GPU (group) or one NCCL rank per process")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the config 4 / 5 factorisation timings")
    ap.add_argument("--no-lambda", action="store_true",
                    help="skip the time-to-lambda_min measurement")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        _spawn_ranks(args.gpus)
    if world and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
