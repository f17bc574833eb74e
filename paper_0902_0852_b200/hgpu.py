"""ctypes binding of libhgpu.so (include/hgpu.h), the B200 LDL^T engine.

Mirrors the reference's C++ entry points for the hot path
(/root/reference/proj/src/ldlt.hpp):

* ``ldlt_det_serial(m, x, capture)``  -> :meth:`HankelMatrixGPU.ldlt`
  (ldlt.hpp:30-31, ldlt.cpp:31-77)
* ``ldlt_det_parallel(m, x, workers)`` -> the same call after
  :meth:`HankelMatrixGPU.set_comm` (one process per GPU; ldlt.hpp:56-57)
* ``LdltCapture`` (ldlt.hpp:16-19)     -> :class:`LdltResult` pivots/ratios
* ``ZeroPivot(pivot_index, frac_bits)`` (errors.hpp:49-58) -> :class:`ZeroPivot`

There is no CPU fallback: importing this module on a machine without the
built library, or factoring without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HGPU_LIB") or os.path.join(_HERE, "libhgpu.so")

HGPU_CAPTURE = 1
HGPU_FOLD = 2
HGPU_PROFILE = 4

STATUS = {
    0: "ok", 1: "invalid argument", 2: "zero pivot", 3: "precision mismatch",
    4: "cuda", 5: "capacity", 6: "internal", 7: "communication",
    8: "precision exhausted", 9: "interval straddle",
}

# every symbol include/hgpu.h declares
EXPORTS = (
    "hgpu_matrix_new", "hgpu_matrix_free", "hgpu_nccl_unique_id",
    "hgpu_matrix_set_comm", "hgpu_ldlt_factor", "hgpu_factor_order",
    "hgpu_factor_frac_bits", "hgpu_factor_pivot", "hgpu_factor_ratio",
    "hgpu_factor_det", "hgpu_factor_device_ms", "hgpu_factor_update_stats",
    "hgpu_factor_launches", "hgpu_factor_free", "hgpu_matrix_plan", "hgpu_block_owner",
    "hgpu_last_zero_pivot", "hgpu_last_error", "hgpu_version",
    "hgpu_smallest_eigenvalue", "hgpu_string_free", "hgpu_inverse_iteration",
    "hgpu_interval_matrix_new", "hgpu_ldlt_interval", "hgpu_factor_pivot_hi",
    "hgpu_factor_det_hi", "hgpu_factor_det_sign", "hgpu_verify_eigenvalue",
    "hgpu_build_moments", "hgpu_buffer_free", "hgpu_matrix_set_capture_rows",
    "hgpu_matrix_new_group", "hgpu_matrix_world", "hgpu_verify_eigenvalue_ex",
    "hgpu_factor_net_ms", "hgpu_trim_pool", "hgpu_matrix_set_strip",
    "hgpu_matrix_new_from_dump", "hgpu_matrix_dump",
)


class HgpuError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"hgpu {STATUS.get(status, status)}: {message}")
        self.status = status


class ZeroPivot(HgpuError):
    """heig::ZeroPivot (errors.hpp:49-58): same pivot index and frac bits."""

    def __init__(self, pivot_index: int, frac_bits: int, message: str):
        super().__init__(2, message)
        self.pivot_index = pivot_index
        self.frac_bits = frac_bits


class PrecisionMismatch(HgpuError):
    pass


class PrecisionExhausted(HgpuError):
    """NoProgress / SignViolation / RootHitAtPrecision (errors.hpp:60-80):
    the working precision is exhausted; the driver escalates frac_bits."""


_lib = None


def load() -> ctypes.CDLL:
    """Loads libhgpu.so (built by ``__graft_entry__.build()``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, u32p, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_uint32), ctypes.c_long
    lib.hgpu_matrix_new.argtypes = [i64, i64, ctypes.POINTER(ctypes.c_int32), u32p, ctypes.c_int,
                                    ctypes.POINTER(vp)]
    lib.hgpu_matrix_free.argtypes = [vp]
    lib.hgpu_matrix_new_group.argtypes = [i64, i64, ctypes.POINTER(ctypes.c_int32), u32p,
                                          ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(vp)]
    lib.hgpu_matrix_new_from_dump.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(vp),
                                              ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long)]
    lib.hgpu_matrix_dump.argtypes = [vp, ctypes.c_char_p]
    lib.hgpu_matrix_world.argtypes = [vp]
    lib.hgpu_matrix_world.restype = ctypes.c_int
    lib.hgpu_nccl_unique_id.argtypes = [ctypes.c_char_p]
    lib.hgpu_matrix_set_comm.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
    lib.hgpu_matrix_set_capture_rows.argtypes = [vp, i64]
    lib.hgpu_ldlt_factor.argtypes = [vp, i32, u32p, i64, ctypes.c_uint, ctypes.POINTER(vp)]
    lib.hgpu_factor_order.argtypes = [vp]
    lib.hgpu_factor_order.restype = i64
    lib.hgpu_factor_frac_bits.argtypes = [vp]
    lib.hgpu_factor_frac_bits.restype = i64
    for name in ("hgpu_factor_pivot",):
        getattr(lib, name).argtypes = [vp, i64, ctypes.POINTER(i32), ctypes.POINTER(u32p)]
    lib.hgpu_factor_ratio.argtypes = [vp, i64, i64, ctypes.POINTER(i32), ctypes.POINTER(u32p)]
    lib.hgpu_factor_det.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(u32p)]
    lib.hgpu_factor_device_ms.argtypes = [vp]
    lib.hgpu_factor_device_ms.restype = ctypes.c_double
    lib.hgpu_factor_update_stats.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(ctypes.c_double)]
    lib.hgpu_trim_pool.argtypes = [ctypes.c_int]
    lib.hgpu_matrix_set_strip.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), u32p]
    lib.hgpu_factor_net_ms.argtypes = [vp]
    lib.hgpu_factor_net_ms.restype = ctypes.c_double
    lib.hgpu_factor_launches.argtypes = [vp]
    lib.hgpu_factor_launches.restype = ctypes.c_longlong
    lib.hgpu_factor_free.argtypes = [vp]
    lib.hgpu_matrix_plan.argtypes = [vp] + [ctypes.POINTER(ctypes.c_int)] * 4 + [ctypes.POINTER(ctypes.c_double)]
    lib.hgpu_block_owner.argtypes = [i64, ctypes.c_int]
    lib.hgpu_block_owner.restype = ctypes.c_int
    lib.hgpu_last_zero_pivot.restype = i64
    lib.hgpu_last_error.restype = ctypes.c_char_p
    lib.hgpu_version.restype = ctypes.c_char_p
    cpp = ctypes.POINTER(ctypes.c_char_p)
    lib.hgpu_smallest_eigenvalue.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                             ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(i64),
                                             ctypes.POINTER(ctypes.c_double)]
    lib.hgpu_string_free.argtypes = [ctypes.c_void_p]
    lib.hgpu_inverse_iteration.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), u32p, i32, u32p,
                                           ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                           ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(i64),
                                           ctypes.POINTER(ctypes.c_double)]
    lib.hgpu_interval_matrix_new.argtypes = [i64, i64, ctypes.POINTER(ctypes.c_int32), u32p,
                                             ctypes.POINTER(ctypes.c_int32), u32p, ctypes.c_int,
                                             ctypes.POINTER(vp)]
    lib.hgpu_ldlt_interval.argtypes = [vp, i32, u32p, i32, u32p, i64, ctypes.c_uint, ctypes.POINTER(vp)]
    lib.hgpu_factor_pivot_hi.argtypes = [vp, i64, ctypes.POINTER(i32), ctypes.POINTER(u32p)]
    lib.hgpu_factor_det_hi.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(u32p)]
    lib.hgpu_factor_det_sign.argtypes = [vp]
    lib.hgpu_factor_det_sign.restype = ctypes.c_int
    lib.hgpu_verify_eigenvalue.argtypes = [vp, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]
    lib.hgpu_verify_eigenvalue_ex.argtypes = [vp, ctypes.c_char_p, ctypes.c_int] + \
        [ctypes.POINTER(ctypes.c_int)] * 4 + [ctypes.POINTER(ctypes.c_void_p)] * 2
    pp32 = ctypes.POINTER(ctypes.POINTER(ctypes.c_int32))
    ppu32 = ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32))
    lib.hgpu_build_moments.argtypes = [i64, ctypes.c_ulong, ctypes.c_ulong, i64, ctypes.c_int,
                                       pp32, ppu32, pp32, ppu32]
    lib.hgpu_buffer_free.argtypes = [ctypes.c_void_p]
    _lib = lib
    return lib


def _check(status: int, frac_bits: int = 0) -> None:
    if status == 0:
        return
    lib = load()
    msg = lib.hgpu_last_error().decode()
    if status == 2:
        raise ZeroPivot(int(lib.hgpu_last_zero_pivot()), frac_bits, msg)
    if status == 3:
        raise PrecisionMismatch(status, msg)
    if status == 8:
        raise PrecisionExhausted(status, msg)
    raise HgpuError(status, msg)


# ----------------------------------------------------------- int <-> limbs --

def int_to_limbs(v: int) -> tuple[int, np.ndarray]:
    """Python int -> (signed size, little-endian uint32 limbs)."""
    mag = -v if v < 0 else v
    nbytes = (mag.bit_length() + 31) // 32 * 4
    limbs = np.frombuffer(mag.to_bytes(nbytes, "little"), dtype=np.uint32) if nbytes else \
        np.zeros(0, dtype=np.uint32)
    n = len(limbs)
    return (-n if v < 0 else n), limbs


def limbs_to_int(size: int, ptr) -> int:
    n = abs(size)
    if n == 0:
        return 0
    raw = ctypes.string_at(ptr, 4 * n)
    mag = int.from_bytes(raw, "little")
    return -mag if size < 0 else mag


def pack_ints(values: list[int]) -> tuple[np.ndarray, np.ndarray]:
    sizes, chunks = [], []
    for v in values:
        s, l = int_to_limbs(v)
        sizes.append(s)
        chunks.append(l)
    limbs = np.concatenate(chunks) if chunks else np.zeros(0, dtype=np.uint32)
    return np.asarray(sizes, dtype=np.int32), np.ascontiguousarray(limbs, dtype=np.uint32)


def _u32p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


# ------------------------------------------------------------------ API ----

@dataclass
class LdltResult:
    """LdltCapture (ldlt.hpp:16-19) plus the folded determinant."""
    n: int
    frac_bits: int
    pivots: list[int]
    ratios: dict = field(default_factory=dict)  # (p, r) -> R_p[r]
    det: int | None = None
    device_ms: float = 0.0
    update_launches: int = 0
    update_ms: float = 0.0
    update_products: float = 0.0
    launches: int = 0
    ratio_sha256: str | None = None
    net_ms: float = 0.0


def _hex(v: int) -> str:
    return ("-" + format(-v, "x")) if v < 0 else format(v, "x")


def ratio_digest(ratios) -> str:
    """sha256 over the ratios R_p[r] in (p, r) order, one lowercase hex
    line each (a leading '-' for negatives): the digest
    ``ldlt(..., ratio_digest=True)`` computes."""
    h = hashlib.sha256()
    for v in ratios:
        h.update(_hex(v).encode() + b"\n")
    return h.hexdigest()


class HankelMatrixGPU:
    """The anti-diagonal strip of M (HankelMatrix, hankel_matrix.hpp:17-42)
    resident on one B200, ready for repeated det(M - xI) evaluations."""

    def __init__(self, strip: list[int], frac_bits: int, device: int = 0,
                 devices: list[int] | None = None):
        """devices=[d0, d1, ...]: an in-process column-block-cyclic rank
        group, one rank per entry (ldlt_det_parallel with workers ->
        ranks; hgpu_matrix_new_group).  A device may repeat."""
        lib = load()
        if len(strip) % 2 == 0 or not strip:
            raise ValueError("strip must hold 2n-1 anti-diagonals")
        self.n = (len(strip) + 1) // 2
        self.frac_bits = frac_bits
        sizes, limbs = pack_ints(strip)
        h = ctypes.c_void_p()
        if devices and len(devices) > 1:
            devs = (ctypes.c_int * len(devices))(*devices)
            _check(lib.hgpu_matrix_new_group(self.n, frac_bits,
                                             sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                             _u32p(limbs), devs, len(devices), ctypes.byref(h)))
        else:
            _check(lib.hgpu_matrix_new(self.n, frac_bits,
                                       sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                       _u32p(limbs), devices[0] if devices else device,
                                       ctypes.byref(h)))
        self._h = h

    @classmethod
    def from_dump(cls, path: str, device: int = 0) -> "HankelMatrixGPU":
        """load_matrix_dump (hankel_matrix.cpp:65-87): the reference's
        "s=.. hex=.. fracbits=.." file straight onto the device."""
        lib = load()
        h = ctypes.c_void_p()
        n, k = ctypes.c_long(), ctypes.c_long()
        _check(lib.hgpu_matrix_new_from_dump(os.fsencode(path), device, ctypes.byref(h),
                                             ctypes.byref(n), ctypes.byref(k)))
        self = cls.__new__(cls)
        self.n, self.frac_bits, self._h = int(n.value), int(k.value), h
        return self

    def dump(self, path: str) -> None:
        """dump_matrix (hankel_matrix.cpp:52-57): the strip in the reference's
        interchange format."""
        _check(load().hgpu_matrix_dump(self._h, os.fsencode(path)))

    def set_strip(self, strip) -> None:
        """New moments of the same order and precision for the next ldlt()
        (hgpu_matrix_set_strip): the handle, plan and workspace are kept.
        `strip`: 2n-1 Python ints, or the (sizes, limbs) arrays of
        :func:`pack_ints` (host buffers, as a C caller passes them)."""
        if isinstance(strip, tuple):
            sizes, limbs = strip
        else:
            if len(strip) != 2 * self.n - 1:
                raise ValueError("strip must hold 2n-1 anti-diagonals")
            sizes, limbs = pack_ints(strip)
        if len(sizes) != 2 * self.n - 1:
            raise ValueError("strip must hold 2n-1 anti-diagonals")
        _check(load().hgpu_matrix_set_strip(self._h, sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                            _u32p(limbs)))

    @property
    def world(self) -> int:
        return int(load().hgpu_matrix_world(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            load().hgpu_matrix_free(self._h)
            self._h = None

    __del__ = close

    def set_comm(self, rank: int, world: int, nccl_id: bytes) -> None:
        _check(load().hgpu_matrix_set_comm(self._h, rank, world, nccl_id))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(load().hgpu_nccl_unique_id(buf))
        return buf.raw

    def plan(self) -> dict:
        lib = load()
        a, b, c, d = (ctypes.c_int() for _ in range(4))
        wb = ctypes.c_double()
        _check(lib.hgpu_matrix_plan(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                    ctypes.byref(d), ctypes.byref(wb)))
        return {"nprimes": a.value, "length": b.value, "digit_bits": c.value,
                "cap_limbs": d.value, "workspace_bytes": wb.value}

    def ldlt(self, x: int, capture: bool = False, fold: bool = False, profile: bool = False,
             x_frac_bits: int | None = None, capture_rows: int = 0,
             ratio_digest: bool = False) -> LdltResult:
        """det(M - xI) via square-root-free LDL^T (ldlt_det_serial).

        capture_rows > 0 keeps only the leading capture_rows block of the
        ratio columns; ratio_digest=True streams them into
        ``LdltResult.ratio_sha256`` (see :func:`ratio_digest`) instead of the
        ``ratios`` dict (a full-size capture is ~10^6 big integers)."""
        lib = load()
        if capture or ratio_digest:
            _check(lib.hgpu_matrix_set_capture_rows(self._h, capture_rows))
            capture = True
        xs, xl = int_to_limbs(x)
        flags = (HGPU_CAPTURE if capture else 0) | (HGPU_FOLD if fold else 0) | \
                (HGPU_PROFILE if profile else 0)
        f = ctypes.c_void_p()
        kx = self.frac_bits if x_frac_bits is None else x_frac_bits
        _check(lib.hgpu_ldlt_factor(self._h, xs, _u32p(xl), kx, flags, ctypes.byref(f)),
               self.frac_bits)
        try:
            n = self.n
            size = ctypes.c_int32()
            ptr = ctypes.POINTER(ctypes.c_uint32)()
            pivots = []
            for p in range(n):
                _check(lib.hgpu_factor_pivot(f, p, ctypes.byref(size), ctypes.byref(ptr)))
                pivots.append(limbs_to_int(size.value, ptr))
            res = LdltResult(n=n, frac_bits=self.frac_bits, pivots=pivots,
                             device_ms=lib.hgpu_factor_device_ms(f),
                             net_ms=lib.hgpu_factor_net_ms(f),
                             launches=int(lib.hgpu_factor_launches(f)))
            if capture:
                nc = min(n, capture_rows) if capture_rows > 0 else n
                h = hashlib.sha256() if ratio_digest else None
                for p in range(nc - 1):
                    for r in range(p + 1, nc):
                        _check(lib.hgpu_factor_ratio(f, p, r, ctypes.byref(size), ctypes.byref(ptr)))
                        v = limbs_to_int(size.value, ptr)
                        if h is None:
                            res.ratios[(p, r)] = v
                        else:
                            h.update(_hex(v).encode() + b"\n")
                if h is not None:
                    res.ratio_sha256 = h.hexdigest()
            if fold:
                _check(lib.hgpu_factor_det(f, ctypes.byref(size), ctypes.byref(ptr)))
                res.det = limbs_to_int(size.value, ptr)
            if profile:
                nl, ms, prod = ctypes.c_long(), ctypes.c_double(), ctypes.c_double()
                _check(lib.hgpu_factor_update_stats(f, ctypes.byref(nl), ctypes.byref(ms), ctypes.byref(prod)))
                res.update_launches, res.update_ms, res.update_products = nl.value, ms.value, prod.value
            return res
        finally:
            lib.hgpu_factor_free(f)


def build_moments(n: int, beta_num: int, beta_den: int, frac_bits: int, interval: bool = False):
    """build_matrix / build_interval_matrix (hankel_matrix.cpp:13-50) on the
    host: the strip (interval=False) or the (lo, hi) bound strips."""
    lib = load()
    ls, ll = ctypes.POINTER(ctypes.c_int32)(), ctypes.POINTER(ctypes.c_uint32)()
    hs, hl = ctypes.POINTER(ctypes.c_int32)(), ctypes.POINTER(ctypes.c_uint32)()
    _check(lib.hgpu_build_moments(n, beta_num, beta_den, frac_bits, int(interval), ctypes.byref(ls),
                                  ctypes.byref(ll), ctypes.byref(hs), ctypes.byref(hl)))

    def unpack(sz, lb):
        out, off = [], 0
        for s in range(2 * n - 1):
            k = sz[s]
            m = abs(k)
            v = 0
            for i in range(m - 1, -1, -1):
                v = (v << 32) | lb[off + i]
            off += m
            out.append(-v if k < 0 else v)
        return out

    try:
        lo, hi = unpack(ls, ll), unpack(hs, hl)
    finally:
        for p in (ls, ll, hs, hl):
            lib.hgpu_buffer_free(ctypes.cast(p, ctypes.c_void_p))
    return (lo, hi) if interval else lo


class IntervalMatrixGPU(HankelMatrixGPU):
    """HankelIntervalMatrix (hankel_matrix.hpp:42) on one B200: lower and
    upper bounds of every moment, for ldlt_det_interval (ldlt.cpp:79-152)
    and verify_eigenvalue (verify.cpp:8-42)."""

    def __init__(self, lo: list[int], hi: list[int], frac_bits: int, device: int = 0):
        lib = load()
        if len(lo) != len(hi) or len(lo) % 2 == 0 or not lo:
            raise ValueError("strips must hold 2n-1 anti-diagonals each")
        self.n = (len(lo) + 1) // 2
        self.frac_bits = frac_bits
        ls, ll = pack_ints(lo)
        hs, hl = pack_ints(hi)
        h = ctypes.c_void_p()
        _check(lib.hgpu_interval_matrix_new(self.n, frac_bits,
                                            ls.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _u32p(ll),
                                            hs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _u32p(hl),
                                            device, ctypes.byref(h)))
        self._h = h

    def ldlt_interval(self, x_lo: int, x_hi: int, fold: bool = False) -> dict:
        """pivot intervals [(lo, hi)], det sign and (fold) det interval."""
        lib = load()
        a, al = int_to_limbs(x_lo)
        b, bl = int_to_limbs(x_hi)
        f = ctypes.c_void_p()
        _check(lib.hgpu_ldlt_interval(self._h, a, _u32p(al), b, _u32p(bl), self.frac_bits,
                                      HGPU_FOLD if fold else 0, ctypes.byref(f)), self.frac_bits)
        try:
            size = ctypes.c_int32()
            ptr = ctypes.POINTER(ctypes.c_uint32)()
            piv = []
            for p in range(self.n):
                _check(lib.hgpu_factor_pivot(f, p, ctypes.byref(size), ctypes.byref(ptr)))
                lo = limbs_to_int(size.value, ptr)
                _check(lib.hgpu_factor_pivot_hi(f, p, ctypes.byref(size), ctypes.byref(ptr)))
                piv.append((lo, limbs_to_int(size.value, ptr)))
            out = {"pivots": piv, "det_sign": int(lib.hgpu_factor_det_sign(f)),
                   "device_ms": lib.hgpu_factor_device_ms(f)}
            if fold:
                _check(lib.hgpu_factor_det(f, ctypes.byref(size), ctypes.byref(ptr)))
                lo = limbs_to_int(size.value, ptr)
                _check(lib.hgpu_factor_det_hi(f, ctypes.byref(size), ctypes.byref(ptr)))
                out["det"] = (lo, limbs_to_int(size.value, ptr))
            return out
        finally:
            lib.hgpu_factor_free(f)


def verify_eigenvalue(m: IntervalMatrixGPU, x_decimal: str, digits: int = 15) -> dict:
    """verify_eigenvalue (verify.cpp:8-42) on the GPU interval LDL^T."""
    lib = load()
    st, ls, us, lz = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    a, b = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib.hgpu_verify_eigenvalue_ex(m._h, x_decimal.encode(), digits, ctypes.byref(st),
                                         ctypes.byref(ls), ctypes.byref(us), ctypes.byref(lz),
                                         ctypes.byref(a), ctypes.byref(b)), m.frac_bits)
    return {"status": ("verified", "refuted", "inconclusive")[st.value], "lower_sign": ls.value,
            "upper_sign": us.value, "lower_exact_zero": bool(lz.value),
            "probe_low": _take_string(a), "probe_high": _take_string(b)}


def _take_string(ptr: ctypes.c_void_p) -> str:
    if not ptr.value:
        return ""
    try:
        return ctypes.string_at(ptr.value).decode()
    finally:
        load().hgpu_string_free(ptr)


def smallest_eigenvalue(m: "HankelMatrixGPU", digits: int = 15) -> dict:
    """secant_smallest_eigenvalue (secant.cpp:27-117) on the GPU determinant:
    returns {"eigenvalue": str, "iterates": [(x, det)], "iterations": int,
    "det_seconds": float}."""
    lib = load()
    ev, tr = ctypes.c_void_p(), ctypes.c_void_p()
    it, secs = ctypes.c_long(), ctypes.c_double()
    _check(lib.hgpu_smallest_eigenvalue(m._h, digits, ctypes.byref(ev), ctypes.byref(tr),
                                        ctypes.byref(it), ctypes.byref(secs)), m.frac_bits)
    eig = _take_string(ev)
    lines = _take_string(tr).split("\n")
    iterates = [tuple(int(v, 16) for v in l.split()) for l in lines if l.strip()]
    return {"eigenvalue": eig, "iterates": iterates, "iterations": it.value,
            "det_seconds": secs.value}


def seeded_start_vector(n: int, frac_bits: int, seed: int = 0) -> list[int]:
    """north-star start vector: numpy default_rng(seed).uniform(-1, 1, n);
    doubles are dyadic, so they are exact at frac_bits >= 1100 or so and are
    otherwise truncated toward zero (mantissas at frac_bits)."""
    from fractions import Fraction
    vals = np.random.default_rng(seed).uniform(-1.0, 1.0, n)
    out = []
    for v in vals:
        f = Fraction(float(v)) * (1 << frac_bits)
        q = abs(f.numerator) // f.denominator
        out.append(q if f >= 0 else -q)
    return out


def inverse_iteration(m: "HankelMatrixGPU", u: list[int], sigma: int = 0, max_iter: int = 40,
                      digits: int = 15) -> dict:
    """Inverse iteration with Rayleigh-quotient shifts on the GPU factors."""
    lib = load()
    sizes, limbs = pack_ints(u)
    ss, sl = int_to_limbs(sigma)
    ev, tr = ctypes.c_void_p(), ctypes.c_void_p()
    it, secs = ctypes.c_long(), ctypes.c_double()
    _check(lib.hgpu_inverse_iteration(m._h, sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                      _u32p(limbs), ss, _u32p(sl), max_iter, digits,
                                      ctypes.byref(ev), ctypes.byref(tr), ctypes.byref(it),
                                      ctypes.byref(secs)), m.frac_bits)
    eig = _take_string(ev)
    rhos = [int(l, 16) for l in _take_string(tr).split("\n") if l.strip()]
    return {"eigenvalue": eig, "rho": rhos, "iterations": it.value, "seconds": secs.value}


def trim_pool(device: int = 0) -> None:
    """Hands the engine's idle pool blocks back to the driver (cold start)."""
    _check(load().hgpu_trim_pool(device))


def block_owner(block: int, world: int) -> int:
    return int(load().hgpu_block_owner(block, world))
