"""Python side of the oracle (TEST INFRASTRUCTURE — never the product path).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg import this module, and only as the checker or as the
timed CPU baseline.

Three independent checkers for the LDL^T hot path:

* ``RefLib`` — the reference sources compiled unchanged from
  ``/root/reference/proj/src`` into ``oracle/_ref/libheig_ref.so`` (see
  ``oracle/Makefile``), driven through ``oracle/ref_bridge.cpp``.
* ``OracleLib`` — our C restatement ``oracle/ldlt_oracle.c`` over GMP.
* ``ldlt_py`` — a pure-Python restatement of ``ldlt.cpp:31-77`` for small
  cases, plus the beta=1 closed form (D_k=(k!)^2,
  L[r][k]=C(r,k) r!/k!).

All numbers are exact Python ints (fixed-point mantissas).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libheig_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")


# --------------------------------------------------------------------------
# exact integer helpers with the reference's rounding (GMP tdiv semantics)
# --------------------------------------------------------------------------

def tdiv_q(a: int, b: int) -> int:
    """mpz_tdiv_q: quotient truncated toward zero (Python // floors)."""
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b > 0) else -q


def tdiv_q_2exp(a: int, k: int) -> int:
    """mpz_tdiv_q_2exp: a / 2^k truncated toward zero."""
    return a >> k if a >= 0 else -((-a) >> k)


def to_hex(v: int) -> str:
    return format(v, "x") if v >= 0 else "-" + format(-v, "x")


def from_hex(s: str) -> int:
    return int(s, 16)


# --------------------------------------------------------------------------
# strips (2n-1 anti-diagonal moments, mantissas at K fractional bits)
# --------------------------------------------------------------------------

def exact_strip(n: int, beta_num: int, beta_den: int, k: int) -> list[int]:
    """M_ij = (1/beta) Gamma((1+i+j)/beta) for beta = p/q with p | q, i.e.
    integer Gamma arguments: the reference's build_matrix is exact there
    (hankel_matrix.cpp:13-31 with gamma.cpp:193-197), so the factorials can be
    written down directly.  Used to cross-check the reference dump."""
    if beta_den % beta_num != 0:
        raise ValueError("exact_strip needs 1/beta integral")
    inv = beta_den // beta_num
    return [inv * math.factorial(inv * (1 + s) - 1) << k for s in range(2 * n - 1)]


def parse_dump(text: str) -> tuple[list[int], int]:
    """hankel_matrix.cpp:52-57 dump format -> (strip, frac_bits)."""
    strip, k = [], None
    for line in text.splitlines():
        if not line.strip():
            continue
        s_tok, h_tok, f_tok = line.split()
        assert s_tok == f"s={len(strip)}"
        strip.append(int(h_tok[4:], 16))
        k = int(f_tok[9:])
    return strip, k


def make_dump(strip: list[int], k: int) -> str:
    return "".join(f"s={s} hex={to_hex(v)} fracbits={k}\n" for s, v in enumerate(strip))


# --------------------------------------------------------------------------
# results
# --------------------------------------------------------------------------

class ZeroPivotError(Exception):
    def __init__(self, pivot_index: int, frac_bits: int):
        super().__init__(f"zero pivot at column {pivot_index} with {frac_bits} fractional bits")
        self.pivot_index = pivot_index
        self.frac_bits = frac_bits


@dataclass
class LdltResult:
    det: int
    pivots: list[int] = field(default_factory=list)
    ratios: dict = field(default_factory=dict)  # (p, r) -> R_p[r]


def parse_ldlt_text(text: str) -> LdltResult:
    if text.startswith("error ZeroPivot"):
        _, _, p, k = text.split()[:4]
        raise ZeroPivotError(int(p), int(k))
    if text.startswith("error"):
        raise RuntimeError(text.strip())
    res = LdltResult(det=0)
    for line in text.splitlines():
        parts = line.split()
        if not parts:
            continue
        if parts[0] == "det":
            res.det = int(parts[1], 16)
        elif parts[0] == "pivot":
            res.pivots.append(int(parts[2], 16))
        elif parts[0] == "ratio":
            res.ratios[(int(parts[1]), int(parts[2]))] = int(parts[3], 16)
    return res


# --------------------------------------------------------------------------
# pure-Python restatement (small cases)
# --------------------------------------------------------------------------

def fold_pivots(pivots: list[int], k: int) -> int:
    """ldlt.cpp:22-27 / fixed_point.cpp:40-53: truncate after every product."""
    det = 1 << k
    for p in pivots:
        det = tdiv_q_2exp(det * p, k)
    return det


def ldlt_py(strip: list[int], x: int, k: int, capture: bool = True) -> LdltResult:
    """ldlt_det_serial (ldlt.cpp:31-77) restated with Python ints."""
    n = (len(strip) + 1) // 2
    k2 = k // 2
    cols = [[strip[r + c] for r in range(c, n)] for c in range(n)]  # :38-44
    for c in range(n):
        cols[c][0] -= x
    pivots, ratios = [], {}
    for p in range(n):
        pivot = cols[p][0]
        if pivot == 0:  # :49-50
            raise ZeroPivotError(p, k)
        pivots.append(pivot)
        if p == n - 1:
            break
        values = [tdiv_q_2exp(cols[p][r - p], k2) for r in range(p, n)]  # :54-55
        if values[0] == 0:  # :56
            raise ZeroPivotError(p, k)
        rat = [tdiv_q(values[r - p] << k2, values[0]) for r in range(p + 1, n)]  # :15-20
        if capture:
            for r in range(p + 1, n):
                ratios[(p, r)] = rat[r - p - 1]
        for c in range(p + 1, n):  # :65-71
            mult = values[c - p]
            col = cols[c]
            for r in range(c, n):
                col[r - c] -= mult * rat[r - p - 1]
    return LdltResult(det=fold_pivots(pivots, k), pivots=pivots, ratios=ratios)


def fdiv_q(a: int, b: int) -> int:
    return a // b


def cdiv_q(a: int, b: int) -> int:
    return -((-a) // b)


@dataclass
class IntervalLdlt:
    det: tuple            # (lo, hi) at k bits
    pivots: list          # [(lo, hi)] per stage (workspace precision k)


def interval_mul(a: tuple, b: tuple, k: int) -> tuple:
    """FixedInterval::mul (fixed_interval.cpp): 4 corners, outward rounding."""
    c = [a[0] * b[0], a[0] * b[1], a[1] * b[0], a[1] * b[1]]
    return (min(c) >> k, -((-max(c)) >> k))


def ldlt_interval_py(lo: list[int], hi: list[int], k: int, x_lo: int, x_hi: int) -> IntervalLdlt:
    """ldlt_det_interval (ldlt.cpp:79-152) restated with Python ints."""
    n = (len(lo) + 1) // 2
    k2 = k // 2
    cols = [[[lo[r + c], hi[r + c]] for r in range(c, n)] for c in range(n)]
    for c in range(n):
        cols[c][0][0] -= x_hi
        cols[c][0][1] -= x_lo
    det = (1 << k, 1 << k)
    pivots = []
    for p in range(n):
        pv = tuple(cols[p][0])
        pivots.append(pv)
        det = interval_mul(det, pv, k)
        if p == n - 1:
            break
        vals = [None] * n
        for r in range(p, n):
            a, b = cols[p][r - p]
            vals[r] = (a >> k2, -((-b) >> k2))          # floor, ceil
        if vals[p][0] <= 0 <= vals[p][1]:
            raise ZeroPivotError(p, k)
        rat = [None] * n
        for r in range(p + 1, n):
            qs_f, qs_c = [], []
            for num in vals[r]:
                for den in vals[p]:
                    sc = num << k2
                    qs_f.append(fdiv_q(sc, den))
                    qs_c.append(cdiv_q(sc, den))
            rat[r] = (min(qs_f), max(qs_c))
        for c in range(p + 1, n):
            m = vals[c]
            col = cols[c]
            for r in range(c, n):
                cs = [m[0] * rat[r][0], m[0] * rat[r][1], m[1] * rat[r][0], m[1] * rat[r][1]]
                col[r - c][0] -= max(cs)
                col[r - c][1] -= min(cs)
    return IntervalLdlt(det=det, pivots=pivots)


def closed_form_beta1(n: int, k: int) -> LdltResult:
    """Known answer for beta=1, x=0: D_p=(p!)^2 exactly, and the
    ratios are integers so every truncation is exact:
    R_p[r] = C(r,p) * r!/p! * 2^(K/2)."""
    k2 = k // 2
    f = [math.factorial(i) for i in range(n)]
    pivots = [(f[p] * f[p]) << k for p in range(n)]
    ratios = {(p, r): (math.comb(r, p) * (f[r] // f[p])) << k2
              for p in range(n - 1) for r in range(p + 1, n)}
    return LdltResult(det=fold_pivots(pivots, k), pivots=pivots, ratios=ratios)


def column_owners(n: int, workers: int) -> list[int]:
    """assignment.hpp:15-23 reflected round-robin."""
    out = []
    for col in range(n):
        r = col % (2 * workers)
        out.append(r if r < workers else 2 * workers - 1 - r)
    return out


# --------------------------------------------------------------------------
# compiled checkers
# --------------------------------------------------------------------------

class _TextLib:
    def __init__(self, path: str, free_name: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built; run `make -C oracle`")
        self.lib = ctypes.CDLL(path)
        self._free = getattr(self.lib, free_name)
        self._free.argtypes = [ctypes.c_void_p]

    def _call(self, name, argtypes, *args) -> str:
        fn = getattr(self.lib, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_void_p
        ptr = fn(*args)
        try:
            return ctypes.string_at(ptr).decode()
        finally:
            self._free(ptr)


class OracleLib(_TextLib):
    """oracle/ldlt_oracle.c (our C restatement over GMP)."""

    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path, "oracle_free")

    def ldlt(self, strip: list[int], x: int, k: int, capture: bool = True) -> LdltResult:
        n = (len(strip) + 1) // 2
        text = self._call("oracle_ldlt",
                          [ctypes.c_long, ctypes.c_long, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int],
                          n, k, " ".join(map(to_hex, strip)).encode(), to_hex(x).encode(), int(capture))
        return parse_ldlt_text(text)

    def fold(self, pivots: list[int], k: int) -> int:
        text = self._call("oracle_fold", [ctypes.c_long, ctypes.c_long, ctypes.c_char_p],
                          len(pivots), k, " ".join(map(to_hex, pivots)).encode())
        return parse_ldlt_text(text).det


class RefLib(_TextLib):
    """The reference's own code (oracle/_ref/libheig_ref.so)."""

    def __init__(self, path: str = REF_SO):
        super().__init__(path, "oref_free")

    def build_strip(self, n: int, beta_num: int, beta_den: int, k: int) -> list[int]:
        text = self._call("oref_build_strip",
                          [ctypes.c_long, ctypes.c_ulong, ctypes.c_ulong, ctypes.c_long],
                          n, beta_num, beta_den, k)
        if text.startswith("error"):
            raise RuntimeError(text)
        return parse_dump(text)[0]

    def ldlt_serial(self, strip: list[int], x: int, k: int, capture: bool = True) -> LdltResult:
        text = self._call("oref_ldlt_serial", [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int],
                          make_dump(strip, k).encode(), to_hex(x).encode(), int(capture))
        return parse_ldlt_text(text)

    def ldlt_parallel(self, strip: list[int], x: int, k: int, workers: int) -> tuple[int, float]:
        text = self._call("oref_ldlt_parallel", [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_long],
                          make_dump(strip, k).encode(), to_hex(x).encode(), workers)
        res = parse_ldlt_text(text)
        secs = float([l.split()[1] for l in text.splitlines() if l.startswith("seconds")][0])
        return res.det, secs

    def secant(self, strip: list[int], k: int) -> dict:
        text = self._call("oref_secant", [ctypes.c_char_p], make_dump(strip, k).encode())
        if text.startswith("error"):
            raise RuntimeError(text)
        out = {"iterates": []}
        for line in text.splitlines():
            parts = line.split()
            if parts[0] == "iterate":
                out["iterates"].append((int(parts[1], 16), int(parts[2], 16)))
            elif parts[0] == "eigenvalue":
                out["eigenvalue"] = parts[1]
            elif parts[0] == "iterations":
                out["iterations"] = int(parts[1])
            elif parts[0] == "exact_root_hit":
                out["exact_root_hit"] = bool(int(parts[1]))
        return out

    def det_sign_decimal(self, strip: list[int], k: int, decimal: str) -> int:
        text = self._call("oref_det_sign_decimal", [ctypes.c_char_p, ctypes.c_char_p],
                          make_dump(strip, k).encode(), decimal.encode())
        if text.startswith("error"):
            raise RuntimeError(text)
        return int(text)

    def det_sign_parallel_decimal(self, strip: list[int], k: int, decimal: str, workers: int) -> dict:
        """Sign and bit length of det(M - xI) through ldlt_det_parallel."""
        text = self._call("oref_det_sign_parallel_decimal",
                          [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_long],
                          make_dump(strip, k).encode(), decimal.encode(), workers)
        if text.startswith("error"):
            raise RuntimeError(text)
        out = {}
        for line in text.splitlines():
            key, val = line.split()
            out[key] = float(val) if key == "seconds" else int(val)
        return out

    def interval_sign_decimal(self, n: int, beta_num: int, beta_den: int, kv: int, decimal: str) -> int:
        text = self._call("oref_interval_sign_decimal",
                          [ctypes.c_long, ctypes.c_ulong, ctypes.c_ulong, ctypes.c_long, ctypes.c_char_p],
                          n, beta_num, beta_den, kv, decimal.encode())
        if text.startswith("error"):
            raise RuntimeError(text)
        return int(text)

    def build_interval_strip(self, n: int, beta_num: int, beta_den: int, k: int):
        """build_interval_matrix (hankel_matrix.cpp) -> (lo strip, hi strip)."""
        text = self._call("oref_build_interval_strip",
                          [ctypes.c_long, ctypes.c_ulong, ctypes.c_ulong, ctypes.c_long],
                          n, beta_num, beta_den, k)
        if text.startswith("error"):
            raise RuntimeError(text)
        lo, hi = [], []
        for line in text.splitlines():
            _, a, b = line.split()
            lo.append(int(a, 16))
            hi.append(int(b, 16))
        return lo, hi

    def ldlt_interval(self, lo: list[int], hi: list[int], k: int, x_lo: int, x_hi: int):
        """ldlt_det_interval (ldlt.cpp:79-152) -> (det_lo, det_hi)."""
        strip = "".join(f"{to_hex(a)} {to_hex(b)}\n" for a, b in zip(lo, hi))
        text = self._call("oref_ldlt_interval",
                          [ctypes.c_char_p, ctypes.c_long, ctypes.c_char_p, ctypes.c_char_p],
                          strip.encode(), k, to_hex(x_lo).encode(), to_hex(x_hi).encode())
        if text.startswith("error"):
            parse_ldlt_text(text)  # raises ZeroPivotError / RuntimeError
        _, a, b = text.split()
        return int(a, 16), int(b, 16)

    def decimal_to_interval(self, decimal: str, k: int) -> tuple[int, int]:
        text = self._call("oref_decimal_to_interval", [ctypes.c_char_p, ctypes.c_long],
                          decimal.encode(), k)
        if text.startswith("error"):
            raise RuntimeError(text)
        a, b = text.split()
        return int(a, 16), int(b, 16)

    def verify(self, n: int, beta_num: int, beta_den: int, kv: int, x_decimal: str) -> dict:
        """verify_eigenvalue (verify.cpp:8-42) on build_interval_matrix(n, beta, kv)."""
        text = self._call("oref_verify",
                          [ctypes.c_long, ctypes.c_ulong, ctypes.c_ulong, ctypes.c_long, ctypes.c_char_p],
                          n, beta_num, beta_den, kv, x_decimal.encode())
        if text.startswith("error"):
            raise RuntimeError(text)
        st, lo, hi, a, b, lz = text.split()
        return {"status": ("verified", "refuted", "inconclusive")[int(st)],
                "lower_sign": int(lo), "upper_sign": int(hi), "lower_exact_zero": bool(int(lz)),
                "probe_low": a, "probe_high": b}

    def truncate_sig_digits(self, x: int, frac_bits: int, digits: int) -> str:
        return self._call("oref_truncate_sig_digits", [ctypes.c_char_p, ctypes.c_long, ctypes.c_int],
                          to_hex(x).encode(), frac_bits, digits)

    def bump_last_digit(self, s: str) -> str:
        return self._call("oref_bump_last_digit", [ctypes.c_char_p], s.encode())

    def column_owners(self, n: int, workers: int) -> list[int]:
        return [int(t) for t in self._call("oref_column_owners", [ctypes.c_long, ctypes.c_long],
                                           n, workers).split()]

    def heig_run(self, n: int, beta: str, k_bits: int = 0, workers: int = 1, verify: bool = False) -> dict:
        """Whole run through the reference's own C ABI (hankel_eig.h:28-81)."""
        L = self.lib
        L.heig_config_new.restype = ctypes.c_void_p
        L.heig_config_set_n.argtypes = [ctypes.c_void_p, ctypes.c_long]
        L.heig_config_set_beta.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.heig_config_set_precision_bits.argtypes = [ctypes.c_void_p, ctypes.c_long]
        L.heig_config_set_workers.argtypes = [ctypes.c_void_p, ctypes.c_long]
        L.heig_config_set_verify.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.heig_run.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        L.heig_result_to_json.argtypes = [ctypes.c_void_p]
        L.heig_result_to_json.restype = ctypes.c_void_p
        L.heig_string_free.argtypes = [ctypes.c_void_p]
        L.heig_result_free.argtypes = [ctypes.c_void_p]
        L.heig_config_free.argtypes = [ctypes.c_void_p]
        L.heig_last_error.restype = ctypes.c_char_p
        cfg = L.heig_config_new()
        try:
            L.heig_config_set_n(cfg, n)
            L.heig_config_set_beta(cfg, beta.encode())
            L.heig_config_set_precision_bits(cfg, k_bits)
            L.heig_config_set_workers(cfg, workers)
            L.heig_config_set_verify(cfg, int(verify))
            res = ctypes.c_void_p()
            st = L.heig_run(cfg, ctypes.byref(res))
            if st != 0:
                raise RuntimeError(f"heig_run status {st}: {L.heig_last_error().decode()}")
            js = L.heig_result_to_json(res)
            import json
            out = json.loads(ctypes.string_at(js).decode())
            L.heig_string_free(js)
            L.heig_result_free(res)
            return out
        finally:
            L.heig_config_free(cfg)


# --------------------------------------------------------------------------
# inverse iteration: no reference code exists;
# this restatement DEFINES the algorithm the GPU path implements
# (paper_0902_0852_b200/csrc/host/rqi.cpp, csrc/solve_kernels.cu) and is the
# bit-exact checker for it.
# --------------------------------------------------------------------------

def solve_py(f: LdltResult, u: list[int], k: int) -> list[int]:
    """(M - sI) y = u with L[r][p] = R_p[r] 2^-k2 and D_p = piv_p 2^-K, one
    truncation toward zero per entry (forward, diagonal, back)."""
    n, k2 = len(u), k // 2
    z, acc = [0] * n, [0] * n
    for p in range(n):
        z[p] = u[p] - tdiv_q_2exp(acc[p], k2)
        for r in range(p + 1, n):
            acc[r] += f.ratios[(p, r)] * z[p]
    w = [tdiv_q(z[p] << k, f.pivots[p]) for p in range(n)]
    y, acc = [0] * n, [0] * n
    for r in range(n - 1, -1, -1):
        y[r] = w[r] - tdiv_q_2exp(acc[r], k2)
        for q in range(r):
            acc[q] += f.ratios[(q, r)] * y[r]
    return y


RQI_SWITCH_BITS = 32   # phase 1 -> 2 when the relative change is < 2^-32
RQI_MAX_PLAIN = 64     # ... or after this many phase-1 steps
RQI_STALL = 2          # stop after this many changes not below the smallest so far


def rqi_final_bits(k: int) -> int:
    """phase 2 -> 3 when the relative change is < 2^-rqi_final_bits(K)"""
    return max(64, k // 16)


def inverse_iteration_py(strip: list[int], k: int, u: list[int], sigma: int = 0,
                         max_iter: int = 40, factor=None) -> list[int]:
    """Shifted inverse iteration with Rayleigh-quotient refactorisation
    (SURVEY §7 hard part (iv), §0 D7); returns every rho (mantissas at k bits).

    Phase 1 keeps the factors of M - sigma I and iterates y = (M - sigma I)^-1 u
    until the Rayleigh quotient's relative change is below 2^-RQI_SWITCH_BITS
    (or RQI_MAX_PLAIN steps), which pins the iteration to the eigenvalue next to
    sigma (lambda_1 for sigma <= 0 on a positive definite M).  Phase 2
    (Rayleigh-quotient iteration) refactors at sigma = rho every step until the
    relative change is below 2^-rqi_final_bits(K).  Phase 3 keeps those last
    factors: with sigma that close to lambda_1 every solve gains ~2 x
    rqi_final_bits bits, for the price of a solve instead of a factorisation.
    Stop when the relative change is below 2^-(K/2), when rho repeats, or when
    RQI_STALL changes have failed to go below the smallest change seen so far
    (the arithmetic noise floor).  factor(strip, x, k) defaults to ldlt_py."""
    factor = factor or (lambda s, x, kk: ldlt_py(s, x, kk, capture=True))
    n, k2 = len(u), k // 2
    final_bits = rqi_final_bits(k)
    rhos, rho_prev, d_min = [], None, None
    stall, plain, phase = 0, 0, 1
    f = None
    for _ in range(max_iter):
        if f is None:
            try:
                f = factor(strip, sigma, k)
            except ZeroPivotError as e:
                if e.pivot_index == n - 1:  # sigma is an eigenvalue at K bits
                    rhos.append(sigma)
                    break
                raise
        y = solve_py(f, u, k)
        num = sum(a * b for a, b in zip(y, u))
        den = sum(a * a for a in y)
        rho = sigma + tdiv_q(num << k, den)
        rhos.append(rho)
        if rho_prev is not None:
            d = abs(rho - rho_prev)
            if d == 0 or (d << k2) <= abs(rho):
                break
            if d_min is not None and d >= d_min:
                stall += 1
                if stall >= RQI_STALL:
                    break
            else:
                d_min = d
            if phase == 1 and ((d << RQI_SWITCH_BITS) <= abs(rho) or plain >= RQI_MAX_PLAIN):
                phase = 2
            elif phase == 2 and (d << final_bits) <= abs(rho):
                phase = 3
        rho_prev = rho
        plain += phase == 1
        mb = max(abs(v).bit_length() for v in y)
        sh = mb - k
        u = [tdiv_q_2exp(v, sh) if sh > 0 else v << -sh for v in y]
        if phase == 2:
            sigma, f = rho, None
    return rhos
