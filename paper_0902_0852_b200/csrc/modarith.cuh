// Word-size modular arithmetic for the residue-number (NTT) representation of
// the LDL^T workspace.  Primes are < 2^28 so that (a) Harvey-lazy butterflies
// stay below 2^30, and (b) a whole panel of up to 256 exact 56-bit products
// sums into one 64-bit accumulator before a single Montgomery reduction.
#pragma once
#include <cstdint>

namespace hgpu {

constexpr int kMaxPrimes = 4;
constexpr int kMaxLogL = 18;  // every prime is 1 mod 2^18

// q_j = a_j * 2^e_j + 1, all in (2^27, 2^28), with a primitive root g_j.
constexpr uint32_t kPrimes[kMaxPrimes] = {263454721u, 261881857u, 260571137u,
                                          257949697u};
constexpr uint32_t kPrimRoots[kMaxPrimes] = {11u, 7u, 3u, 5u};

struct PrimeConsts {
  uint32_t q;      // modulus
  uint32_t qneg;   // -q^{-1} mod 2^32 (Montgomery)
  uint32_t r32;    // 2^32 mod q
  uint32_t r32s;   // Shoup companion of r32
  uint32_t r64;    // 2^64 mod q (Montgomery form of r32)
  uint32_t one_s;  // Shoup companion of 1 (x mod q = mul_shoup(x, 1, one_s))
};

__host__ __device__ __forceinline__ uint32_t shoup_companion(uint32_t w,
                                                             uint32_t q) {
  return (uint32_t)(((uint64_t)w << 32) / q);
}

// a*w mod q in [0, 2q) for any a < 2^32, w < q, wp = shoup_companion(w, q).
__device__ __forceinline__ uint32_t mul_shoup(uint32_t a, uint32_t w,
                                              uint32_t wp, uint32_t q) {
  uint32_t hi = __umulhi(a, wp);
  return a * w - hi * q;
}

__device__ __forceinline__ uint32_t reduce_2q(uint32_t x, uint32_t q) {
  return x >= q ? x - q : x;
}

// Montgomery REDC of t < 2^61: returns t * 2^-32 mod q, in [0, q + 2^29).
__device__ __forceinline__ uint32_t redc(uint64_t t, uint32_t q,
                                         uint32_t qneg) {
  uint32_t m = (uint32_t)t * qneg;
  return (uint32_t)((t + (uint64_t)m * q) >> 32);
}

// Full reduction of any 64-bit sum of products (each < q^2 < 2^56, at most
// 256 of them) to (sum * 2^-32) mod q in [0, q).
__device__ __forceinline__ uint32_t reduce_sum64(uint64_t t,
                                                 const PrimeConsts& c) {
  uint64_t t1 = (t >> 32) * (uint64_t)c.r32 + (uint32_t)t;  // < 2^60.01
  uint32_t r = redc(t1, c.q, c.qneg);                        // < 2q + 2
  r = r >= c.q ? r - c.q : r;
  r = r >= c.q ? r - c.q : r;
  return r >= c.q ? r - c.q : r;
}

}  // namespace hgpu
