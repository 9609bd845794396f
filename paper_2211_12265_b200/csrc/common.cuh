// common.cuh -- parameter sets, Z_q arithmetic and rounding for the sm_100a kernels.
//
// Reference semantics (not code): proj/include/dilithium/params.hpp:8-55,
// reduce.hpp:33-82, rounding.hpp:13-59.  Only canonical values ever reach a codec
// or a hash, so internal representations are chosen for the GPU: signed
// Montgomery products on the IMAD pipe, no to_mont passes (the inverse NTT's final
// constants absorb the stray R^-1), lazy reductions sized to stay inside int32.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tables.inc"

namespace dlb {

constexpr int32_t kQ = 8380417;
constexpr uint32_t kQInv = 58728449u;  // q^-1 mod 2^32
constexpr int kN = 256;

template <int LEVEL>
struct Params;

template <>
struct Params<2> {
  static constexpr int LEVEL = 2, K = 4, L = 4, ETA = 2, TAU = 39, BETA = 78, GAMMA1 = 1 << 17,
                       GAMMA2 = (kQ - 1) / 88, OMEGA = 80, ETA_BITS = 3, Z_BITS = 18,
                       W1_BITS = 6;
};
template <>
struct Params<3> {
  static constexpr int LEVEL = 3, K = 6, L = 5, ETA = 4, TAU = 49, BETA = 196, GAMMA1 = 1 << 19,
                       GAMMA2 = (kQ - 1) / 32, OMEGA = 55, ETA_BITS = 4, Z_BITS = 20,
                       W1_BITS = 4;
};
template <>
struct Params<5> {
  static constexpr int LEVEL = 5, K = 8, L = 7, ETA = 2, TAU = 60, BETA = 120, GAMMA1 = 1 << 19,
                       GAMMA2 = (kQ - 1) / 32, OMEGA = 75, ETA_BITS = 3, Z_BITS = 20,
                       W1_BITS = 4;
};

// derived wire sizes (params.hpp:36-50)
template <class P>
struct Sizes {
  static constexpr int ETA_POLY = kN * P::ETA_BITS / 8;
  static constexpr int Z_POLY = kN * P::Z_BITS / 8;
  static constexpr int W1_POLY = kN * P::W1_BITS / 8;
  static constexpr int T1_POLY = 320, T0_POLY = 416;
  static constexpr int PK = 32 + P::K * T1_POLY;
  static constexpr int SK = 96 + (P::K + P::L) * ETA_POLY + P::K * T0_POLY;
  static constexpr int HINT = P::OMEGA + P::K;
  static constexpr int SIG = 32 + P::L * Z_POLY + HINT;
  static constexpr int W1_ALL = P::K * W1_POLY;
  static constexpr int SK_S1 = 96, SK_S2 = SK_S1 + P::L * ETA_POLY,
                       SK_T0 = SK_S2 + P::K * ETA_POLY;
};
static_assert(Sizes<Params<2>>::PK == 1312 && Sizes<Params<2>>::SK == 2528 &&
              Sizes<Params<2>>::SIG == 2420, "level 2 sizes");
static_assert(Sizes<Params<3>>::PK == 1952 && Sizes<Params<3>>::SK == 4000 &&
              Sizes<Params<3>>::SIG == 3293, "level 3 sizes");
static_assert(Sizes<Params<5>>::PK == 2592 && Sizes<Params<5>>::SK == 4864 &&
              Sizes<Params<5>>::SIG == 4595, "level 5 sizes");

// ---- Montgomery arithmetic, R = 2^32 (values as reduce.hpp:44-51) ---------------

// a*b*R^-1 mod q in (-q, q); needs |a*b| < 2^31 q.  lo(a*b - t*q) == 0 by
// construction, so the quotient is just the difference of the two high words.
__device__ __forceinline__ int32_t mont_mul(int32_t a, int32_t b) {
  const int32_t lo = a * b;
  const int32_t hi = __mulhi(a, b);
  const int32_t t = lo * (int32_t)kQInv;
  return hi - __mulhi(t, kQ);
}

// same with the constant operand's b*qinv supplied (twiddles): 3 IMAD + 1 IADD
__device__ __forceinline__ int32_t mont_mul_pre(int32_t a, int32_t b, int32_t bq) {
  const int32_t t = a * bq;
  return __mulhi(a, b) - __mulhi(t, kQ);
}

// a mod q, |result| <= 2^22 + 2^8*8191 < q, for any int32 a (cf. reduce.hpp:58-65
// without the final centering steps)
__device__ __forceinline__ int32_t reduce32(int32_t a) {
  const int32_t t = (a + (1 << 22)) >> 23;
  return a - t * kQ;
}

// (-q, q) -> [0, q)
__device__ __forceinline__ int32_t caddq(int32_t a) { return a + ((a >> 31) & kQ); }

// any int32 -> canonical [0, q)
__device__ __forceinline__ int32_t freeze(int32_t a) { return caddq(reduce32(a)); }

// canonical [0,q) -> centered (-(q-1)/2 .. (q-1)/2]
__device__ __forceinline__ int32_t center(int32_t a) {
  return a - ((((kQ - 1) / 2 - a) >> 31) & kQ);
}

// ---- rounding (values as rounding.hpp:13-59; standard round-3 formulas) -------------

__device__ __forceinline__ void power2round(int32_t a, int32_t& a1, int32_t& a0) {
  a1 = (a + 4095) >> 13;
  a0 = a - (a1 << 13);
}

template <int GAMMA2>
__device__ __forceinline__ int32_t decompose(int32_t a, int32_t& a0) {
  int32_t a1 = (a + 127) >> 7;
  if (GAMMA2 == (kQ - 1) / 32) {
    a1 = (a1 * 1025 + (1 << 21)) >> 22;
    a1 &= 15;
  } else {
    a1 = (a1 * 11275 + (1 << 23)) >> 24;
    a1 ^= ((43 - a1) >> 31) & a1;
  }
  a0 = a - a1 * 2 * GAMMA2;
  a0 -= (((kQ - 1) / 2 - a0) >> 31) & kQ;
  return a1;
}

template <int GAMMA2>
__device__ __forceinline__ int32_t highbits(int32_t a) {
  int32_t a0;
  return decompose<GAMMA2>(a, a0);
}

// r canonical; returns HighBits(r + z) given the hint bit
template <int GAMMA2>
__device__ __forceinline__ int32_t use_hint(int h, int32_t r) {
  constexpr int32_t M = (kQ - 1) / (2 * GAMMA2);
  int32_t r0;
  const int32_t r1 = decompose<GAMMA2>(r, r0);
  if (!h) return r1;
  if (r0 > 0) return r1 + 1 == M ? 0 : r1 + 1;
  return r1 == 0 ? M - 1 : r1 - 1;
}

// ---- small utilities -----------------------------------------------------------

// unaligned little-endian loads from global memory (byte-granular key/sig/msg offsets)
__device__ __forceinline__ uint32_t load_u32_unaligned(const uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  const unsigned sh = (a & 3) * 8;
  const uint32_t lo = __ldg(w);
  if (sh == 0) return lo;
  return __funnelshift_r(lo, __ldg(w + 1), sh);
}

// bits [bit, bit+width) of an LSB-first little-endian stream, width <= 24.
// Reads up to 3 bytes past the field's last byte within the same aligned words, so
// callers keep streams inside 4-byte-padded allocations.
__device__ __forceinline__ uint32_t load_bits(const uint8_t* base, unsigned bit, unsigned width) {
  const uint8_t* p = base + (bit >> 3);
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  const unsigned sh = (unsigned)(a & 3) * 8 + (bit & 7);
  const uint32_t lo = __ldg(w);
  uint32_t v = lo >> sh;
  if (sh + width > 32) v |= __ldg(w + 1) << (32 - sh);
  return v & ((1u << width) - 1);
}

#define DLB_CUDA_CHECK(x)                                   \
  do {                                                      \
    cudaError_t e_ = (x);                                   \
    if (e_ != cudaSuccess) return -1000 - (int)e_;          \
  } while (0)

}  // namespace dlb
