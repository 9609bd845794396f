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
// FIPS 204 (ML-DSA-44 / 65 / 87): the ring, samplers, bounds and codecs of the round-3 sets;
// what differs is hashing only -- H(xi || k || l) in key generation, a 64-byte tr, the
// message prefix 0 || |ctx| || ctx, rho'' = H(K || rnd || mu), and a commitment hash of
// lambda/4 = 32 / 48 / 64 bytes that SampleInBall absorbs whole (FIPS 204 Alg. 6-8, 29).
// Selected through the flags below; the round-3 instantiations compile to the same code as
// before.  Deterministic signing (rnd = 0) with an empty context string.
template <>
struct Params<44> : Params<2> {
  static constexpr int LEVEL = 44;
};
template <>
struct Params<65> : Params<3> {
  static constexpr int LEVEL = 65;
};
template <>
struct Params<87> : Params<5> {
  static constexpr int LEVEL = 87;
};

template <class P>
struct Hashing {
  static constexpr bool MLDSA = P::LEVEL > 5;
  static constexpr int TR = MLDSA ? 64 : 32;                                      // bytes of tr
  static constexpr int CT = P::LEVEL == 65 ? 48 : (P::LEVEL == 87 ? 64 : 32);     // bytes of c~
  static constexpr int TRW = TR / 8, CTW = CT / 8;                                // 64-bit words
};

// derived wire sizes (params.hpp:36-50)
template <class P>
struct Sizes {
  static constexpr int ETA_POLY = kN * P::ETA_BITS / 8;
  static constexpr int Z_POLY = kN * P::Z_BITS / 8;
  static constexpr int W1_POLY = kN * P::W1_BITS / 8;
  static constexpr int T1_POLY = 320, T0_POLY = 416;
  static constexpr int PK = 32 + P::K * T1_POLY;
  static constexpr int SK_S1 = 64 + Hashing<P>::TR, SK_S2 = SK_S1 + P::L * ETA_POLY,
                       SK_T0 = SK_S2 + P::K * ETA_POLY;
  static constexpr int SK = SK_T0 + P::K * T0_POLY;
  static constexpr int HINT = P::OMEGA + P::K;
  static constexpr int SIG_Z = Hashing<P>::CT;  // offset of z behind the commitment hash
  static constexpr int SIG = SIG_Z + P::L * Z_POLY + HINT;
  static constexpr int W1_ALL = P::K * W1_POLY;
};
static_assert(Sizes<Params<2>>::PK == 1312 && Sizes<Params<2>>::SK == 2528 &&
              Sizes<Params<2>>::SIG == 2420, "level 2 sizes");
static_assert(Sizes<Params<3>>::PK == 1952 && Sizes<Params<3>>::SK == 4000 &&
              Sizes<Params<3>>::SIG == 3293, "level 3 sizes");
static_assert(Sizes<Params<5>>::PK == 2592 && Sizes<Params<5>>::SK == 4864 &&
              Sizes<Params<5>>::SIG == 4595, "level 5 sizes");
static_assert(Sizes<Params<44>>::PK == 1312 && Sizes<Params<44>>::SK == 2560 &&
              Sizes<Params<44>>::SIG == 2420, "ML-DSA-44 sizes (FIPS 204 table 2)");
static_assert(Sizes<Params<65>>::PK == 1952 && Sizes<Params<65>>::SK == 4032 &&
              Sizes<Params<65>>::SIG == 3309, "ML-DSA-65 sizes");
static_assert(Sizes<Params<87>>::PK == 2592 && Sizes<Params<87>>::SK == 4896 &&
              Sizes<Params<87>>::SIG == 4627, "ML-DSA-87 sizes");

// ---- Montgomery arithmetic, R = 2^32 (values as reduce.hpp:44-51) ---------------

// a*b*R^-1 mod q in (-q, q); needs |a*b| < 2^31 q.  With t = lo(p) * q^-1 the low words of p
// and t*q are equal, so (p - t*q) / 2^32 is exactly hi(p) - hi(t*q): one IMAD.HI and one
// subtraction, no carry chain (a 64-bit `mad.wide` of -q onto p compiles to five instructions).
__device__ __forceinline__ int32_t mont_fold(int64_t p, int32_t t) {
  return (int32_t)(p >> 32) - __mulhi(t, kQ);
}

__device__ __forceinline__ int32_t mont_mul(int32_t a, int32_t b) {
  int64_t p;
  asm("mul.wide.s32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
  const int32_t t = (int32_t)p * (int32_t)kQInv;
  return mont_fold(p, t);
}

// 64-bit multiply-accumulate and a single Montgomery fold at the end: a row of the
// matrix-vector product costs L IMAD.WIDE + 2 instead of L full Montgomery products.
// |acc| must stay below 2^31 q: L <= 7 terms of |a| < 2^23 times |b| < 2^27.
__device__ __forceinline__ int64_t mac_wide(int64_t acc, int32_t a, int32_t b) {
  // plain C++: ptxas keeps this as one IMAD.WIDE with a 64-bit addend, while the same
  // operation written as inline `mad.wide.s32` is split into IMAD.WIDE + IADD3 + IMAD.X
  return acc + (int64_t)a * (int64_t)b;
}

__device__ __forceinline__ int32_t mont_reduce64(int64_t p) {
  const int32_t t = (int32_t)p * (int32_t)kQInv;
  return mont_fold(p, t);
}

// same with the constant operand's b*qinv supplied (last inverse-NTT level): IMAD + 2 IMAD.WIDE
__device__ __forceinline__ int32_t mont_mul_pre(int32_t a, int32_t b, int32_t bq) {
  const int32_t t = a * bq;
  int64_t p;
  asm("mul.wide.s32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
  return mont_fold(p, t);
}

// a mod q, |result| <= 2^22 + 2^8*8191 < q, for any int32 a (cf. reduce.hpp:58-65
// without the final centering steps)
__device__ __forceinline__ int32_t reduce32(int32_t a) {
  const int32_t t = (a + (1 << 22)) >> 23;
  return a - t * kQ;
}

// [-q, 2^31 - q) -> a + q if negative: as unsigned numbers the wrong candidate is the huge
// one, so an unsigned minimum picks the representative (two instructions, no mask)
__device__ __forceinline__ int32_t caddq(int32_t a) {
  const uint32_t u = (uint32_t)a;
  return (int32_t)min(u, u + (uint32_t)kQ);
}

// (-q, 2q) -> [0, q): the one candidate of a - q, a, a + q that is not negative or too large
__device__ __forceinline__ int32_t freeze_near(int32_t a) {
  const uint32_t u = (uint32_t)a;
  return (int32_t)min(min(u, u + (uint32_t)kQ), u - (uint32_t)kQ);
}

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
    a1 = (int32_t)min((uint32_t)a1, (uint32_t)a1 - 44u);  // a1 in [0, 44]: 44 -> 0
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

// Coherent ("weak", L1-cacheable) global loads that the compiler may not turn into the
// read-only ld.global.nc form.  The signing scheduler reads data of batches that were
// published after its kernel started; each CTA orders those reads behind an acquire load of the
// batch's gate word (which also drops stale L1 lines), a guarantee the non-coherent path is
// outside of.  Not volatile: the loads may be scheduled freely behind their address.
__device__ __forceinline__ uint64_t ld_weak(const uint64_t* p) {
  uint64_t v;
  asm("ld.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_weak(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int4 ld_weak(const int4* p) {
#ifdef DLB_AB_LDG
  return __ldg(p);  // A/B measurement only: the non-coherent path is not safe here
#endif
  int4 v;
  asm("ld.global.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint8_t ld_weak(const uint8_t* p) {
  uint32_t v;
  asm("ld.global.u8 %0, [%1];" : "=r"(v) : "l"(p));
  return (uint8_t)v;
}

// unaligned little-endian loads from global memory (byte-granular key/sig/msg offsets)
// (NC = false: coherent loads, see ld_weak)
template <bool NC = true>
__device__ __forceinline__ uint32_t load_u32_unaligned(const uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  const unsigned sh = (a & 3) * 8;
  const uint32_t lo = NC ? __ldg(w) : ld_weak(w);
  if (sh == 0) return lo;
  return __funnelshift_r(lo, NC ? __ldg(w + 1) : ld_weak(w + 1), sh);
}

// bits [bit, bit+width) of an LSB-first little-endian stream, width <= 24.
// Reads whole aligned 32-bit words, so it never touches a word that holds no byte of
// the field.  NC = true uses the read-only (ld.global.nc) path and is only for buffers
// that no thread writes during the kernel; scratch written inside the persistent
// signing kernel is read with NC = false.
template <bool NC>
__device__ __forceinline__ uint32_t load_bits_t(const uint8_t* base, unsigned bit, unsigned width) {
  const uint8_t* p = base + (bit >> 3);
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  const unsigned sh = (unsigned)(a & 3) * 8 + (bit & 7);
  const uint32_t lo = NC ? __ldg(w) : *w;
  uint32_t v = lo >> sh;
  if (sh + width > 32) v |= (NC ? __ldg(w + 1) : w[1]) << (32 - sh);
  return v & ((1u << width) - 1);
}

__device__ __forceinline__ uint32_t load_bits(const uint8_t* base, unsigned bit, unsigned width) {
  return load_bits_t<true>(base, bit, width);
}

__device__ __forceinline__ uint32_t load_bits_rw(const uint8_t* base, unsigned bit, unsigned width) {
  return load_bits_t<false>(base, bit, width);
}

// L1 prefetch of [p, p+bytes) by one warp (128-byte lines)
__device__ __forceinline__ void prefetch_l1(const void* p, unsigned bytes, int lane) {
  const char* c = static_cast<const char*>(p);
  for (unsigned o = lane * 128u; o < bytes; o += 32u * 128u)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(c + o));
}

#define DLB_CUDA_CHECK(x)                                   \
  do {                                                      \
    cudaError_t e_ = (x);                                   \
    if (e_ != cudaSuccess) return -1000 - (int)e_;          \
  } while (0)

}  // namespace dlb
