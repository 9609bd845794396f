// verify_keygen.cuh -- ring-arithmetic kernels of verification and key generation,
// one warp per task, everything between the packed inputs and the packed outputs in
// registers / per-warp shared memory.
//
// Semantics: scheme.hpp:277-318 (verify), :68-104 (keygen); codecs packing.hpp:56-98,
// strict hint decode packing.hpp:122-140; UseHint / Power2Round rounding.hpp:13-59.
#pragma once
#include "ntt.cuh"

// Matrix loads in flight per thread in the arithmetic kernels' accumulation loops (2 x 16 bytes
// per unrolled iteration).  These kernels stream every task's matrix from HBM (22 KB per
// Dilithium2 key, 3.4 TB/s while they run); four iterations in flight measured +0.4 / +1.9 /
// +3.9 % keygen throughput at Dilithium2 / 3 / 5 against one, eight no better
// (profiles/r02_arith_unroll_ab.txt).
// k_verify_arith at L = 4 is the exception: fully unrolled it needs 86 registers instead of 64,
// loses three resident CTAs per SM and 3 % (28.8 -> 27.9 M verify/s), so it keeps one iteration.
#ifndef DLB_ARITH_J_UNROLL
#define DLB_ARITH_J_UNROLL 4
#endif
#ifndef DLB_VERIFY_J_UNROLL
#define DLB_VERIFY_J_UNROLL (P::L > 4 ? DLB_ARITH_J_UNROLL : 1)
#endif
#define DLB_PRAGMA_(x) _Pragma(#x)
#define DLB_PRAGMA(x) DLB_PRAGMA_(x)
#define DLB_ARITH_J_PRAGMA DLB_PRAGMA(unroll DLB_ARITH_J_UNROLL)
#define DLB_VERIFY_J_PRAGMA DLB_PRAGMA(unroll DLB_VERIFY_J_UNROLL)

namespace dlb {

// per-warp shared scratch
template <class P>
struct WarpScratch {
  int32_t tile[kTileWords];            // NTT transposes / value staging
  int32_t vhat[P::L][8][32];           // transformed vector, lane-private slots
  uint32_t hbits[P::K][8];             // hint bitmap (verify)
  __align__(16) uint8_t bytes[20 * 32];  // bit-packing scratch (max 20 bits/coeff)
};

// ---- verify -----------------------------------------------------------------------
// Inputs per task t: pk (pk_stride apart; 0 = one shared key), sig (sig_stride), the
// expanded matrix A[key][K*L][256] (raw ExpandA output, [0,q)), the challenge c8[t][256].
// Outputs: w1buf[t][W1_ALL] packed w1' and pre_ok[t] (strict hint decode and z-norm).
template <class P, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_verify_arith(unsigned n, const uint8_t* __restrict__ pk, size_t pk_stride,
                   const uint8_t* __restrict__ sig, size_t sig_stride,
                   const int32_t* __restrict__ A, size_t a_stride /* int32 per key, 0 shared */,
                   const uint32_t* __restrict__ key_idx /* nullable: key of task t, else t */,
                   const int8_t* __restrict__ c8, uint8_t* __restrict__ w1buf,
                   uint8_t* __restrict__ pre_ok) {
  using S = Sizes<P>;
  __shared__ __align__(16) int2 zs[256], nzs[256];
  __shared__ __align__(16) WarpScratch<P> scratch[WARPS];
  load_twiddles(zs, nzs);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned t = blockIdx.x * WARPS + warp;
  if (t >= n) return;
  WarpScratch<P>& ws = scratch[warp];
  const size_t kt = key_idx ? (size_t)__ldg(key_idx + t) : (size_t)t;
  const uint8_t* tpk = pk + kt * pk_stride;
  const uint8_t* tsig = sig + (size_t)t * sig_stride;
  const int32_t* tA = A + kt * a_stride;
  bool ok = true;

  // -- strict hint decode into a bitmap (packing.hpp:122-140)
  {
    const uint8_t* hint = tsig + S::SIG_Z + P::L * S::Z_POLY;
    unsigned cnt[P::K];
    unsigned prev = 0;
#pragma unroll
    for (int i = 0; i < P::K; ++i) {
      cnt[i] = __ldg(hint + P::OMEGA + i);
      if (cnt[i] < prev || cnt[i] > (unsigned)P::OMEGA) ok = false;
      prev = cnt[i];
    }
    for (int w = lane; w < P::K * 8; w += 32) (&ws.hbits[0][0])[w] = 0;
    __syncwarp();
    for (unsigned j = lane; j < (unsigned)P::OMEGA; j += 32) {
      const unsigned pos = __ldg(hint + j);
      int poly = -1;
      unsigned start = 0;
#pragma unroll
      for (int i = 0; i < P::K; ++i) {
        if (poly < 0) {
          if (j < cnt[i]) poly = i;
          else start = max(start, cnt[i]);
        }
      }
      if (poly >= 0) {
        if (j > start && pos <= (unsigned)__ldg(hint + j - 1)) ok = false;
        atomicOr(&ws.hbits[poly][pos >> 5], 1u << (pos & 31));
      } else if (pos != 0) {
        ok = false;
      }
    }
    __syncwarp();
  }

  int32_t r[8];
  // -- z: unpack, infinity-norm check, transform (scheme.hpp:284,291-292)
#pragma unroll 1
  for (int j = 0; j < P::L; ++j) {
    const uint8_t* zb = tsig + S::SIG_Z + j * S::Z_POLY;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const unsigned c = lane + 32 * i;
      const int32_t z = P::GAMMA1 - (int32_t)load_bits(zb, c * P::Z_BITS, P::Z_BITS);
      if (abs(z) >= P::GAMMA1 - P::BETA) ok = false;
      r[i] = z;
    }
    ntt_fwd(r, ws.tile, zs, lane);
#pragma unroll
    for (int m = 0; m < 8; ++m) ws.vhat[j][m][lane] = r[m];
  }
  // -- challenge
  int32_t ch[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) ch[i] = c8[(size_t)t * kN + lane + 32 * i];
  ntt_fwd(ch, ws.tile, zs, lane);

  // -- rows: w1' = UseHint(h, A z - c t1 2^d)  (scheme.hpp:299-309)
#pragma unroll 1
  for (int i = 0; i < P::K; ++i) {
    const uint8_t* t1b = tpk + 32 + i * S::T1_POLY;
#pragma unroll
    for (int e = 0; e < 8; ++e) r[e] = (int32_t)(load_bits(t1b, (lane + 32 * e) * 10, 10) << 13);
    ntt_fwd(r, ws.tile, zs, lane);
    // 64-bit accumulation of A z - c t1, one Montgomery fold per coefficient.  t1hat is
    // reduced first so |c t1| < 2^27 * 2^23 like every other term (8 terms max).
    int64_t acc64[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) acc64[m] = mac_wide(0, -ch[m], reduce32(r[m]));
    DLB_VERIFY_J_PRAGMA
    for (int j = 0; j < P::L; ++j) {
      const int4* ap = reinterpret_cast<const int4*>(tA + (size_t)(i * P::L + j) * kN) + 2 * lane;
      const int4 a0 = __ldg(ap), a1 = __ldg(ap + 1);
      const int32_t a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int m = 0; m < 8; ++m) acc64[m] = mac_wide(acc64[m], a[m], ws.vhat[j][m][lane]);
    }
    int32_t acc[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) acc[m] = mont_reduce64(acc64[m]);
    ntt_inv(acc, ws.tile, nzs, lane);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int h = (ws.hbits[i][e] >> lane) & 1;  // coefficient lane + 32 e
      ws.tile[lane + 36 * e] = use_hint<P::GAMMA2>(h, caddq(acc[e]));
    }
    __syncwarp();
    pack_tile<P::W1_BITS>(ws.tile, ws.bytes, w1buf + (size_t)t * S::W1_ALL + i * S::W1_POLY, lane);
  }
  ok = __all_sync(0xffffffffu, ok);
  if (lane == 0) pre_ok[t] = ok ? 1 : 0;
}

// ---- keygen -----------------------------------------------------------------------
// Inputs per task: seeds[t][128] = rho | rho' | K, s8[t][L+K][256] (ExpandS output),
// A[t][K*L][256].  Outputs: pk (all but nothing missing), sk except tr (bytes 64..95),
// which k_hash_tr fills from the finished pk.
template <class P, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_keygen_arith(unsigned n, const uint8_t* __restrict__ seeds, const int8_t* __restrict__ s8,
                   const int32_t* __restrict__ A, uint8_t* __restrict__ pk,
                   uint8_t* __restrict__ sk) {
  using S = Sizes<P>;
  __shared__ __align__(16) int2 zs[256], nzs[256];
  __shared__ __align__(16) WarpScratch<P> scratch[WARPS];
  load_twiddles(zs, nzs);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned t = blockIdx.x * WARPS + warp;
  if (t >= n) return;
  WarpScratch<P>& ws = scratch[warp];
  uint8_t* tpk = pk + (size_t)t * S::PK;
  uint8_t* tsk = sk + (size_t)t * S::SK;
  const int8_t* ts = s8 + (size_t)t * (P::K + P::L) * kN;
  const int32_t* tA = A + (size_t)t * P::K * P::L * kN;

  // rho -> pk, sk; K -> sk (packing.hpp:174-213)
  {
    const uint32_t* sd = reinterpret_cast<const uint32_t*>(seeds + (size_t)t * 128);
    if (lane < 8) {
      const uint32_t w = sd[lane];
      reinterpret_cast<uint32_t*>(tpk)[lane] = w;
      reinterpret_cast<uint32_t*>(tsk)[lane] = w;
    } else if (lane < 16) {
      reinterpret_cast<uint32_t*>(tsk)[lane] = sd[24 + lane - 8];  // K = seed bytes 96..127
    }
  }
  int32_t r[8];
#pragma unroll 1
  for (int j = 0; j < P::L; ++j) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      r[i] = ts[j * kN + lane + 32 * i];
      ws.tile[lane + 36 * i] = P::ETA - r[i];
    }
    __syncwarp();
    pack_tile<P::ETA_BITS>(ws.tile, ws.bytes, tsk + S::SK_S1 + j * S::ETA_POLY, lane);
    ntt_fwd(r, ws.tile, zs, lane);
#pragma unroll
    for (int m = 0; m < 8; ++m) ws.vhat[j][m][lane] = r[m];
  }
#pragma unroll 1
  for (int i = 0; i < P::K; ++i) {
    int64_t acc64[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) acc64[m] = 0;
    DLB_ARITH_J_PRAGMA
    for (int j = 0; j < P::L; ++j) {
      const int4* ap = reinterpret_cast<const int4*>(tA + (size_t)(i * P::L + j) * kN) + 2 * lane;
      const int4 a0 = __ldg(ap), a1 = __ldg(ap + 1);
      const int32_t a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int m = 0; m < 8; ++m) acc64[m] = mac_wide(acc64[m], a[m], ws.vhat[j][m][lane]);
    }
    int32_t acc[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) acc[m] = mont_reduce64(acc64[m]);
    ntt_inv(acc, ws.tile, nzs, lane);
    // t = A s1 + s2 canonical; Power2Round; s2, t1, t0 codecs (scheme.hpp:91-99)
    int32_t s2v[8], t0v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      s2v[e] = ts[(P::L + i) * kN + lane + 32 * e];
      const int32_t tc = freeze(acc[e] + s2v[e]);
      int32_t hi;
      power2round(tc, hi, t0v[e]);
      ws.tile[lane + 36 * e] = hi;
    }
    __syncwarp();
    pack_tile<10>(ws.tile, ws.bytes, tpk + 32 + i * S::T1_POLY, lane);
#pragma unroll
    for (int e = 0; e < 8; ++e) ws.tile[lane + 36 * e] = 4096 - t0v[e];
    __syncwarp();
    pack_tile<13>(ws.tile, ws.bytes, tsk + S::SK_T0 + i * S::T0_POLY, lane);
#pragma unroll
    for (int e = 0; e < 8; ++e) ws.tile[lane + 36 * e] = P::ETA - s2v[e];
    __syncwarp();
    pack_tile<P::ETA_BITS>(ws.tile, ws.bytes, tsk + S::SK_S2 + i * S::ETA_POLY, lane);
  }
}

}  // namespace dlb
