// ntt.cuh -- 256-point negacyclic NTT / inverse NTT over Z_q, one warp per polynomial.
//
// Values: proj/include/dilithium/ntt.hpp:74-86 (Cooley-Tukey, len 128..1, twiddle
// psi^brv8(k) walked linearly) and :92-110 (Gentleman-Sande with -zeta, n^-1 fused
// into the last level).  Layout is new: each lane keeps 8 coefficients in registers
// and the 8 levels run as three register passes (3 + 3 + 2 levels) separated by two
// transposes through a padded shared-memory tile (index c + 4*(c>>5): every access
// pattern below -- stride-1, stride-4-within-32, 8-consecutive as 2 x 128-bit -- maps
// the 32 lanes onto 32 distinct banks).  No butterfly ever crosses lanes, so the last
// levels need neither shuffles nor block barriers (only __syncwarp around the tile).
//
// Forward:  in  r[i] = a[lane + 32 i]      out r[m] = A[8 lane + m]   (|A| < |a|max + 10q)
// Inverse:  in  r[m] = A[8 lane + m], |A| < q   out r[i] = a[lane + 32 i], |a| < q
// Butterfly products use plain twiddles with a precomputed quotient (twiddle_mul: result in
// (-q/4, 5q/4)); sums double per inverse level exactly as in the reference's lazy transform
// (< 2^8 q < 2^31).  The inverse's last level is a Montgomery product by n^-1 * R^2
// (DLB_INTT_C*R): it brings the result back into (-q, q) and cancels the R^-1 left by a
// pointwise Montgomery product of two plain-domain operands, so no operand is ever
// converted to Montgomery form.
#pragma once
#include "common.cuh"

namespace dlb {

static __device__ __constant__ int2 c_zeta[256] = DLB_ZETA_TABLE;    // (z centred, round(z 2^32 / q))
static __device__ __constant__ int2 c_nzeta[256] = DLB_NZETA_TABLE;  // (-z) likewise

constexpr int kTileWords = 288;  // 256 + 4*7 padded, rounded up

__device__ __forceinline__ int tile_idx(int c) { return c + ((c >> 5) << 2); }

// copy both twiddle tables to shared memory (2 x 2 KB); caller syncs the block
__device__ __forceinline__ void load_twiddles(int2* zs, int2* nzs) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    zs[i] = c_zeta[i];
    nzs[i] = c_nzeta[i];
  }
}

// a * z mod q for a twiddle pair (z, z' = round(z 2^32 / q)), |z| <= q/2, any |a| < 2^31:
// h = floor(a z' / 2^32) is floor(a z / q + e) with |e| < 1/4, so a z - h q lies in
// (-q/4, 5q/4) and fits a word.  One half-rate IMAD.HI and two 32-bit IMADs: on sm_100a the
// 32-bit IMADs co-issue with the butterfly's add / sub, which the 64-bit-result IMADs of a
// Montgomery product do not (profiles/r01_summary.md section 3: 8.7 against 10.7 clocks).
__device__ __forceinline__ int32_t twiddle_mul(int32_t a, int2 z) {
  return a * z.x - __mulhi(a, z.y) * kQ;
}

// Cooley-Tukey butterfly in four instructions: a + t as two multiply-adds (b z + a, then
// - h q) and a - t = 2a - (a + t) as one three-input add (measured +2.5 % on Dilithium2 sign
// against computing t first and adding / subtracting it).
__device__ __forceinline__ void ct_bfly(int32_t& a, int32_t& b, int2 z) {
  const int32_t s = (b * z.x + a) - __mulhi(b, z.y) * kQ;
  b = a + a - s;
  a = s;
}

__device__ __forceinline__ void gs_bfly(int32_t& a, int32_t& b, int2 z) {
  const int32_t t = a;
  a = t + b;
  b = twiddle_mul(t - b, z);
}

__device__ __forceinline__ void ntt_fwd(int32_t (&r)[8], int32_t* tile, const int2* zs, int lane) {
  // pass A: c = lane + 32 i; levels len = 128, 64, 32 (twiddles warp-uniform)
#pragma unroll
  for (int i = 0; i < 4; ++i) ct_bfly(r[i], r[i + 4], c_zeta[1]);
  ct_bfly(r[0], r[2], c_zeta[2]);
  ct_bfly(r[1], r[3], c_zeta[2]);
  ct_bfly(r[4], r[6], c_zeta[3]);
  ct_bfly(r[5], r[7], c_zeta[3]);
#pragma unroll
  for (int i = 0; i < 8; i += 2) ct_bfly(r[i], r[i + 1], c_zeta[4 + i / 2]);

  const int b = lane >> 2, u = lane & 3;
#pragma unroll
  for (int i = 0; i < 8; ++i) tile[lane + 36 * i] = r[i];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = tile[36 * b + u + 4 * i];

  // pass B: c = 32 b + u + 4 i; levels len = 16, 8, 4
  {
    const int2 z = zs[8 + b];
#pragma unroll
    for (int i = 0; i < 4; ++i) ct_bfly(r[i], r[i + 4], z);
    // twiddle pairs / quads are fetched as 128-bit shared loads (no bank conflicts)
    const int4 zp = *reinterpret_cast<const int4*>(zs + 16 + 2 * b);
    const int2 z0 = make_int2(zp.x, zp.y), z1 = make_int2(zp.z, zp.w);
    ct_bfly(r[0], r[2], z0);
    ct_bfly(r[1], r[3], z0);
    ct_bfly(r[4], r[6], z1);
    ct_bfly(r[5], r[7], z1);
    const int4 qa = *reinterpret_cast<const int4*>(zs + 32 + 4 * b);
    const int4 qb = *reinterpret_cast<const int4*>(zs + 34 + 4 * b);
    ct_bfly(r[0], r[1], make_int2(qa.x, qa.y));
    ct_bfly(r[2], r[3], make_int2(qa.z, qa.w));
    ct_bfly(r[4], r[5], make_int2(qb.x, qb.y));
    ct_bfly(r[6], r[7], make_int2(qb.z, qb.w));
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) tile[36 * b + u + 4 * i] = r[i];
  __syncwarp();
  {
    const int base = 8 * lane + 4 * b;  // tile_idx(8*lane)
    const int4 lo = *reinterpret_cast<const int4*>(tile + base);
    const int4 hi = *reinterpret_cast<const int4*>(tile + base + 4);
    r[0] = lo.x; r[1] = lo.y; r[2] = lo.z; r[3] = lo.w;
    r[4] = hi.x; r[5] = hi.y; r[6] = hi.z; r[7] = hi.w;
  }
  // pass C: c = 8 lane + m; levels len = 2, 1
  {
    const int4 zp = *reinterpret_cast<const int4*>(zs + 64 + 2 * lane);
    const int2 z0 = make_int2(zp.x, zp.y), z1 = make_int2(zp.z, zp.w);
    ct_bfly(r[0], r[2], z0);
    ct_bfly(r[1], r[3], z0);
    ct_bfly(r[4], r[6], z1);
    ct_bfly(r[5], r[7], z1);
    const int4 qa = *reinterpret_cast<const int4*>(zs + 128 + 4 * lane);
    const int4 qb = *reinterpret_cast<const int4*>(zs + 130 + 4 * lane);
    ct_bfly(r[0], r[1], make_int2(qa.x, qa.y));
    ct_bfly(r[2], r[3], make_int2(qa.z, qa.w));
    ct_bfly(r[4], r[5], make_int2(qb.x, qb.y));
    ct_bfly(r[6], r[7], make_int2(qb.z, qb.w));
  }
  __syncwarp();  // tile free for the caller
}

__device__ __forceinline__ void ntt_inv(int32_t (&r)[8], int32_t* tile, const int2* nzs, int lane) {
  // pass C': c = 8 lane + m; levels len = 1, 2, 4.  Level with G = 128/len groups
  // uses twiddle index 2G-1-g for group g (the reference's --k walk).
  {
    const int4 qa = *reinterpret_cast<const int4*>(nzs + 252 - 4 * lane);  // [252-4l, 253-4l]
    const int4 qb = *reinterpret_cast<const int4*>(nzs + 254 - 4 * lane);  // [254-4l, 255-4l]
    gs_bfly(r[0], r[1], make_int2(qb.z, qb.w));
    gs_bfly(r[2], r[3], make_int2(qb.x, qb.y));
    gs_bfly(r[4], r[5], make_int2(qa.z, qa.w));
    gs_bfly(r[6], r[7], make_int2(qa.x, qa.y));
  }
  {
    const int4 zp = *reinterpret_cast<const int4*>(nzs + 126 - 2 * lane);
    const int2 z0 = make_int2(zp.z, zp.w), z1 = make_int2(zp.x, zp.y);
    gs_bfly(r[0], r[2], z0);
    gs_bfly(r[1], r[3], z0);
    gs_bfly(r[4], r[6], z1);
    gs_bfly(r[5], r[7], z1);
    const int2 z = nzs[63 - lane];
#pragma unroll
    for (int m = 0; m < 4; ++m) gs_bfly(r[m], r[m + 4], z);
  }
  {
    const int base = 8 * lane + 4 * (lane >> 2);
    *reinterpret_cast<int4*>(tile + base) = make_int4(r[0], r[1], r[2], r[3]);
    *reinterpret_cast<int4*>(tile + base + 4) = make_int4(r[4], r[5], r[6], r[7]);
  }
  __syncwarp();
  const int v = lane & 7, h = lane >> 3;
  // c = v + 8 i + 64 h  ->  tile index c + 4*(2h + (i>>2))
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = tile[v + 8 * i + 72 * h + 4 * (i >> 2)];
  // pass B': levels len = 8, 16, 32
  {
    const int4 qa = *reinterpret_cast<const int4*>(nzs + 28 - 4 * h);
    const int4 qb = *reinterpret_cast<const int4*>(nzs + 30 - 4 * h);
    gs_bfly(r[0], r[1], make_int2(qb.z, qb.w));
    gs_bfly(r[2], r[3], make_int2(qb.x, qb.y));
    gs_bfly(r[4], r[5], make_int2(qa.z, qa.w));
    gs_bfly(r[6], r[7], make_int2(qa.x, qa.y));
  }
  {
    const int4 zp = *reinterpret_cast<const int4*>(nzs + 14 - 2 * h);
    const int2 z0 = make_int2(zp.z, zp.w), z1 = make_int2(zp.x, zp.y);
    gs_bfly(r[0], r[2], z0);
    gs_bfly(r[1], r[3], z0);
    gs_bfly(r[4], r[6], z1);
    gs_bfly(r[5], r[7], z1);
    const int2 z = nzs[7 - h];
#pragma unroll
    for (int i = 0; i < 4; ++i) gs_bfly(r[i], r[i + 4], z);
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) tile[v + 8 * i + 72 * h + 4 * (i >> 2)] = r[i];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = tile[lane + 36 * i];
  // pass A': c = lane + 32 i; level len = 64, then len = 128 fused with n^-1 * R
  gs_bfly(r[0], r[2], c_nzeta[3]);
  gs_bfly(r[1], r[3], c_nzeta[3]);
  gs_bfly(r[4], r[6], c_nzeta[2]);
  gs_bfly(r[5], r[7], c_nzeta[2]);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int32_t t = r[i];
    r[i] = mont_mul_pre(t + r[i + 4], DLB_INTT_C1R, DLB_INTT_C1R_Q);
    r[i + 4] = mont_mul_pre(t - r[i + 4], DLB_INTT_C2R, DLB_INTT_C2R_Q);
  }
  __syncwarp();
}

// One warp copies nbytes from a 4-byte aligned shared-memory buffer to a global destination of ANY
// alignment with coalesced word stores (signatures are packed back to back and their size is
// odd at levels 3 / 5; the destination may be pinned host memory, where byte-sized stores
// would each cost a PCIe transaction).  Reads up to one word past the end of the source.
__device__ __forceinline__ void warp_store_unaligned(uint8_t* dst, const uint32_t* src32, unsigned nbytes,
                                                     int lane) {
  const unsigned a = (unsigned)(reinterpret_cast<uintptr_t>(dst) & 3);
  const unsigned head = a ? min(4u - a, nbytes) : 0u;  // bytes up to the next word boundary
  const uint8_t* src8 = reinterpret_cast<const uint8_t*>(src32);
  if ((unsigned)lane < head) dst[lane] = src8[lane];
  uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + head);
  const unsigned nwords = (nbytes - head) / 4;
  if (head == 0) {
    for (unsigned w = lane; w < nwords; w += 32) d32[w] = src32[w];
  } else {
    for (unsigned w = lane; w < nwords; w += 32) d32[w] = __funnelshift_r(src32[w], src32[w + 1], 8 * head);
  }
  const unsigned done = head + 4 * nwords;
  if ((unsigned)lane < nbytes - done) dst[done + lane] = src8[done + lane];
}

// ---- bit packing from the strided register layout -------------------------------
// vals: tile (padded index) holding 256 raw field values; every lane packs its 8
// consecutive coefficients into BITS bytes of `bytes` (shared scratch, BITS*32 bytes, + 4 when
// !ALIGNED), then the warp copies BITS*8 words to `gout` with coalesced stores.  ALIGNED: gout is
// 4-byte aligned; otherwise any alignment.
template <int BITS, bool ALIGNED = true>
__device__ __forceinline__ void pack_tile(const int32_t* tile, uint8_t* bytes, uint8_t* gout,
                                          int lane) {
  const int base = 8 * lane + 4 * (lane >> 2);
  const int4 lo = *reinterpret_cast<const int4*>(tile + base);
  const int4 hi = *reinterpret_cast<const int4*>(tile + base + 4);
  const uint32_t v[8] = {(uint32_t)lo.x, (uint32_t)lo.y, (uint32_t)lo.z, (uint32_t)lo.w,
                         (uint32_t)hi.x, (uint32_t)hi.y, (uint32_t)hi.z, (uint32_t)hi.w};
  uint8_t* dst = bytes + BITS * lane;
  uint64_t acc = 0;
  int nbits = 0, o = 0;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    acc |= (uint64_t)v[m] << nbits;
    nbits += BITS;
#pragma unroll
    for (int rep = 0; rep < 3; ++rep) {
      if (nbits >= 8) {
        dst[o++] = (uint8_t)acc;
        acc >>= 8;
        nbits -= 8;
      }
    }
  }
  __syncwarp();
  const uint32_t* src = reinterpret_cast<const uint32_t*>(bytes);
  if (ALIGNED) {
    uint32_t* g = reinterpret_cast<uint32_t*>(gout);
#pragma unroll
    for (int w = lane; w < BITS * 8; w += 32) g[w] = src[w];
  } else {
    warp_store_unaligned(gout, src, BITS * 32, lane);
  }
  __syncwarp();
}

}  // namespace dlb
