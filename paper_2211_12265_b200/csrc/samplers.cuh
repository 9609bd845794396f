// samplers.cuh -- SHAKE-based samplers and hashes, one sponge per thread.
//
// Semantics: proj/include/dilithium/sampling.hpp:16-24 (order-preserving rejection),
// :42-56 ExpandA, :61-79 ExpandS, :83-92 ExpandMask, :97-120 SampleInBall;
// scheme.hpp:70-76,102,240-248,158-163 for the scheme hashes.
//
// A warp runs 32 independent streams in lockstep.  Rejection sampling is done by
// each lane on its own stream (sequential, hence trivially order-preserving and equal
// to rej_compact); accepted coefficients are staged per lane in bank-conflict-free
// padded shared memory and flushed by the whole warp as coalesced 128-byte stores, so
// polynomials land in HBM in plain [poly][256] order.
#pragma once
#include "keccak.cuh"

namespace dlb {

constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ uint64_t load_u64_unaligned(const uint8_t* p) {
  return (uint64_t)load_u32_unaligned(p) | ((uint64_t)load_u32_unaligned(p + 4) << 32);
}

// --------------------------------------------------------------------- ExpandA
// One stream per matrix polynomial: stream p -> key p/(K*L), entry (i,j) row-major.
// out[p][256] int32 in [0,q).  rho of key n at rho_base + n*rho_stride.
constexpr int kExpandAStageStride = 57;  // 56 candidates per block, odd stride

// One warp, 32 consecutive streams starting at p0 (the warp-uniform first stream); stage = the
// warp's [32][kExpandAStageStride] shared-memory rows.  NC = false inside the persistent signing
// kernel (keys published after the kernel started are read with coherent loads).
template <class P, bool NC>
__device__ __forceinline__ void expand_a_warp(const uint8_t* __restrict__ rho_base, size_t rho_stride,
                                              unsigned p0, unsigned n_streams, int32_t* __restrict__ out,
                                              int32_t (*stage)[kExpandAStageStride], int lane) {
  const unsigned p = p0 + lane;
  const bool active = p < n_streams;
  constexpr int KL = P::K * P::L;

  uint64_t s[25];
  keccak_clear(s);
  if (active) {
    const unsigned key = p / KL, r = p % KL;
    const unsigned i = r / P::L, j = r % P::L;
    const uint8_t* rho = rho_base + (size_t)key * rho_stride;
#pragma unroll
    for (int w = 0; w < 4; ++w)
      s[w] = (uint64_t)load_u32_unaligned<NC>(rho + 8 * w) | ((uint64_t)load_u32_unaligned<NC>(rho + 8 * w + 4) << 32);
    // nonce (i<<8)|j little-endian, then the 0x1F suffix; 0x80 closes the 168-byte block
    s[4] = (uint64_t)j | ((uint64_t)i << 8) | ((uint64_t)0x1F << 16);
    s[20] = 0x8000000000000000ull;
  }
  unsigned ctr = active ? 0u : (unsigned)kN;
  int32_t* row = stage[lane];

  while (true) {
    keccak_f1600(s);
    unsigned n = 0;
#pragma unroll
    for (int g = 0; g < 7; ++g) {
      const uint64_t w0 = s[3 * g], w1 = s[3 * g + 1], w2 = s[3 * g + 2];
      const uint32_t c[8] = {
          (uint32_t)w0,         (uint32_t)(w0 >> 24), (uint32_t)((w0 >> 48) | (w1 << 16)),
          (uint32_t)(w1 >> 8),  (uint32_t)(w1 >> 32), (uint32_t)((w1 >> 56) | (w2 << 8)),
          (uint32_t)(w2 >> 16), (uint32_t)(w2 >> 40)};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t t = c[e] & 0x7FFFFF;
        row[n] = (int32_t)t;  // overwritten by the next candidate when rejected
        n += t < (uint32_t)kQ;
      }
    }
    // copy-out: row src holds cnt <= 56 accepted values that go to coefficients [base, base + cnt)
    // of stream p0 + src -- one shuffle of the packed (cnt, base) per row, two predicated copies
    const unsigned desc = min(n, (unsigned)kN - ctr) | (ctr << 8);
    int32_t* obase = out + (size_t)p0 * kN + lane;
    __syncwarp();
#pragma unroll 8
    for (int src = 0; src < 32; ++src) {
      const unsigned d = __shfl_sync(kFullMask, desc, src);
      const unsigned cnt = d & 0xFFu;
      int32_t* dst = obase + src * kN + (d >> 8);
      if ((unsigned)lane < cnt) dst[0] = stage[src][lane];
      if ((unsigned)lane + 32u < cnt) dst[32] = stage[src][lane + 32];
    }
    ctr = min((unsigned)kN, ctr + n);
    __syncwarp();
    if (__all_sync(kFullMask, ctr >= (unsigned)kN)) break;
  }
}

template <class P, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_expand_a(const uint8_t* __restrict__ rho_base, size_t rho_stride, unsigned n_streams,
               int32_t* __restrict__ out) {
  __shared__ int32_t stage[WARPS][32][kExpandAStageStride];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned p0 = (blockIdx.x * WARPS + warp) * 32;
  if (p0 >= n_streams) return;  // whole warp idle
  expand_a_warp<P, true>(rho_base, rho_stride, p0, n_streams, out, stage[warp], lane);
}

// --------------------------------------------------------------------- ExpandS
// Streams: task t, polynomial r in [0, L+K) (s1 then s2), nonce = r.
// rho' of task t at seeds + t*seed_stride (64 bytes, 8-byte aligned).
// out8[t][r][256] int8 in [-eta, eta].
constexpr int kByteRowStride = 260;  // 65 words: odd word stride, 4-byte aligned rows

template <class P, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_expand_s(const uint8_t* __restrict__ seeds, size_t seed_stride, unsigned n_streams,
               int8_t* __restrict__ out8) {
  __shared__ __align__(16) int8_t stage[WARPS][32][kByteRowStride];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned p0 = (blockIdx.x * WARPS + warp) * 32;
  if (p0 >= n_streams) return;
  const unsigned p = p0 + lane;
  const bool active = p < n_streams;
  constexpr int PV = P::K + P::L;

  uint64_t s[25];
  keccak_clear(s);
  if (active) {
    const unsigned task = p / PV, r = p % PV;
    const uint64_t* rp = reinterpret_cast<const uint64_t*>(seeds + (size_t)task * seed_stride);
#pragma unroll
    for (int w = 0; w < 8; ++w) s[w] = __ldg(rp + w);
    s[8] = (uint64_t)r | ((uint64_t)0x1F << 16);
    s[16] = 0x8000000000000000ull;
  }
  unsigned ctr = active ? 0u : (unsigned)kN;
  int8_t* row = stage[warp][lane];

  while (true) {
    keccak_f1600(s);
#pragma unroll
    for (int w = 0; w < kWords256; ++w) {
#ifndef DLB_EXPAND_S_NO_EARLY_EXIT
      // The last block of a stream is mostly surplus (eta = 2: 256 of the first 272 nibbles are
      // accepted on average, the second block supplies the last few): stop at the first word
      // pair by which every lane of the warp is full.
      if (w > 0 && (w & 1) == 0 && __all_sync(kFullMask, ctr >= (unsigned)kN)) break;
#endif
      const uint64_t v = s[w];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const uint32_t t = (uint32_t)(v >> (4 * e)) & 0xF;  // low nibble of each byte first
        bool ok;
        int32_t val;
        if (P::ETA == 2) {
          ok = t < 15;
          val = 2 - (int32_t)(t - ((205 * t) >> 10) * 5);
        } else {
          ok = t < 9;
          val = 4 - (int32_t)t;
        }
        if (ok && ctr < (unsigned)kN) row[ctr++] = (int8_t)val;
      }
    }
    if (__all_sync(kFullMask, ctr >= (unsigned)kN)) break;
  }
  __syncwarp();
#pragma unroll 1
  for (int src = 0; src < 32; ++src) {
    if (p0 + src >= n_streams) break;
    const uint32_t* srow = reinterpret_cast<const uint32_t*>(stage[warp][src]);
    uint32_t* dst = reinterpret_cast<uint32_t*>(out8 + (size_t)(p0 + src) * kN);
    dst[lane] = srow[lane];
    dst[lane + 32] = srow[lane + 32];
  }
}

// ------------------------------------------------------------------ ExpandMask
// Streams: slot a (one rejection-loop attempt), column j in [0,L): SHAKE256(rho' ||
// le16(kappa_a + j)).  Emits the squeezed bytes themselves (32*Z_BITS per stream);
// consumers decode gamma1 - raw with the same bit reader as the signature's z field,
// which is exactly how the reference defines the mask (sampling.hpp:86-90).
// Works on one sponge already positioned by the caller; used by the sign kernel.
// NC = false: rho' is read with coherent loads -- the signing scheduler serves batches that
// were published after its kernel started, which the read-only (ld.global.nc) path must not touch.
template <class P, bool NC = true>
__device__ __forceinline__ void expand_mask_stream(const uint64_t* __restrict__ rho_prime,
                                                   unsigned nonce, uint8_t* __restrict__ dst) {
  constexpr int BYTES = 32 * P::Z_BITS;              // 576 / 640
  constexpr int FULL = BYTES / kRate256;             // 4 full blocks
  constexpr int TAILW = (BYTES % kRate256) / 8;      // 4 / 12 words
  uint64_t s[25];
  keccak_clear(s);
#pragma unroll
  for (int w = 0; w < 8; ++w) s[w] = NC ? __ldg(rho_prime + w) : ld_weak(rho_prime + w);
  s[8] = (uint64_t)(nonce & 0xFFFF) | ((uint64_t)0x1F << 16);
  s[16] = 0x8000000000000000ull;
  uint64_t* out = reinterpret_cast<uint64_t*>(dst);
#pragma unroll 1
  for (int blk = 0; blk <= FULL; ++blk) {  // one permutation call site
    keccak_f1600(s);
    if (blk < FULL) {
#pragma unroll
      for (int w = 0; w < kWords256; ++w) out[blk * kWords256 + w] = s[w];
    } else {
#pragma unroll
      for (int w = 0; w < TAILW; ++w) out[FULL * kWords256 + w] = s[w];
    }
  }
}

// ---------------------------------------------------------------- SampleInBall
// One challenge per thread.  c_tilde: 32 bytes (any alignment).  The Fisher-Yates walk
// needs a randomly indexed 256-entry array per stream: a padded int8 row in shared
// memory.  Squeezed bytes are consumed straight from the state registers (static
// indices; every lane walks all byte positions under predication).
template <int TAU, int CTW>
__device__ __forceinline__ void sample_in_ball_words(const uint64_t (&ct)[CTW],
                                                     int8_t* row /* smem, 256 entries */) {
  uint64_t s[25];
  keccak_clear(s);
#pragma unroll
  for (int w = 0; w < CTW; ++w) s[w] = ct[w];  // 32 bytes (round 3), lambda/4 bytes (FIPS 204)
  s[CTW] = 0x1F;
  s[16] = 0x8000000000000000ull;
  uint32_t* row32 = reinterpret_cast<uint32_t*>(row);
#pragma unroll
  for (int w = 0; w < 64; ++w) row32[w] = 0;
  // One permutation call site and a rolled walk over the squeezed words keep this
  // (once-per-attempt, inherently sequential) routine small in the instruction cache;
  // lanes leave the walk as soon as their tau positions are placed.
  uint64_t signs = 0;
  unsigned i = kN - TAU;
  int wstart = 1;  // bytes 0..7 of the first block are the sign bits
  while (true) {
    keccak_f1600(s);
    if (wstart) signs = s[0];
#pragma unroll 1
    for (int w = wstart; w < kWords256 && i < (unsigned)kN; ++w) {
      uint64_t v = s[0];
#pragma unroll
      for (int k = 1; k < kWords256; ++k) v = (w == k) ? s[k] : v;  // register select, no local mem
      // (the byte walk is only two-way unrolled: it runs ~60 times per challenge, and the signing
      // kernel gains more from the smaller code than it loses in loop overhead)
#pragma unroll 2
      for (int e = 0; e < 8; ++e) {
        const unsigned b = (unsigned)(v >> (8 * e)) & 0xFF;
        if (i < (unsigned)kN && b <= i) {
          row[i] = row[b];
          row[b] = (int8_t)(1 - 2 * (int)(signs & 1));
          signs >>= 1;
          ++i;
        }
      }
    }
    if (i >= (unsigned)kN) break;
    wstart = 0;
  }
}

template <int TAU, int CTW>
__device__ __forceinline__ void sample_in_ball_stream(const uint8_t* __restrict__ c_tilde,
                                                      int8_t* row) {
  uint64_t ct[CTW];
#pragma unroll
  for (int w = 0; w < CTW; ++w) ct[w] = load_u64_unaligned(c_tilde + 8 * w);
  sample_in_ball_words<TAU, CTW>(ct, row);
}

template <class P, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_sample_in_ball(const uint8_t* __restrict__ ct_base, size_t ct_stride, unsigned n,
                     int8_t* __restrict__ out8) {
  __shared__ __align__(16) int8_t stage[WARPS][32][kByteRowStride];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned p0 = (blockIdx.x * WARPS + warp) * 32;
  if (p0 >= n) return;
  const unsigned p = min(p0 + lane, n - 1);  // tail lanes redo the last stream (no divergence)
  sample_in_ball_stream<P::TAU, Hashing<P>::CTW>(ct_base + (size_t)p * ct_stride, stage[warp][lane]);
  __syncwarp();
#pragma unroll 1
  for (int src = 0; src < 32; ++src) {
    if (p0 + src >= n) break;
    const uint32_t* srow = reinterpret_cast<const uint32_t*>(stage[warp][src]);
    uint32_t* dst = reinterpret_cast<uint32_t*>(out8 + (size_t)(p0 + src) * kN);
    dst[lane] = srow[lane];
    dst[lane + 32] = srow[lane + 32];
  }
}

// ------------------------------------------------------------------ hash kernels

// keygen seed expansion: SHAKE256(zeta, 128) -> rho(32) | rho'(64) | K(32)
// (scheme.hpp:70-76).  zetas packed 32 bytes per task; out 128 bytes per task.
// `domain`: 0 for round 3; (k | l << 8) | 1 << 16 for FIPS 204, whose Alg. 6 hashes xi || k || l.
static __global__ void k_keygen_seed(const uint8_t* __restrict__ zetas, unsigned n,
                              uint64_t* __restrict__ out, unsigned domain) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint64_t s[25];
  keccak_clear(s);
#pragma unroll
  for (int w = 0; w < 4; ++w) s[w] = load_u64_unaligned(zetas + (size_t)t * 32 + 8 * w);
  s[4] = (domain >> 16) ? ((uint64_t)(domain & 0xFFFF) | ((uint64_t)0x1F << 16)) : 0x1F;
  s[16] = 0x8000000000000000ull;
  keccak_f1600(s);
#pragma unroll
  for (int w = 0; w < 16; ++w) out[(size_t)t * 16 + w] = s[w];
}

// tr = SHAKE256(pk, 32)  (scheme.hpp:102,287).  One thread per key.
// tr_words: 4 (32-byte tr, round 3) or 8 (64 bytes, FIPS 204).
static __global__ void k_hash_tr(const uint8_t* __restrict__ pk, size_t pk_stride, unsigned pk_bytes,
                          unsigned n, uint8_t* __restrict__ tr_out, size_t tr_stride,
                          int tr_words) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint64_t s[25];
  keccak_clear(s);
  {
    const uint8_t* msg = pk + (size_t)t * pk_stride;
    const size_t nblocks = pk_bytes / kRate256 + 1;
    // packed public keys are 32 + 320 k bytes: whole 64-bit words, and 8-byte aligned whenever the
    // array is -- then the absorb loop is plain word loads (no byte assembly, no length tests)
    const bool aligned = ((reinterpret_cast<uintptr_t>(msg) | pk_bytes) & 7) == 0;
    const unsigned nwords = pk_bytes / 8;
#pragma unroll 1
    for (size_t blk = 0; blk < nblocks; ++blk) {
      if (aligned) {
        const uint64_t* m64 = reinterpret_cast<const uint64_t*>(msg) + blk * kWords256;
        const unsigned left = nwords - (unsigned)(blk * kWords256);  // words from this block on
#pragma unroll
        for (int w = 0; w < kWords256; ++w)
          s[w] ^= (unsigned)w < left ? __ldg(m64 + w) : ((unsigned)w == left ? 0x1Full : 0ull);
      } else {
#pragma unroll
        for (int w = 0; w < kWords256; ++w)
          s[w] ^= padded_word(msg, pk_bytes, blk * kRate256 + 8 * w);
      }
      if (blk == nblocks - 1) s[kWords256 - 1] ^= 0x8000000000000000ull;
      keccak_f1600(s);
    }
  }
  uint64_t* o = reinterpret_cast<uint64_t*>(tr_out + (size_t)t * tr_stride);
#pragma unroll
  for (int w = 0; w < 8; ++w)
    if (w < tr_words) o[w] = s[w];
}

// mu = SHAKE256(tr || M, 64) and optionally rho' = SHAKE256(K || mu, 64)
// (scheme.hpp:240-248) of one task.  tr and K (32 B) of the task's key, 8-byte aligned.
// MLDSA (FIPS 204 Alg. 2 / 7, deterministic variant): tr is 64 bytes,
// mu = H(tr || 0 || |ctx| || ctx || M, 64) with the 2 + |ctx| prefix bytes at `pfx`
// (plen of them), and rho'' = H(K || 0^32 || mu, 64).  Round 3: pfx unused, plen = 0.
// NC = false reads every input with coherent loads (the signing scheduler hashes tasks of
// batches that were published after its kernel started).
template <bool MLDSA, bool NC>
__device__ __forceinline__ void hash_mu_task(const uint64_t* tr, const uint64_t* key,
                                             const uint8_t* pfx, unsigned plen, const uint8_t* msg,
                                             size_t msg_len, uint64_t* mu_out,
                                             uint64_t* rho_prime_out) {
  constexpr int TRW = MLDSA ? 8 : 4;
  uint64_t s[25];
  uint64_t pre[TRW];
#pragma unroll
  for (int w = 0; w < TRW; ++w) pre[w] = NC ? __ldg(tr + w) : ld_weak(tr + w);
  shake_absorb_pre<kWords256, TRW, NC>(s, pre, pfx, MLDSA ? plen : 0u, msg, msg_len);
  uint64_t mu[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    mu[w] = s[w];
    mu_out[w] = s[w];
  }
  if (rho_prime_out != nullptr) {
    keccak_clear(s);
#pragma unroll
    for (int w = 0; w < 4; ++w) s[w] = NC ? __ldg(key + w) : ld_weak(key + w);
    constexpr int MU0 = MLDSA ? 8 : 4;  // rnd = 0^32 sits between K and mu
#pragma unroll
    for (int w = 0; w < 8; ++w) s[MU0 + w] = mu[w];
    s[MU0 + 8] = 0x1F;
    s[16] ^= 0x8000000000000000ull;
    keccak_f1600(s);
#pragma unroll
    for (int w = 0; w < 8; ++w) rho_prime_out[w] = s[w];
  }
}

// One thread per task; task t uses key key_idx[t] (key_idx == nullptr: key t), strides 0 = one
// shared key.
template <bool MLDSA>
static __global__ void k_hash_mu(const uint8_t* __restrict__ tr_base, size_t tr_stride,
                          const uint8_t* __restrict__ key_base, size_t key_stride,
                          const uint32_t* __restrict__ key_idx,
                          const uint8_t* __restrict__ pfx, unsigned plen,
                          const uint8_t* __restrict__ msgs, const uint64_t* __restrict__ msg_off,
                          unsigned n, uint64_t* __restrict__ mu_out,
                          uint64_t* __restrict__ rho_prime_out) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const size_t kt = key_idx ? (size_t)__ldg(key_idx + t) : (size_t)t;
  const uint64_t m0 = msg_off[t], m1 = msg_off[t + 1];
  hash_mu_task<MLDSA, true>(reinterpret_cast<const uint64_t*>(tr_base + kt * tr_stride),
                            reinterpret_cast<const uint64_t*>(key_base + kt * key_stride), pfx, plen,
                            msgs + m0, (size_t)(m1 - m0), mu_out + (size_t)t * 8,
                            rho_prime_out ? rho_prime_out + (size_t)t * 8 : nullptr);
}

// c~ = SHAKE256(mu || w1_packed, 32)  (scheme.hpp:158-163,311-317) for one stream:
// mu 8 words (global, aligned), w1 W1_ALL bytes (global, 8-byte aligned).
template <int W1_ALL, bool NC = true, int CTW = 4>
__device__ __forceinline__ void hash_ctilde_stream(const uint64_t* __restrict__ mu,
                                                   const uint64_t* w1, uint64_t (&out)[CTW]) {
  static_assert(W1_ALL % 8 == 0, "w1 block is word aligned");
  constexpr int TOTALW = 8 + W1_ALL / 8;          // message words
  constexpr int NBLK = TOTALW / kWords256 + 1;    // incl. the padding block
  uint64_t s[25];
  keccak_clear(s);
#pragma unroll 1
  for (int blk = 0; blk < NBLK; ++blk) {
#pragma unroll
    for (int w = 0; w < kWords256; ++w) {
      const int idx = blk * kWords256 + w;  // message word index
      uint64_t v = 0;
      if (idx < 8) v = NC ? __ldg(mu + idx) : ld_weak(mu + idx);
      else if (idx < TOTALW) v = NC ? __ldg(w1 + (idx - 8)) : w1[idx - 8];
      else if (idx == TOTALW) v = 0x1F;
      s[w] ^= v;
    }
    if (blk == NBLK - 1) s[kWords256 - 1] ^= 0x8000000000000000ull;
    keccak_f1600(s);
  }
#pragma unroll
  for (int w = 0; w < CTW; ++w) out[w] = s[w];
}

}  // namespace dlb
