// sign.cu -- batched signing: per-key precomputation, message digests, and the
// persistent rejection-loop kernel with its device-side nonce scheduler.
//
// Reference semantics: scheme.hpp:106-125 (make_precomp), :133-219 (one attempt),
// :240-266 (mu, rho', the kappa loop); batch.hpp:53-137 (batch_sign);
// scheduler.hpp:44-186 (NonceScheduler: one next-nonce attempt per open task, then
// breadth-first speculation; smallest valid nonce wins once all smaller are resolved).
//
// GPU design.  One persistent kernel; every CTA owns SLOTS attempt slots and a small
// table of open tasks pulled from a global device work queue (atomic head counter).
// A CTA round runs all its slots through four stages, each with the thread mapping
// that suits it:
//   S1  ExpandMask         one sponge per thread, L passes      (sampling.hpp:83-92)
//   S2  w = A y, w1        one warp per slot                    (scheme.hpp:144-156)
//   S3  c~ = H(mu||w1), c  one sponge per thread                (scheme.hpp:158-165)
//   S4  z, r0, ct0, hints  one warp per slot, early abort       (scheme.hpp:167-215)
// then commits: per task the smallest valid attempt of the round wins (all smaller
// attempts of that task ran in this or earlier rounds and failed), its staged
// signature is copied out, rejected tasks stay in the CTA's table with their nonce
// advanced, and freed capacity is refilled from the global queue.  Slots left over
// when the queue runs dry run speculative future nonces of the CTA's open tasks,
// breadth first, exactly the reference's pass 2.  CTAs never wait on each other, so
// variable repetition counts cannot idle an SM while work remains.
#include <cstdlib>

#include "engine.cuh"
#include "samplers.cuh"
#include "verify_keygen.cuh"

#ifndef DLB_R0_MIN
#define DLB_R0_MIN 0
#endif
namespace dlb {

#ifndef DLB_SIGN_MINB
#define DLB_SIGN_MINB 4  // resident CTAs per SM: 5 (96 regs) was measured slower -- it squeezes L1 to ~10 KB
#endif
constexpr int kSignThreads = 128;          // threads = attempt slots per CTA
constexpr int kSignWarps = kSignThreads / 32;
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;
constexpr int kChunkBytes = 1024;  // cp.async landing buffer: one packed polynomial

// ---- per-key precomputation -----------------------------------------------------------
// One warp per (key, polynomial): s1 (L), s2 (K), t0 (K) unpacked from the secret key,
// range-checked (packing.hpp:79-86), transformed; stored reduced, natural order.
template <class P, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_sign_unpack(unsigned n_keys, const uint8_t* __restrict__ sks, size_t sk_stride,
                  int32_t* __restrict__ shat, unsigned* __restrict__ key_bad) {
  using S = Sizes<P>;
  constexpr int PV = P::L + 2 * P::K;
  __shared__ __align__(16) int2 zs[256], nzs[256];
  __shared__ __align__(16) int32_t tiles[WARPS][kTileWords];
  load_twiddles(zs, nzs);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned id = blockIdx.x * WARPS + warp;
  if (id >= n_keys * PV) return;
  const unsigned key = id / PV, p = id % PV;
  const uint8_t* sk = sks + (size_t)key * sk_stride;
  int32_t r[8];
  bool bad = false;
  if (p < (unsigned)(P::L + P::K)) {
    const uint8_t* src = sk + S::SK_S1 + p * S::ETA_POLY;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t raw = load_bits(src, (lane + 32 * e) * P::ETA_BITS, P::ETA_BITS);
      bad = bad || raw > 2u * P::ETA;
      r[e] = P::ETA - (int32_t)raw;
    }
  } else {
    const uint8_t* src = sk + S::SK_T0 + (p - P::L - P::K) * S::T0_POLY;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      r[e] = 4096 - (int32_t)load_bits(src, (lane + 32 * e) * 13, 13);
  }
  ntt_fwd(r, tiles[warp], zs, lane);
  int4* dst = reinterpret_cast<int4*>(shat + (size_t)id * kN) + 2 * lane;
  dst[0] = make_int4(reduce32(r[0]), reduce32(r[1]), reduce32(r[2]), reduce32(r[3]));
  dst[1] = make_int4(reduce32(r[4]), reduce32(r[5]), reduce32(r[6]), reduce32(r[7]));
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(key_bad, 1u);
}

// ---- device-side scheduler state -----------------------------------------------------

struct SignQueue {
  unsigned head;          // next unclaimed task of the batch (the device work queue)
  unsigned key_bad;       // some secret key failed the eta range check
  unsigned long long rounds, attempts, speculative, idle_slots, accepted_sum, failed;
  unsigned long long t_first_start, t_last_start, t_first_exit, t_last_exit;  // %globaltimer, ns
  unsigned long long trace_count;  // per-round trace records produced (may exceed the capacity)
};

struct SignArgs {
  unsigned n;                 // tasks
  unsigned tcap;              // max open tasks per CTA (<= slots)
  unsigned slots;             // attempt slots a CTA uses (<= 128): small batches are spread
                              // over more CTAs with fewer slots each to cut round latency
  unsigned max_attempt;       // (65535 - (L-1)) / L   (scheduler.hpp:52)
  int speculate;
  unsigned spec_depth;        // deepest speculative attempt per task and round (pass-2 cap)
  int single_round;           // stage-test mode: exactly one round, then fail open tasks
  const uint64_t* mu;         // n * 8
  const uint64_t* rho_prime;  // n * 8
  const uint32_t* kappa0;     // nullable: first nonce per task (stage tests)
  const int32_t* A;           // keys * K*L*256
  const int32_t* shat;        // keys * (L+2K)*256
  unsigned key_stride;        // 0 shared key, 1 per-task keys (when key_idx == nullptr)
  const uint32_t* key_idx;    // nullable: key table index of each task
  uint32_t* trace;            // nullable: per-round records of 8 words (dlb_round_trace)
  unsigned trace_cap;
  // per-CTA scratch in HBM/L2, indexed [cta][slot]
  uint8_t* ybytes;
  int32_t* wbuf;
  uint8_t* w1buf;
  uint64_t* ctbuf;
  int8_t* c8buf;
  uint8_t* staging;
  // outputs
  uint8_t* sigs;
  uint32_t* attempts_out;     // nullable
  uint8_t* failed_out;        // nullable
  uint8_t* dbg_ctilde;        // nullable: n*32, c~ of each task's first executed attempt
  SignQueue* q;
};

template <class P>
struct SignSizes {
  using S = Sizes<P>;
  static constexpr int Y_SLOT = P::L * S::Z_POLY;           // bytes
  static constexpr int W_SLOT = P::K * kN;                  // int32
  static constexpr int SIG_PAD = (S::SIG + 15) / 16 * 16;   // staging stride
};

// per-warp scratch of the signing stages; bit-packing borrows a free cp.async ring buffer
template <class P>
struct SignWarpScratch {
  int32_t tile[kTileWords];
  int32_t vhat[P::L][8][32];
  uint32_t hbits[P::K][8];
};

constexpr int kHeadBytes = 256;  // the challenge c as int8
constexpr int kPreBytes = 2 * kHeadBytes + 2 * kChunkBytes;

template <class P>
struct SignSmem {
  int2 zs[256], nzs[256];
  union {
    struct {
      SignWarpScratch<P> ws[kSignWarps];
      uint8_t pre[kSignWarps][kPreBytes];  // cp.async landing buffers: head x2, ring x2
    } a;
    int8_t rows[kSignThreads][kByteRowStride];
  } u;
  uint32_t utask[kSignThreads];    // open tasks of this CTA (compact)
  uint32_t unext[kSignThreads];    // their next unresolved attempt ordinal
  uint32_t slot_task[kSignThreads];     // global task id or kNoSlot
  uint32_t slot_attempt[kSignThreads];
  uint8_t slot_valid[kSignThreads];
  int32_t winner[kSignThreads];    // per open task: winning slot, -1 none, -2 failed
  uint32_t warp_sums[kSignWarps];
  unsigned U, newU, got, base;
  unsigned cursor2, cursor4;  // next unclaimed slot of stages S2 / S4 (warps pull slots)
  unsigned r_on, r_spec;      // this round's assigned / speculative slots (trace)
  unsigned long long st_rounds, st_attempts, st_spec, st_idle;  // per-CTA counters
};

// ---- asynchronous scratch prefetch ----------------------------------------------------
// The per-slot scratch (masks y, w) of all resident CTAs is far larger than L2, so the
// warp-per-slot stages would eat one DRAM latency per polynomial.  Each warp therefore
// streams its inputs through small shared-memory buffers with cp.async, one chunk
// (= one packed polynomial, <= 1 KiB) ahead of the arithmetic: `head` holds c | y_0 of
// a slot (fetched while the previous slot is processed), `ring` the remaining chunks.

struct SlotPipe {
  uint8_t* base;  // kPreBytes of shared memory: head 0, head 1, ring 0, ring 1
  unsigned k;     // ring chunks issued so far (buffer = k & 1), warp-uniform
  __device__ __forceinline__ uint8_t* head(int par) const { return base + (par & 1) * kHeadBytes; }
  __device__ __forceinline__ uint8_t* ring(unsigned i) const {
    return base + 2 * kHeadBytes + (i & 1) * kChunkBytes;
  }
};

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// one warp copies `bytes` (multiple of 16, 16-byte aligned) global -> shared, no commit
template <unsigned BYTES>
__device__ __forceinline__ void warp_fetch(uint8_t* sdst, const void* gsrc, int lane) {
  static_assert(BYTES % 16 == 0, "whole 16-byte pieces");
  const uint8_t* g = static_cast<const uint8_t*>(gsrc);
#pragma unroll
  for (unsigned it = 0; it < (BYTES + 511) / 512; ++it) {  // compile-time trip count, last one predicated
    const unsigned o = it * 512u + lane * 16u;
    if ((it + 1) * 512u <= BYTES || o < BYTES) cp_async16(sdst + o, g + o);
  }
}

// Raw BITS-wide fields of coefficients lane, lane + 32, ..., lane + 224 of a packed
// polynomial in a 4-byte aligned shared-memory buffer.  32 * BITS is a multiple of 32, so
// the eight fields of a lane share one shift and sit BITS words apart: two loads, one
// funnel shift and one mask per coefficient, all offsets immediate.  (Reads one word past
// the last field: buffers are kChunkBytes long, fields end well before.)
template <int BITS>
__device__ __forceinline__ void unpack_strided(const uint8_t* sbase, int lane, uint32_t (&raw)[8]) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(sbase) + ((lane * BITS) >> 5);
  const unsigned sh = (unsigned)(lane * BITS) & 31u;
#pragma unroll
  for (int e = 0; e < 8; ++e)
    raw[e] = __funnelshift_r(w[BITS * e], w[BITS * e + 1], sh) & ((1u << BITS) - 1);
}

// S2: w = INTT(A * NTT(y)), w1 = HighBits(w) packed (scheme.hpp:141-156).
// Precondition: ring chunk y_0 of this slot already issued; `next_y` = y bytes of the
// warp's next active slot (nullptr if none): its y_0 is issued during the last polynomial.
template <class P>
__device__ __forceinline__ void stage_w(SignWarpScratch<P>& ws, SlotPipe& pp, const int2* zs,
                                        const int2* nzs, int lane, const uint8_t* ybytes,
                                        const uint8_t* next_y, const int32_t* A, int32_t* wout,
                                        uint8_t* w1out) {
  using S = Sizes<P>;
  int32_t r[8];
#pragma unroll 1
  for (int j = 0; j < P::L; ++j) {
    const uint8_t* cur = pp.ring(pp.k - 1);  // chunk y_j
    if (j + 1 < P::L) warp_fetch<S::Z_POLY>(pp.ring(pp.k), ybytes + (j + 1) * S::Z_POLY, lane);
    else if (next_y) warp_fetch<S::Z_POLY>(pp.ring(pp.k), next_y, lane);
    cp_async_commit();
    ++pp.k;
    cp_async_wait<1>();
    __syncwarp();
    {
      uint32_t raw[8];
      unpack_strided<P::Z_BITS>(cur, lane, raw);
#pragma unroll
      for (int e = 0; e < 8; ++e) r[e] = P::GAMMA1 - (int32_t)raw[e];
    }
    ntt_fwd(r, ws.tile, zs, lane);
#pragma unroll
    for (int m = 0; m < 8; ++m) ws.vhat[j][m][lane] = r[m];
  }
#pragma unroll 1
  for (int i = 0; i < P::K; ++i) {
    int64_t acc64[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) acc64[m] = 0;
    // (No software prefetch of the next matrix polynomial: the register copies it needs cost
    // more issue slots than the L1-resident loads' latency, measured +2 %.)
    const int4* ap = reinterpret_cast<const int4*>(A + (size_t)(i * P::L) * kN) + 2 * lane;
#pragma unroll 1
    for (int j = 0; j < P::L; ++j) {
      const int4 a0 = __ldg(ap + j * (kN / 4)), a1 = __ldg(ap + j * (kN / 4) + 1);
      const int32_t a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int m = 0; m < 8; ++m) acc64[m] = mac_wide(acc64[m], a[m], ws.vhat[j][m][lane]);
    }
    int32_t acc[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) acc[m] = mont_reduce64(acc64[m]);  // |.| < q: ready for the INTT
    ntt_inv(acc, ws.tile, nzs, lane);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int32_t w = caddq(acc[e]);
      wout[i * kN + lane + 32 * e] = w;
      ws.tile[lane + 36 * e] = highbits<P::GAMMA2>(w);
    }
    __syncwarp();
    // packing scratch = the ring buffer whose chunk was consumed last (nothing in flight there)
    pack_tile<P::W1_BITS>(ws.tile, pp.ring(pp.k), w1out + i * S::W1_POLY, lane);
  }
}

// c * shat_p -> INTT, result at coefficient lane + 32 e, in (-q, q)
__device__ __forceinline__ void mul_challenge(int32_t (&out)[8], const int32_t (&ch)[8],
                                              const int32_t* shat_poly, int32_t* tile,
                                              const int2* nzs, int lane) {
  const int4* sp = reinterpret_cast<const int4*>(shat_poly) + 2 * lane;
  const int4 s0 = __ldg(sp), s1 = __ldg(sp + 1);
  const int32_t s[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
  for (int m = 0; m < 8; ++m) out[m] = mont_mul(ch[m], s[m]);
  ntt_inv(out, tile, nzs, lane);
}

// issue the head chunk (the challenge c, 256 bytes) of a slot into pp.head(par); caller commits
__device__ __forceinline__ void fetch_head(SlotPipe& pp, int par, const int8_t* c8, int lane) {
  warp_fetch<kN>(pp.head(par), c8, lane);
}

// S4: everything after the challenge (scheme.hpp:165-215) + signature packing into the
// slot's staging buffer (packing.hpp:236-254).  Warp-uniform return: accepted?
//
// The reference checks z, then r0, then ct0 / hints (scheme.hpp:167-215); accept/reject
// does not depend on the order, so the checks run in the order that
// rejects soonest per transform spent: the K rows of r0 = LowBits(w - c s2) first (each
// fails with the highest probability), then the L rows of z, and only survivors of both
// pay for c t0 and the hints.  w - c s2 overwrites w in the slot's scratch row so the hint
// phase can pick it up again.
//
// Precondition: head[par] (c) of this slot issued (possibly still in flight).  next_c8 is
// the challenge of the warp's next active slot (nullptr if none); it goes to head[par ^ 1].
template <class P>
__device__ __forceinline__ bool stage_finish(SignWarpScratch<P>& ws, SlotPipe& pp, int par,
                                             const int2* zs, const int2* nzs, int lane,
                                             const uint8_t* ybytes, int32_t* wrows,
                                             const int8_t* next_c8, const uint64_t* ct,
                                             const int32_t* shat, uint8_t* stage_sig) {
  using S = Sizes<P>;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int R = P::K + P::L;  // ring chunks of a slot: w_0..w_{K-1}, y_0..y_{L-1}
  auto ring_fetch = [&](int r) {  // chunk r -> the ring buffer next in line
    if (r < P::K) warp_fetch<kN * 4>(pp.ring(pp.k), wrows + (size_t)r * kN, lane);
    else warp_fetch<S::Z_POLY>(pp.ring(pp.k), ybytes + (r - P::K) * S::Z_POLY, lane);
  };

  // ring chunk 0, then the next slot's head; then wait for everything older (our head).
  // (The buffer it lands in was read by the whole warp while finishing the previous slot;
  // that slot ended on a warp vote -- the explicit barrier states the ordering.)
  __syncwarp();
  ring_fetch(0);
  cp_async_commit();
  ++pp.k;
  if (next_c8) fetch_head(pp, par ^ 1, next_c8, lane);
  cp_async_commit();
  cp_async_wait<2>();
  __syncwarp();

  int32_t ch[8], t[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) ch[e] = reinterpret_cast<const int8_t*>(pp.head(par))[lane + 32 * e];
  ntt_fwd(ch, ws.tile, zs, lane);

  // One loop over the K + L + K products c*s2_i, c*s1_j, c*t0_i: a single inverse-NTT
  // instance in the instruction stream (the kernel is sensitive to code size: every extra
  // copy of a transform costs instruction-cache misses in all stages).  Iterations p < R
  // consume ring chunk p; the t0 rows read w - c s2 back from the slot's scratch.  Every
  // exit is warp-uniform.
  //   r0 = LowBits(w - c s2), ||r0|| < gamma2 - beta            (scheme.hpp:177-190)
  //   z = y + c s1, ||z|| < gamma1 - beta                      (scheme.hpp:167-174)
  //   ||c t0|| < gamma2, h = [HB(w - c s2 + c t0) != HB(w - c s2)]   (scheme.hpp:192-215)
  unsigned weight = 0;
#pragma unroll 1
  for (int p = 0; p < R + P::K; ++p) {
    // shat order: s1 (L), s2 (K), t0 (K); visiting order: s2 rows, s1 rows, t0 rows
    const int poly = p < P::K ? P::L + p : (p < R ? p - P::K : p - R + P::L + P::K);
    int32_t wcs2[8];
    if (p >= R) {  // issue the read-back before the transform hides its latency
#pragma unroll
      for (int e = 0; e < 8; ++e) wcs2[e] = wrows[(size_t)(p - R) * kN + lane + 32 * e];
    }
    mul_challenge(t, ch, shat + (size_t)poly * kN, ws.tile, nzs, lane);
    const uint8_t* cur = pp.ring(pp.k - 1);
    if (p < R) {  // consume the oldest ring chunk; keep one more in flight behind it
      if (p + 1 < R) ring_fetch(p + 1);
      cp_async_commit();
      ++pp.k;
      cp_async_wait<1>();
      __syncwarp();
    }
    // The exact product c*s1 has coefficients in [-beta, beta] (tau non-zero challenge
    // entries times eta) and c*t0 in (-2^22, 2^22), so the inverse NTT's output in (-q, q) is
    // that small value or the same +-q: reduce32 returns the centred value itself.
    bool bad = false;
    if (p < P::K) {
      const int32_t* wrow = reinterpret_cast<const int32_t*>(cur);
      int32_t* wdst = wrows + (size_t)p * kN;
#if DLB_R0_MIN
      uint32_t worst = 0;
#endif
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int32_t d = freeze_near(wrow[lane + 32 * e] - t[e]);  // [0, q) - (-q, q)
#if DLB_R0_MIN
        // |r0| < B without materialising the centred r0: a0 = d - r1 * 2 gamma2 is r0 or, when
        // HighBits wrapped to 0, r0 + q; shifted by B - 1 the valid one lands in [0, 2B - 1)
        constexpr int32_t B = P::GAMMA2 - P::BETA;
        const int32_t a0 = d - highbits<P::GAMMA2>(d) * 2 * P::GAMMA2;
        const uint32_t u = (uint32_t)(a0 + B - 1);
        worst = max(worst, min(u, u - (uint32_t)kQ));
#else
        int32_t r0;
        decompose<P::GAMMA2>(d, r0);
        bad = bad || abs(r0) >= P::GAMMA2 - P::BETA;
#endif
        wdst[lane + 32 * e] = d;  // read back by this same lane in the hint phase
      }
#if DLB_R0_MIN
      bad = worst >= 2u * (P::GAMMA2 - P::BETA) - 1u;
#endif
    } else if (p < R) {
      uint32_t raw[8];
      unpack_strided<P::Z_BITS>(cur, lane, raw);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int32_t y = P::GAMMA1 - (int32_t)raw[e];
        const int32_t z = y + reduce32(t[e]);  // |y| <= gamma1, |c s1| <= beta: no wrap, centred
        bad = bad || abs(z) >= P::GAMMA1 - P::BETA;
        ws.vhat[p - P::K][e][lane] = z;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int32_t vt = reduce32(t[e]);  // |c t0| <= tau * 2^12 < 2^22: already centred
        bad = bad || abs(vt) >= P::GAMMA2;
        const int h = highbits<P::GAMMA2>(freeze_near(wcs2[e] + vt)) != highbits<P::GAMMA2>(wcs2[e]);
        const unsigned mask = __ballot_sync(FULL, h);
        if (lane == 0) ws.hbits[p - R][e] = mask;
        weight += __popc(mask);
      }
    }
    if (__any_sync(FULL, bad)) return false;
  }
  if (weight > (unsigned)P::OMEGA) return false;

  // accepted: c~ | z | hints into the staging slot
  if (lane < 2 * Hashing<P>::CTW) reinterpret_cast<uint32_t*>(stage_sig)[lane] =
      reinterpret_cast<const uint32_t*>(ct)[lane];
#pragma unroll 1
  for (int j = 0; j < P::L; ++j) {
#pragma unroll
    for (int e = 0; e < 8; ++e) ws.tile[lane + 36 * e] = P::GAMMA1 - ws.vhat[j][e][lane];
    __syncwarp();
    pack_tile<P::Z_BITS>(ws.tile, pp.ring(pp.k), stage_sig + S::SIG_Z + j * S::Z_POLY, lane);
  }
  uint8_t* hint = stage_sig + S::SIG_Z + P::L * S::Z_POLY;
  // (the padding behind the signature is cleared too: the word-wise commit copy reads it)
  for (int b = lane; b < S::HINT + (SignSizes<P>::SIG_PAD - S::SIG); b += 32) hint[b] = 0;
  __syncwarp();
  unsigned count = 0;
#pragma unroll 1
  for (int i = 0; i < P::K; ++i) {
#pragma unroll 1
    for (int e = 0; e < 8; ++e) {
      const unsigned mask = ws.hbits[i][e];
      if ((mask >> lane) & 1) hint[count + __popc(mask & ((1u << lane) - 1))] = (uint8_t)(32 * e + lane);
      count += __popc(mask);
    }
    if (lane == 0) hint[P::OMEGA + i] = (uint8_t)count;
  }
  return true;
}

template <class P>
__global__ void __launch_bounds__(kSignThreads, (P::LEVEL == 2 || P::LEVEL == 44) ? DLB_SIGN_MINB : 4)
    k_sign_persistent(SignArgs a) {
  using S = Sizes<P>;
  using Z = SignSizes<P>;
  extern __shared__ __align__(16) unsigned char sign_smem_raw[];  // dynamic: > 48 KB at levels 3/5
  SignSmem<P>& sm = *reinterpret_cast<SignSmem<P>*>(sign_smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t cta = blockIdx.x;
  uint8_t* ybytes = a.ybytes + cta * kSignThreads * Z::Y_SLOT;
  int32_t* wbuf = a.wbuf + cta * kSignThreads * Z::W_SLOT;
  uint8_t* w1buf = a.w1buf + cta * kSignThreads * S::W1_ALL;
  constexpr int CTW = Hashing<P>::CTW;  // 64-bit words of the commitment hash c~
  uint64_t* ctbuf = a.ctbuf + cta * kSignThreads * CTW;
  int8_t* c8buf = a.c8buf + cta * kSignThreads * kN;
  uint8_t* staging = a.staging + cta * kSignThreads * Z::SIG_PAD;

  load_twiddles(sm.zs, sm.nzs);
  if (tid == 0) {
    sm.U = 0;
    sm.st_rounds = sm.st_attempts = sm.st_spec = sm.st_idle = 0;
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    atomicMin(&a.q->t_first_start, now);
    atomicMax(&a.q->t_last_start, now);
  }
  __syncthreads();

  while (true) {
    // ---- refill from the device work queue -----------------------------------------
    if (tid == 0) {
      const unsigned U = sm.U;
      unsigned got = 0, base = 0;
      if (U < a.tcap && !(a.single_round && sm.st_rounds > 0)) {
        const unsigned want = a.tcap - U;
        if (*(volatile unsigned*)&a.q->head < a.n) {
          base = atomicAdd(&a.q->head, want);
          if (base < a.n) got = min(want, a.n - base);
        }
      }
      sm.got = got;
      sm.base = base;
    }
    __syncthreads();
    {
      const unsigned U = sm.U, got = sm.got;
      if ((unsigned)tid < got) {
        sm.utask[U + tid] = sm.base + tid;
        sm.unext[U + tid] = 0;
      }
      __syncthreads();
      if (tid == 0) sm.U = U + got;
      __syncthreads();
    }
    const unsigned U = sm.U;
    if (U == 0) break;

    // ---- schedule: slot s -> open task s % U, depth s / U (scheduler.hpp:58-92) ------
    {
      const unsigned u = tid % U, depth = tid / U;
      const unsigned att = sm.unext[u] + depth;
      const bool on = (unsigned)tid < a.slots && (depth == 0 || (a.speculate && depth <= a.spec_depth)) &&
                      att <= a.max_attempt;
      sm.slot_task[tid] = on ? sm.utask[u] : kNoSlot;
      sm.slot_attempt[tid] = att;
      sm.slot_valid[tid] = 0;
      if (tid == 0) sm.cursor2 = sm.cursor4 = 0;
      const unsigned n_on = __syncthreads_count(on);
      const unsigned n_spec = __syncthreads_count(on && depth > 0);
      if (tid == 0) {
        sm.st_rounds += 1;
        sm.st_attempts += n_on;
        sm.st_spec += n_spec;
        sm.st_idle += a.slots - n_on;
        sm.r_on = n_on;
        sm.r_spec = n_spec;
      }
    }
    const unsigned my_task = sm.slot_task[tid];

    // ---- S1: masks ---------------------------------------------------------------
    // One sponge per (slot, polynomial): the L mask polynomials of an attempt are independent
    // streams (nonces kappa .. kappa + L - 1), so when a round runs fewer slots than the CTA
    // has threads -- small batches, the tail of a large one -- they spread over the idle
    // threads and the round's longest sequential Keccak chain shrinks from 5 L permutations
    // towards 5.  Active slots are a prefix [0, span); items are laid out polynomial-major so
    // the lanes of a warp share j.  With all 128 slots active this is thread t -> slot t,
    // j = 0 .. L-1, as before.
    {
      const unsigned cap = a.speculate ? a.spec_depth + 1u : 1u;
      const unsigned span = min(a.slots, U * cap);
#pragma unroll 1
      for (unsigned item = tid; item < span * P::L; item += kSignThreads) {
        const unsigned slot = item % span, j = item / span;
        const unsigned task = sm.slot_task[slot];
        if (task == kNoSlot) continue;
        const unsigned k0 = a.kappa0 ? a.kappa0[task] : 0u;
        const unsigned kappa = k0 + sm.slot_attempt[slot] * P::L;
        expand_mask_stream<P>(a.rho_prime + (size_t)task * 8, kappa + j,
                              ybytes + (size_t)slot * Z::Y_SLOT + j * S::Z_POLY);
      }
    }
    __syncthreads();

    // ---- S2: w, w1 ---------------------------------------------------------------
    SlotPipe pp;
    pp.base = &sm.u.a.pre[warp][0];
    pp.k = 0;
    // Warps pull slots from a CTA-wide cursor instead of owning a fixed stripe: S4's work
    // per slot varies with the early aborts, and a static split leaves warps waiting at
    // the stage barrier.  Returns kSignThreads when the stage has no slot left.
    auto grab = [&](unsigned* cursor) {
      unsigned s = kSignThreads;
      if (lane == 0) {
        do s = atomicAdd(cursor, 1u);
        while (s < (unsigned)kSignThreads && sm.slot_task[s] == kNoSlot);
        if (s > (unsigned)kSignThreads) s = kSignThreads;
      }
      return (int)__shfl_sync(0xffffffffu, s, 0);
    };
    {
      int s = grab(&sm.cursor2);
      if (s < kSignThreads) {  // prologue: first mask polynomial of the first slot
        warp_fetch<S::Z_POLY>(pp.ring(pp.k), ybytes + (size_t)s * Z::Y_SLOT, lane);
        cp_async_commit();
        ++pp.k;
      }
#pragma unroll 1
      while (s < kSignThreads) {
        const int nx = grab(&sm.cursor2);
        const size_t key = a.key_idx ? (size_t)__ldg(a.key_idx + sm.slot_task[s])
                                     : (size_t)sm.slot_task[s] * a.key_stride;
        stage_w<P>(sm.u.a.ws[warp], pp, sm.zs, sm.nzs, lane, ybytes + (size_t)s * Z::Y_SLOT,
                   nx < kSignThreads ? ybytes + (size_t)nx * Z::Y_SLOT : nullptr,
                   a.A + key * (P::K * P::L * kN), wbuf + (size_t)s * Z::W_SLOT,
                   w1buf + (size_t)s * S::W1_ALL);
        s = nx;
      }
      cp_async_wait<0>();
    }
    __syncthreads();

    // ---- S3: challenge -----------------------------------------------------------
    {
      if (my_task != kNoSlot) {
        uint64_t ct[CTW];
        hash_ctilde_stream<S::W1_ALL, false, CTW>(
            a.mu + (size_t)my_task * 8,
            reinterpret_cast<const uint64_t*>(w1buf + (size_t)tid * S::W1_ALL), ct);
#pragma unroll
        for (int w = 0; w < CTW; ++w) ctbuf[tid * CTW + w] = ct[w];
        sample_in_ball_words<P::TAU, CTW>(ct, sm.u.rows[tid]);
      }
      __syncwarp();
#pragma unroll 1
      for (int src = 0; src < 32; ++src) {
        const int s = warp * 32 + src;
        if (sm.slot_task[s] == kNoSlot) continue;
        const uint32_t* srow = reinterpret_cast<const uint32_t*>(sm.u.rows[s]);
        uint32_t* dst = reinterpret_cast<uint32_t*>(c8buf + (size_t)s * kN);
        dst[lane] = srow[lane];
        dst[lane + 32] = srow[lane + 32];
      }
    }
    __syncthreads();

    // ---- S4: finish --------------------------------------------------------------
    {
      int s = grab(&sm.cursor4);
      int par = 0;
      if (s < kSignThreads) {  // prologue: head chunk (c) of the first slot
        fetch_head(pp, par, c8buf + (size_t)s * kN, lane);
        cp_async_commit();
      }
#pragma unroll 1
      while (s < kSignThreads) {
        const int nx = grab(&sm.cursor4);
        const size_t key = a.key_idx ? (size_t)__ldg(a.key_idx + sm.slot_task[s])
                                     : (size_t)sm.slot_task[s] * a.key_stride;
        const bool ok = stage_finish<P>(
            sm.u.a.ws[warp], pp, par, sm.zs, sm.nzs, lane, ybytes + (size_t)s * Z::Y_SLOT,
            wbuf + (size_t)s * Z::W_SLOT, nx < kSignThreads ? c8buf + (size_t)nx * kN : nullptr,
            ctbuf + s * CTW, a.shat + key * ((P::L + 2 * P::K) * kN),
            staging + (size_t)s * Z::SIG_PAD);
        if (lane == 0) sm.slot_valid[s] = ok ? 1 : 0;
        s = nx;
        par ^= 1;
      }
      cp_async_wait<0>();
    }
    __syncthreads();

    // ---- commit: smallest valid attempt per task wins (scheduler.hpp:97-136) --------
    bool keep = false;
    unsigned my_u_task = 0, my_u_next = 0;
    if ((unsigned)tid < U) {
      const unsigned task = sm.utask[tid];
      unsigned next = sm.unext[tid];
      int win = -1;
      unsigned ran = 0;
      for (unsigned s = tid; s < a.slots; s += U) {
        if (sm.slot_task[s] == kNoSlot) break;
        ++ran;
        if (sm.slot_valid[s]) {
          win = (int)s;
          break;
        }
      }
      if (a.dbg_ctilde) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(ctbuf + tid * CTW);
        uint32_t* dst = reinterpret_cast<uint32_t*>(a.dbg_ctilde + (size_t)task * Hashing<P>::CT);
        for (int w = 0; w < 2 * CTW; ++w) dst[w] = src[w];
      }
      if (win >= 0) {
        const unsigned ordinal = sm.slot_attempt[win] + 1;
        if (a.attempts_out) a.attempts_out[task] = ordinal;
        if (a.failed_out) a.failed_out[task] = 0;
        atomicAdd(&a.q->accepted_sum, (unsigned long long)ordinal);
      } else {
        next += ran;
        if (next > a.max_attempt || a.single_round) {
          win = -2;  // nonce space exhausted (scheduler.hpp:122-128)
          if (a.attempts_out) a.attempts_out[task] = 0;
          if (a.failed_out) a.failed_out[task] = 1;
          atomicAdd(&a.q->failed, 1ull);
        }
      }
      sm.winner[tid] = win;
      keep = win == -1;
      my_u_task = task;
      my_u_next = next;
    }
    // compact the open-task table
    {
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) sm.warp_sums[warp] = __popc(bal);
      __syncthreads();
      unsigned off = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kSignWarps; ++w) {
        if (w < warp) off += sm.warp_sums[w];
        total += sm.warp_sums[w];
      }
      const unsigned pos = off + __popc(bal & ((1u << lane) - 1));
      // copy winners' staged signatures out before the table is overwritten
#pragma unroll 1
      for (unsigned u = warp; u < U; u += kSignWarps) {
        const int win = sm.winner[u];
        if (win < 0) continue;
        const uint8_t* src = staging + (size_t)win * Z::SIG_PAD;
        uint8_t* dst = a.sigs + (size_t)sm.utask[u] * S::SIG;
        // word-granular, coalesced copy to a destination of any alignment (sig_bytes is
        // odd at levels 3/5): the destination may be pinned host memory, where 128-byte
        // write bursts matter
        const unsigned head = (4u - (unsigned)(reinterpret_cast<uintptr_t>(dst) & 3)) & 3u;
        if (lane < (int)head) dst[lane] = src[lane];
        const unsigned nwords = (S::SIG - head) / 4;
        uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + head);
        const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);  // staging is 16-byte aligned
        for (unsigned w = lane; w < nwords; w += 32)
          d32[w] = head ? __funnelshift_r(s32[w], s32[w + 1], 8 * head) : s32[w];
        const unsigned done = head + 4 * nwords;
        if (lane < (int)(S::SIG - done)) dst[done + lane] = src[done + lane];
      }
      __syncthreads();
      if (keep) {
        sm.utask[pos] = my_u_task;
        sm.unext[pos] = my_u_next;
      }
      if (tid == 0) {
        if (a.trace) {  // RoundTrace of this CTA's round (scheduler.hpp:21-28)
          const unsigned long long idx = atomicAdd(&a.q->trace_count, 1ull);
          if (idx < a.trace_cap) {
            uint4* rec = reinterpret_cast<uint4*>(a.trace + idx * 8);
            rec[0] = make_uint4(blockIdx.x, (unsigned)sm.st_rounds - 1u, U, sm.r_on);
            rec[1] = make_uint4(sm.r_spec, a.slots - sm.r_on, U - total, 0u);
          }
        }
        sm.U = total;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    atomicMin(&a.q->t_first_exit, now);
    atomicMax(&a.q->t_last_exit, now);
    atomicAdd(&a.q->rounds, sm.st_rounds);
    atomicAdd(&a.q->attempts, sm.st_attempts);
    atomicAdd(&a.q->speculative, sm.st_spec);
    atomicAdd(&a.q->idle_slots, sm.st_idle);
  }
}

// ---- host side ---------------------------------------------------------------------

template <class P>
static int sign_core(dlb_ctx* c, size_t n, const uint8_t* d_sks, size_t sk_stride, size_t n_keys,
                     const uint32_t* d_key_idx, const uint8_t* d_msgs, const uint64_t* d_msg_off, const uint64_t* d_mu_in,
                     const uint8_t* d_rho_prime, const uint32_t* d_kappa0, size_t psi,
                     int speculate, int single_round, uint8_t* d_sigs, uint32_t* d_attempts,
                     uint8_t* d_failed, uint8_t* d_dbg_ct, dlb_sign_stats* stats) {
  using S = Sizes<P>;
  using Z = SignSizes<P>;
  constexpr int KL = P::K * P::L, PV = P::L + 2 * P::K;
  if (n == 0) return 0;
  if (n > 0x7fffffffu) return DLB_E_ARG;
  cudaStream_t st = c->s();
  if (d_key_idx && (n_keys == 0 || sk_stride == 0)) return DLB_E_ARG;
  // distinct keys to precompute: the key table, one key per task, or one shared key
  const size_t nk = d_key_idx ? n_keys : (sk_stride ? n : 1);

  int32_t *A, *shat;
  uint64_t *mu, *rp;
  SignQueue* q;
  DLB_TRY(dalloc(c, "s.A", nk * KL * kN, &A));
  DLB_TRY(dalloc(c, "s.shat", nk * PV * kN, &shat));
  DLB_TRY(dalloc(c, "s.mu", n * 8, &mu));
  DLB_TRY(dalloc(c, "s.rp", n * 8, &rp));
  DLB_TRY(dalloc(c, "s.q", 1, &q));
  DLB_CUDA_CHECK(cudaMemsetAsync(q, 0, sizeof(SignQueue), st));
  DLB_CUDA_CHECK(cudaMemsetAsync(&q->t_first_start, 0xFF, 8, st));
  DLB_CUDA_CHECK(cudaMemsetAsync(&q->t_first_exit, 0xFF, 8, st));

  // per-key precomputation (scheme.hpp:106-125)
  k_expand_a<P, 4><<<cdiv(nk * KL, 128), 128, 0, st>>>(d_sks, sk_stride, (unsigned)(nk * KL), A);
  k_sign_unpack<P, 4><<<cdiv(nk * PV, 4), 128, 0, st>>>((unsigned)nk, d_sks, sk_stride, shat,
                                                        &q->key_bad);
  c->launches += 2;
  // mu = H(tr || M), rho' = H(K || mu)  (scheme.hpp:240-248)
  const uint64_t* mu_use = mu;
  const uint64_t* rp_use = rp;
  if (d_mu_in) {
    mu_use = d_mu_in;  // stage tests supply mu and rho' directly
    rp_use = reinterpret_cast<const uint64_t*>(d_rho_prime);
  } else {
    const uint8_t* pfx = nullptr;
    unsigned plen = 0;
    if (Hashing<P>::MLDSA) DLB_TRY(mldsa_prefix(c, st, &pfx, &plen));
    k_hash_mu<Hashing<P>::MLDSA><<<cdiv(n, 128), 128, 0, st>>>(
        d_sks + 64, sk_stride, d_sks + 32, sk_stride, d_key_idx, pfx, plen, d_msgs, d_msg_off,
        (unsigned)n, mu, d_rho_prime ? nullptr : rp);
    c->launches += 1;
    if (d_rho_prime) rp_use = reinterpret_cast<const uint64_t*>(d_rho_prime);
  }

  // grid: resident CTAs of the persistent kernel
  int occ = 0;
  size_t smem_bytes = sizeof(SignSmem<P>);
  if (const char* e = getenv("DLB_SIGN_PAD_SMEM")) smem_bytes += (size_t)atoi(e);  // occupancy experiments
  DLB_CUDA_CHECK(cudaFuncSetAttribute(k_sign_persistent<P>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
  DLB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sign_persistent<P>,
                                                               kSignThreads, smem_bytes));
  if (occ < 1) occ = 1;
  const size_t grid_max = (size_t)c->sm_count * occ;
  // Psi = resident attempt slots (BatchConfig::psi).  Default (measured, profiles/
  // r01_summary.md): nine slots per task -- the speculation depth cap plus one -- while that
  // fits one warp's worth of slots per CTA (batches up to ~2,000 tasks: latency is what
  // matters there and the unluckiest task should advance nine nonces per round), about three
  // per task up to the machine's capacity, every resident slot beyond.  A Psi below the
  // machine's capacity is spread over as many CTAs as there are tasks (up to the resident
  // maximum), each using fewer of its 128 slots: the warp-per-slot stages of a round then
  // take proportionally less time.
  size_t want_slots = psi;
  if (!want_slots) {
    if (!speculate) want_slots = n;
    else want_slots = 9 * n <= grid_max * 32 ? 9 * n : 3 * n;
  }
  if (want_slots < 1) want_slots = 1;
  size_t slots_per = kSignThreads, grid = grid_max;
  if (want_slots < grid_max * kSignThreads) {
    slots_per = (want_slots + grid_max - 1) / grid_max;
    slots_per = (slots_per + 31) / 32 * 32;
    if (slots_per > (size_t)kSignThreads) slots_per = kSignThreads;
    grid = (want_slots + slots_per - 1) / slots_per;
    const size_t spread = n < grid_max ? n : grid_max;  // one task per CTA while CTAs are free
    if (grid < spread) {
      grid = spread;
      slots_per = ((want_slots + grid - 1) / grid + 31) / 32 * 32;
    }
    if (grid > grid_max) grid = grid_max;
  }
  size_t tcap = (n + grid - 1) / grid;
  if (tcap > slots_per) tcap = slots_per;
  if (single_round) {
    slots_per = kSignThreads;
    tcap = kSignThreads;
    grid = (n + kSignThreads - 1) / kSignThreads;
  }

  SignArgs a;
  memset(&a, 0, sizeof a);
  a.n = (unsigned)n;
  a.tcap = (unsigned)tcap;
  a.slots = (unsigned)slots_per;
  a.max_attempt = (65535u - (P::L - 1)) / P::L;
  a.speculate = single_round ? 0 : speculate;
  // Deepest speculative attempt a task may run in one round.  Filling every idle slot
  // (the reference's pass 2) wastes work once few tasks remain: attempt d is only needed
  // with probability (1-p)^d.  Measured on B200 (profiles/r01_summary.md): cap 8 gives the
  // best batch-10k latency and batch-100k throughput; speculate > 1 sets the cap explicitly.
  a.spec_depth = speculate > 1 ? (unsigned)speculate : 8u;
  if (const char* e = getenv("DLB_SPEC_DEPTH")) a.spec_depth = (unsigned)atoi(e);  // experiments
  a.single_round = single_round;
  a.mu = mu_use;
  a.rho_prime = rp_use;
  a.kappa0 = d_kappa0;
  a.A = A;
  a.shat = shat;
  a.key_stride = sk_stride ? 1u : 0u;
  a.key_idx = d_key_idx;
  if (c->trace_cap && !single_round) {
    DLB_TRY(dalloc(c, "s.trace", c->trace_cap * 8, &a.trace));
    a.trace_cap = (unsigned)(c->trace_cap > 0xFFFFFFFFu ? 0xFFFFFFFFu : c->trace_cap);
  }
  const size_t slots = grid * kSignThreads;
  DLB_TRY(dalloc(c, "s.y", slots * Z::Y_SLOT + 16, &a.ybytes));
  DLB_TRY(dalloc(c, "s.w", slots * Z::W_SLOT, &a.wbuf));
  DLB_TRY(dalloc(c, "s.w1", slots * S::W1_ALL, &a.w1buf));
  DLB_TRY(dalloc(c, "s.ct", slots * Hashing<P>::CTW, &a.ctbuf));
  DLB_TRY(dalloc(c, "s.c8", slots * kN, &a.c8buf));
  DLB_TRY(dalloc(c, "s.stage", slots * Z::SIG_PAD, &a.staging));
  a.sigs = d_sigs;
  a.attempts_out = d_attempts;
  a.failed_out = d_failed;
  a.dbg_ctilde = d_dbg_ct;
  a.q = q;
  cudaEventRecord(c->ev2, st);
  k_sign_persistent<P><<<(unsigned)grid, kSignThreads, smem_bytes, st>>>(a);
  cudaEventRecord(c->ev3, st);
  c->launches += 1;
  DLB_LAUNCH_CHECK();

  SignQueue hq;
  DLB_CUDA_CHECK(cudaMemcpyAsync(&hq, q, sizeof hq, cudaMemcpyDeviceToHost, st));
  DLB_CUDA_CHECK(cudaStreamSynchronize(st));
  cudaEventElapsedTime(&c->last_main_ms, c->ev2, c->ev3);
  if (stats) {
    stats->rounds = hq.rounds;
    stats->attempts = hq.attempts;
    stats->speculative = hq.speculative;
    stats->idle_slot_rounds = hq.idle_slots;
    stats->accepted_attempt_sum = hq.accepted_sum;
    stats->failed_tasks = hq.failed;
    stats->t_first_start_ns = hq.t_first_start;
    stats->t_last_start_ns = hq.t_last_start;
    stats->t_first_exit_ns = hq.t_first_exit;
    stats->t_last_exit_ns = hq.t_last_exit;
  }
  c->trace_count = a.trace ? hq.trace_count : 0;
  if (hq.key_bad) return DLB_E_KEY;
  return 0;
}

template <class P>
int sign_dev(dlb_ctx* c, size_t n, const uint8_t* d_sks, size_t sk_stride, size_t n_keys,
             const uint32_t* d_key_idx, const uint8_t* d_msgs, const uint64_t* d_msg_off,
             const uint8_t* d_rho_prime, size_t psi, int speculate, uint8_t* d_sigs,
             uint32_t* d_attempts, uint8_t* d_failed, dlb_sign_stats* stats) {
  return sign_core<P>(c, n, d_sks, sk_stride, n_keys, d_key_idx, d_msgs, d_msg_off, nullptr,
                      d_rho_prime, nullptr, psi, speculate, 0, d_sigs, d_attempts, d_failed, nullptr,
                      stats);
}

#define DLB_INST(LV)                                                                            \
  template int sign_dev<Params<LV>>(dlb_ctx*, size_t, const uint8_t*, size_t, size_t,           \
                                    const uint32_t*, const uint8_t*, const uint64_t*,           \
                                    const uint8_t*, size_t, int, uint8_t*, uint32_t*, uint8_t*, \
                                    dlb_sign_stats*);
DLB_INST(2)
DLB_INST(3)
DLB_INST(5)
DLB_INST(44)
DLB_INST(65)
DLB_INST(87)

}  // namespace dlb

using namespace dlb;

// sign_attempt<P> for n independent (key, mu, rho', kappa) tuples: one scheduler round
// with one attempt per task; z and hints are decoded back from the staged signature.
extern "C" int dlb_dbg_sign_attempt(dlb_ctx* c, int level, size_t n, const uint8_t* sks,
                                    size_t sk_stride, const uint8_t* mus, const uint8_t* rho_primes,
                                    const uint32_t* kappas, uint8_t* accepted, uint8_t* c_tilde,
                                    int32_t* z, int32_t* hints) {
  if (!c || !sks || !mus || !rho_primes || !kappas || !accepted || !c_tilde || !z || !hints)
    return DLB_E_ARG;
  cudaSetDevice(c->device);
  auto run = [&](auto p) -> int {
    using P = decltype(p);
    using S = Sizes<P>;
    const size_t nk = sk_stride ? n : 1;
    uint8_t *dsk, *dsig, *dfail, *dct, *drp;
    uint64_t* dmu;
    uint32_t *dk, *datt;
    DLB_TRY(dalloc(c, "io.sk", nk * S::SK, &dsk));
    DLB_TRY(dalloc(c, "dbg.a", n * 8, &dmu));
    DLB_TRY(dalloc(c, "dbg.b", n * 64, &drp));
    DLB_TRY(dalloc(c, "dbg.c", n, &dk));
    DLB_TRY(dalloc(c, "io.sig", n * S::SIG + 8, &dsig));
    DLB_TRY(dalloc(c, "io.att", n, &datt));
    DLB_TRY(dalloc(c, "io.fail", n, &dfail));
    DLB_TRY(dalloc(c, "dbg.d", n * Hashing<P>::CT, &dct));
    cudaStream_t st = c->s();
    DLB_CUDA_CHECK(cudaMemcpyAsync(dsk, sks, nk * S::SK, cudaMemcpyHostToDevice, st));
    DLB_CUDA_CHECK(cudaMemcpyAsync(dmu, mus, n * 64, cudaMemcpyHostToDevice, st));
    DLB_CUDA_CHECK(cudaMemcpyAsync(drp, rho_primes, n * 64, cudaMemcpyHostToDevice, st));
    DLB_CUDA_CHECK(cudaMemcpyAsync(dk, kappas, n * 4, cudaMemcpyHostToDevice, st));
    DLB_CUDA_CHECK(cudaMemsetAsync(dsig, 0, n * S::SIG, st));
    DLB_TRY(sign_core<P>(c, n, dsk, sk_stride, 0, nullptr, nullptr, nullptr, dmu, drp, dk, 0, 0, 1,
                         dsig, datt, dfail, dct, nullptr));
    uint8_t* hsig = new uint8_t[n * S::SIG];
    uint8_t* hfail = new uint8_t[n];
    cudaMemcpyAsync(hsig, dsig, n * S::SIG, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hfail, dfail, n, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(c_tilde, dct, n * Hashing<P>::CT, cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
      memset(z, 0, n * P::L * kN * 4);
      memset(hints, 0, n * P::K * kN * 4);
      for (size_t t = 0; t < n; ++t) {
        accepted[t] = hfail[t] ? 0 : 1;
        if (!accepted[t]) continue;
        const uint8_t* sg = hsig + t * S::SIG;
        for (int j = 0; j < P::L; ++j)
          for (int m = 0; m < kN; ++m) {
            const size_t bit = (size_t)m * P::Z_BITS;
            uint32_t raw = 0;
            for (int b = 0; b < P::Z_BITS; ++b)
              raw |= (uint32_t)((sg[S::SIG_Z + j * S::Z_POLY + ((bit + b) >> 3)] >> ((bit + b) & 7)) & 1) << b;
            z[(t * P::L + j) * kN + m] = P::GAMMA1 - (int32_t)raw;
          }
        const uint8_t* h = sg + S::SIG_Z + P::L * S::Z_POLY;
        unsigned prev = 0;
        for (int i = 0; i < P::K; ++i) {
          const unsigned cnt = h[P::OMEGA + i];
          for (unsigned k = prev; k < cnt && k < (unsigned)P::OMEGA; ++k)
            hints[(t * P::K + i) * kN + h[k]] = 1;
          prev = cnt;
        }
      }
    }
    delete[] hsig;
    delete[] hfail;
    return e == cudaSuccess ? 0 : -1000 - (int)e;
  };
  switch (level) {
    case 2: return run(Params<2>{});
    case 3: return run(Params<3>{});
    case 5: return run(Params<5>{});
    case 44: return run(Params<44>{});
    case 65: return run(Params<65>{});
    case 87: return run(Params<87>{});
    default: return DLB_E_LEVEL;
  }
}
