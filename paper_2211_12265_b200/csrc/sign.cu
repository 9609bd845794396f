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
#define DLB_R0_MIN 1  // S4's r0 norm check as an unsigned minimum (+0.5 %, parity campaign green)
#endif
namespace dlb {

// matrix-row iterations in flight in S2's accumulation loop (A/B knob: with one key per task the
// matrix streams from HBM; profiles/r02_summary.md section 2)
#ifndef DLB_SIGN_J_UNROLL
#define DLB_SIGN_J_UNROLL 1
#endif
#define DLB_SIGN_PRAGMA_(x) _Pragma(#x)
#define DLB_SIGN_PRAGMA(x) DLB_SIGN_PRAGMA_(x)
#define DLB_SIGN_J_PRAGMA DLB_SIGN_PRAGMA(unroll DLB_SIGN_J_UNROLL)
#ifndef DLB_SIGN_MINB
#define DLB_SIGN_MINB 4  // resident CTAs per SM: 5 (96 regs) was measured slower -- it squeezes L1 to ~10 KB
#endif
constexpr int kSignThreads = 128;          // threads = attempt slots per CTA
constexpr int kSignWarps = kSignThreads / 32;
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;
constexpr int kChunkBytes = 1024;  // cp.async landing buffer: one packed polynomial
constexpr int kPrepKeys = 16;       // keys a scheduler CTA precomputes per claim

// ---- per-key precomputation -----------------------------------------------------------
// One warp per (key, polynomial): s1 (L), s2 (K), t0 (K) unpacked from the secret key,
// range-checked (packing.hpp:79-86), transformed; stored reduced, natural order.
template <class P, bool NC>
__device__ __forceinline__ void sign_unpack_poly(unsigned id, const uint8_t* __restrict__ sks, size_t sk_stride,
                                                 int32_t* __restrict__ shat, unsigned* __restrict__ key_bad,
                                                 int32_t* tile, const int2* zs, int lane) {
  using S = Sizes<P>;
  constexpr int PV = P::L + 2 * P::K;
  const unsigned key = id / PV, p = id % PV;
  const uint8_t* sk = sks + (size_t)key * sk_stride;
  int32_t r[8];
  bool bad = false;
  if (p < (unsigned)(P::L + P::K)) {
    const uint8_t* src = sk + S::SK_S1 + p * S::ETA_POLY;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t raw = load_bits_t<NC>(src, (lane + 32 * e) * P::ETA_BITS, P::ETA_BITS);
      bad = bad || raw > 2u * P::ETA;
      r[e] = P::ETA - (int32_t)raw;
    }
  } else {
    const uint8_t* src = sk + S::SK_T0 + (p - P::L - P::K) * S::T0_POLY;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      r[e] = 4096 - (int32_t)load_bits_t<NC>(src, (lane + 32 * e) * 13, 13);
  }
  ntt_fwd(r, tile, zs, lane);
  int4* dst = reinterpret_cast<int4*>(shat + (size_t)id * kN) + 2 * lane;
  dst[0] = make_int4(reduce32(r[0]), reduce32(r[1]), reduce32(r[2]), reduce32(r[3]));
  dst[1] = make_int4(reduce32(r[4]), reduce32(r[5]), reduce32(r[6]), reduce32(r[7]));
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(key_bad, 1u);
}

template <class P, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_sign_unpack(unsigned n_keys, const uint8_t* __restrict__ sks, size_t sk_stride,
                  int32_t* __restrict__ shat, unsigned* __restrict__ key_bad) {
  constexpr int PV = P::L + 2 * P::K;
  __shared__ __align__(16) int2 zs[256], nzs[256];
  __shared__ __align__(16) int32_t tiles[WARPS][kTileWords];
  load_twiddles(zs, nzs);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned id = blockIdx.x * WARPS + warp;
  if (id >= n_keys * PV) return;
  sign_unpack_poly<P, true>(id, sks, sk_stride, shat, key_bad, tiles[warp], zs, lane);
}

// ---- device-side scheduler state -----------------------------------------------------
//
// Batches in flight.  A submitted batch is described by one SignBatch in a device ring
// (slot = ticket % kRing).  Every scheduler CTA, whichever ticket its kernel was launched for,
// serves every published batch of its parameter set: lane p of warp 0 watches ring slot p, and
// the CTA refills its open-task table from ANY batch with unclaimed tasks, oldest ticket first,
// before it speculates (the reference's pass 1 before pass 2, scheduler.hpp:58-92, extended
// across batches -- the paper's in-flight batches), so the tail of one batch
// overlaps the body of the next ones and, while work keeps arriving, every slot runs a first
// attempt.  A view of a ring slot is tagged with the gate value (ticket + 1) it was loaded for
// and tasks are claimed by compare-and-swap on the batch's (ticket + 1 : next task) word, so a
// view that outlived its batch can never claim from the slot's next occupant: CTAs may stay
// resident for as long as the flow lasts, and a slot is reused as soon as its ticket was waited
// for.  One kernel is still launched per ticket (kLanes stream lanes, one scratch set each): it
// provides the CTAs when none are resident and always serves its own batch, so no batch is ever
// without a kernel that will take it.  Batches of another parameter set (or stage tests, which
// only their own kernel serves) are honoured first come first served: a CTA claims nothing
// younger than the oldest batch it cannot serve, retires when its table is empty, and that
// batch's own kernel gets the SMs.  A CTA never waits for anything; it exits when its table is
// empty and nothing it may serve has unclaimed tasks.  Completion is per batch (SignBatch::done
// reaching n raises a flag in mapped host memory), not per kernel.

// what a CTA keeps in shared memory of the batch in ring slot i: the fields the
// stages read per slot.  Everything else (output arrays of the commit step, the inputs of the
// digest stage, test hooks) is read from the descriptor itself when needed -- immutable, and
// fetched behind the acquire that made the batch visible.
struct BatchView {
  unsigned n, tcap, max_attempt, spec_depth, key_stride, ticket1;  // ticket1 = gate value the view was loaded for
  int level;
  unsigned exclusive;
  unsigned stage_out;  // never write a signature in place (host-mapped output, DLB_HOST_STAGE)
  unsigned prep_n;   // keys the scheduler precomputes for this batch (0: none)
  unsigned prep_ok;  // ... and they have all been seen done (behind an acquire)
  const uint64_t* mu;
  const uint64_t* rho_prime;
  const uint32_t* kappa0;
  const int32_t* A;
  const int32_t* shat;
  const uint32_t* key_idx;
  uint8_t* sigs;
  SignBatch* g;  // the descriptor in the ring (cold fields, mutable counters)
};

struct SignArgs {             // one scheduler-kernel instance
  SignBatch* ring;            // kRing descriptors
  unsigned ticket;            // own ticket
  unsigned window;            // 1: the kernel serves its own batch only (stage tests); else every batch in flight
  unsigned slots;             // attempt slots a CTA fills with speculation (<= 128): small batches are
                              // spread over more CTAs with fewer slots each to cut round latency
  int single_round;           // stage-test mode: exactly one round, then fail open tasks
  unsigned boost_thr;         // a task past this many failed attempts is a straggler (0 = no boost)
  unsigned boost_depth;       // extra nonces a straggler runs per round while work is queued
  uint32_t* trace;            // nullable: per-round records of 8 words (dlb_round_trace)
  unsigned trace_cap;
  uint32_t* alog;             // nullable: per executed attempt 4 words (dlb_assignment)
  unsigned alog_cap;
  SignLog* log;
  // per-CTA scratch in HBM/L2, indexed [cta][slot] (one set per stream lane)
  uint8_t* ybytes;
  int32_t* wbuf;
  uint8_t* w1buf;
  uint64_t* ctbuf;
  int8_t* c8buf;
  uint8_t* staging;
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
  uint32_t utask[kSignThreads];    // open tasks of this CTA (compact): task id within its batch
  uint32_t unext[kSignThreads];    // their next unresolved attempt ordinal
  uint8_t ubatch[kSignThreads];    // their batch: ring slot (ticket % kRing)
  uint32_t slot_task[kSignThreads];     // task id or kNoSlot
  uint32_t slot_attempt[kSignThreads];
  uint8_t slot_batch[kSignThreads];
  uint8_t slot_valid[kSignThreads];
  int32_t winner[kSignThreads];    // per open task: winning slot, -1 none, -2 failed
  uint32_t warp_sums[kSignWarps];
  BatchView bv[kRing];             // descriptor of the batch last seen published in each ring slot
  unsigned bcnt[kRing];            // open tasks held per batch
  unsigned bfin[kRing];            // tasks of each batch finished in the current round
  unsigned U, Uold, span, need_hash;
  unsigned B;                      // tasks (table front) that share the slots behind the first U
  unsigned cursor2, cursor4;  // next unclaimed slot of stages S2 / S4 (warps pull slots)
  unsigned r_on, r_spec;      // this round's assigned / speculative slots (trace)
  unsigned rounds;            // rounds this CTA has run
  unsigned prep_slot, prep_k0, prep_cnt;  // keys to precompute before this round (prep_cnt 0: none)
  unsigned prep_wait;         // a servable batch's precomputation is in other CTAs' hands
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
    DLB_SIGN_J_PRAGMA
    for (int j = 0; j < P::L; ++j) {
      const int4 a0 = ld_weak(ap + j * (kN / 4)), a1 = ld_weak(ap + j * (kN / 4) + 1);
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
  const int4 s0 = ld_weak(sp), s1 = ld_weak(sp + 1);
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
//
// Returns 0 when the attempt is accepted.  DBG = false: any other value means rejected (the
// first failing check ends the attempt).  DBG = true (stage tests, scheme.hpp:133-138 with
// injectable bounds): nothing is skipped and the value is 1 + the RejectStage the reference
// would report -- the first failing check in ITS order (z, r0, c t0, hint weight).
template <class P, bool DBG>
__device__ __forceinline__ int stage_finish(SignWarpScratch<P>& ws, SlotPipe& pp, int par,
                                            const int2* zs, const int2* nzs, int lane,
                                            const uint8_t* ybytes, int32_t* wrows,
                                            const int8_t* next_c8, const uint64_t* ct,
                                            const int32_t* shat, uint8_t* stage_sig, bool direct,
                                            const int32_t* bounds) {
  const int32_t z_bound = DBG ? bounds[0] : P::GAMMA1 - P::BETA;
  const int32_t r0_bound = DBG ? bounds[1] : P::GAMMA2 - P::BETA;
  const int32_t vt_bound = DBG ? bounds[2] : P::GAMMA2;
  unsigned fails = 0;  // DBG: bit 0 z, bit 1 r0, bit 2 c t0
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
      constexpr bool R0MIN = DLB_R0_MIN && !DBG;
      uint32_t worst = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int32_t d = freeze_near(wrow[lane + 32 * e] - t[e]);  // [0, q) - (-q, q)
        if constexpr (R0MIN) {
          // |r0| < B without materialising the centred r0: a0 = d - r1 * 2 gamma2 is r0 or, when
          // HighBits wrapped to 0, r0 + q; shifted by B - 1 the valid one lands in [0, 2B - 1)
          constexpr int32_t B = P::GAMMA2 - P::BETA;
          const int32_t a0 = d - highbits<P::GAMMA2>(d) * 2 * P::GAMMA2;
          const uint32_t u = (uint32_t)(a0 + B - 1);
          worst = max(worst, min(u, u - (uint32_t)kQ));
        } else {
          int32_t r0;
          decompose<P::GAMMA2>(d, r0);
          bad = bad || abs(r0) >= r0_bound;
        }
        wdst[lane + 32 * e] = d;  // read back by this same lane in the hint phase
      }
      if constexpr (R0MIN) bad = worst >= 2u * (P::GAMMA2 - P::BETA) - 1u;
    } else if (p < R) {
      uint32_t raw[8];
      unpack_strided<P::Z_BITS>(cur, lane, raw);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int32_t y = P::GAMMA1 - (int32_t)raw[e];
        const int32_t z = y + reduce32(t[e]);  // |y| <= gamma1, |c s1| <= beta: no wrap, centred
        bad = bad || abs(z) >= z_bound;
        ws.vhat[p - P::K][e][lane] = z;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int32_t vt = reduce32(t[e]);  // |c t0| <= tau * 2^12 < 2^22: already centred
        bad = bad || abs(vt) >= vt_bound;
        const int h = highbits<P::GAMMA2>(freeze_near(wcs2[e] + vt)) != highbits<P::GAMMA2>(wcs2[e]);
        const unsigned mask = __ballot_sync(FULL, h);
        if (lane == 0) ws.hbits[p - R][e] = mask;
        weight += __popc(mask);
      }
    }
    if (__any_sync(FULL, bad)) {
      if (!DBG) return 1;
      fails |= p < P::K ? 2u : (p < R ? 1u : 4u);
    }
  }
  if (DBG && fails) return 1 + (int)(__ffs(fails) - 1);
  if (weight > (unsigned)P::OMEGA) return DBG ? 4 : 1;

  // accepted: c~ | z | hints into the staging slot -- or, for a task's next unresolved nonce
  // (depth 0: if it is valid it IS the winner, scheduler.hpp:117), straight into the task's
  // signature (`direct`; any alignment), so that the commit step has nothing to copy
  // (every piece is assembled in shared memory and leaves as whole coalesced words: the
  // destination may be pinned host memory)
  uint32_t* scr = reinterpret_cast<uint32_t*>(pp.ring(pp.k));  // free ring buffer, 1 KiB
  if (lane < 2 * Hashing<P>::CTW) scr[lane] = reinterpret_cast<const uint32_t*>(ct)[lane];
  __syncwarp();
  warp_store_unaligned(stage_sig, scr, Hashing<P>::CT, lane);
  __syncwarp();
#pragma unroll 1
  for (int j = 0; j < P::L; ++j) {
#pragma unroll
    for (int e = 0; e < 8; ++e) ws.tile[lane + 36 * e] = P::GAMMA1 - ws.vhat[j][e][lane];
    __syncwarp();
    if (direct)
      pack_tile<P::Z_BITS, false>(ws.tile, pp.ring(pp.k), stage_sig + S::SIG_Z + j * S::Z_POLY, lane);
    else
      pack_tile<P::Z_BITS, true>(ws.tile, pp.ring(pp.k), stage_sig + S::SIG_Z + j * S::Z_POLY, lane);
  }
  // hint section (packing.hpp:105-118): positions ascending per polynomial, cumulative counts
  // behind them, unused bytes zero.  (staging: the padding behind the signature is cleared
  // too, the word-wise commit copy reads it)
  constexpr int HWORDS = (S::HINT + (SignSizes<P>::SIG_PAD - S::SIG) + 3) / 4;
  uint8_t* hsm = reinterpret_cast<uint8_t*>(scr);
  for (int w = lane; w < HWORDS; w += 32) scr[w] = 0;
  __syncwarp();
  unsigned count = 0;
#pragma unroll 1
  for (int i = 0; i < P::K; ++i) {
#pragma unroll 1
    for (int e = 0; e < 8; ++e) {
      const unsigned mask = ws.hbits[i][e];
      if ((mask >> lane) & 1) hsm[count + __popc(mask & ((1u << lane) - 1))] = (uint8_t)(32 * e + lane);
      count += __popc(mask);
    }
    if (lane == 0) hsm[P::OMEGA + i] = (uint8_t)count;
  }
  __syncwarp();
  warp_store_unaligned(stage_sig + S::SIG_Z + P::L * S::Z_POLY, scr,
                       direct ? S::HINT : S::HINT + (SignSizes<P>::SIG_PAD - S::SIG), lane);
  __syncwarp();
  return 0;
}

template <class P, bool DBG>
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
    sm.rounds = 0;
  }
  if (tid < kRing) {
    sm.bcnt[tid] = sm.bfin[tid] = 0;
    sm.bv[tid].ticket1 = 0;
  }
  __syncthreads();

  while (true) {
    // ---- refill from the device work queues of the batches in flight -----------------------
    // Warp 0, lane p looks at ring slot p.  A batch becomes visible through an acquire load of
    // its gate word (the host writes it after the descriptor and all inputs are in place; the
    // acquire also drops stale L1 lines of whatever occupied those arenas before).  Tasks are
    // claimed oldest ticket first, up to tcap open tasks per batch and 128 per CTA, with a
    // compare-and-swap on the batch's 64-bit queue word (ticket + 1 : next task): a claim can
    // only ever succeed against the batch the view was loaded for, so a CTA may outlive its own
    // batch for as long as work keeps arriving and ring slots are reused under it.
    if (warp == 0) {
      unsigned U = sm.U;
      if (lane == 0) {
        sm.span = 0;
        sm.Uold = U;
        sm.need_hash = 0;
        sm.prep_cnt = 0;
        sm.prep_wait = 0;
      }
      // Stragglers.  With work queued every slot runs a first attempt, so a task deep in its
      // rejection loop advances one nonce per full-length round and its batch completes long
      // after its siblings (a pipeline of bounded depth then stalls on it).  The table is ordered
      // by age; the tasks at its front that are past boost_thr failed attempts keep boost_depth
      // slots each free of new work and run that many extra nonces per round -- a few percent of the
      // slots (0.765^16 = 1.4 % of the tasks are that deep) for half the tail.
      unsigned n_s = 0;
      if (a.boost_thr && U) {
        const bool deep = (unsigned)lane < U && sm.unext[lane] >= a.boost_thr && sm.bv[sm.ubatch[lane]].spec_depth > 0;
        const unsigned m = __ballot_sync(0xffffffffu, deep);
        n_s = m == 0xffffffffu ? 32u : (unsigned)__ffs(~m) - 1u;  // length of the leading run
        n_s = min(n_s, 32u / a.boost_depth);
      }
      const unsigned cap = (unsigned)kSignThreads - n_s * a.boost_depth;
      if (U < cap && !(a.single_round && sm.rounds > 0)) {
        // a.window == 1 (stage tests): only the kernel's own batch
        unsigned tk = 0xFFFFFFFFu, blocked = 0xFFFFFFFFu, ptk = 0xFFFFFFFFu;
        bool pwait = false;
        if (a.window > 1u || (unsigned)lane == a.ticket % kRing) {
          SignBatch* g = a.ring + lane;
          const unsigned g1 = ld_acquire(&g->gate);
          BatchView& v = sm.bv[lane];
          const bool own = g1 == a.ticket + 1u;
          if (g1 != 0 && v.ticket1 != g1 && sm.bcnt[lane] == 0) {
            // (a view is only replaced when none of the previous occupant's tasks is open here,
            // which its completion -- the precondition of the slot's reuse -- implies)
            v.n = g->n;
            v.tcap = g->tcap;
            v.max_attempt = g->max_attempt;
            v.spec_depth = g->spec_depth;
            v.key_stride = g->key_stride;
            v.level = g->level;
            v.exclusive = g->exclusive;
            v.prep_n = g->prep_n;
            v.stage_out = g->stage_out;
            v.prep_ok = 0;
            v.mu = g->mu;
            v.rho_prime = g->rho_prime;
            v.kappa0 = g->kappa0;
            v.A = g->A;
            v.shat = g->shat;
            v.key_idx = g->key_idx;
            v.sigs = g->sigs;
            v.g = g;
            v.ticket1 = g1;
          }
          if (g1 != 0 && v.ticket1 == g1) {
            const bool mine = v.level == P::LEVEL && (own || (!v.exclusive && a.window > 1u));
            bool ready = true;
#ifndef DLB_AB_NO_PREP  // (A/B switch: the scheduler without its precomputation code; shared cached keys only)
            if (v.prep_n && !v.prep_ok) {  // keys still being precomputed (by scheduler CTAs, below)
              if (ld_acquire(&g->prep_done) >= v.prep_n) {
                v.prep_ok = 1;
              } else {
                ready = false;
                const unsigned long long pq = ld_relaxed(&g->prep_q);
                if (mine && (unsigned)(pq >> 32) == g1) {
                  if ((unsigned)pq < v.prep_n) ptk = g1 - 1u;
                  else pwait = true;
                }
              }
            }
#endif
            const unsigned long long q = ld_relaxed(&g->head);
            const bool open = (unsigned)(q >> 32) == g1 && (unsigned)q < v.n;
            if (open) {
              if (mine) {
                if (ready && sm.bcnt[lane] < v.tcap) tk = g1 - 1u;
              } else {
                blocked = g1 - 1u;  // unclaimed work this kernel cannot serve
              }
            }
          }
        }
        __syncwarp();  // the views written above are read by every lane below
        // First come, first served across parameter sets: nothing younger than the oldest batch
        // this kernel cannot serve is claimed (its own kernel gets the SMs as these CTAs retire),
        // except the kernel's own batch, which it always serves -- no batch is left without a
        // kernel that will take it.
        blocked = __reduce_min_sync(0xffffffffu, blocked);
        if (tk != 0xFFFFFFFFu && tk > blocked && tk != a.ticket) tk = 0xFFFFFFFFu;
        while (U < cap) {
          const unsigned best = __reduce_min_sync(0xffffffffu, tk);
          if (best == 0xFFFFFFFFu) break;
          const int i = (int)(best % kRing);
          if (lane == i) tk = 0xFFFFFFFFu;
          const BatchView& v = sm.bv[i];
          const unsigned want = min(v.tcap - sm.bcnt[i], cap - U);
          unsigned base = 0, got = 0;
          if (lane == 0) {
            unsigned long long q = ld_relaxed(&v.g->head);
            while ((unsigned)(q >> 32) == v.ticket1 && (unsigned)q < v.n) {
              const unsigned take = min(want, v.n - (unsigned)q);
              const unsigned long long old = atomicCAS(&v.g->head, q, q + take);
              if (old == q) {
                base = (unsigned)q;
                got = take;
                break;
              }
              q = old;
            }
            if (got) {
              unsigned long long now;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
              atomicMin(&v.g->t_first_start, now);
              atomicMax(&v.g->t_last_start, now);
              sm.bcnt[i] += got;
              if (v.g->msg_off) sm.need_hash = 1;
            }
          }
          base = __shfl_sync(0xffffffffu, base, 0);
          got = __shfl_sync(0xffffffffu, got, 0);
          for (unsigned t = lane; t < got; t += 32) {
            sm.utask[U + t] = base + t;
            sm.unext[U + t] = 0;
            sm.ubatch[U + t] = (uint8_t)i;
          }
          U += got;
        }
        // Per-key precomputation of a batch whose keys are not cached: a run of keys is claimed
        // like tasks are and expanded by this CTA before the round (the precomputation of the next
        // batches thus overlaps the signing of the current ones; a separate kernel could not become
        // resident beside the scheduler grid).  Oldest batch first.
        ptk = __reduce_min_sync(0xffffffffu, ptk);
        pwait = __any_sync(0xffffffffu, pwait);
        if (lane == 0) {
          sm.prep_wait = pwait ? 1u : 0u;
          if (ptk != 0xFFFFFFFFu) {
            const BatchView& v = sm.bv[ptk % kRing];
            unsigned long long q = ld_relaxed(&v.g->prep_q);
            while ((unsigned)(q >> 32) == v.ticket1 && (unsigned)q < v.prep_n) {
              const unsigned take = min((unsigned)kPrepKeys, v.prep_n - (unsigned)q);
              const unsigned long long old = atomicCAS(&v.g->prep_q, q, q + take);
              if (old == q) {
                sm.prep_slot = ptk % kRing;
                sm.prep_k0 = (unsigned)q;
                sm.prep_cnt = take;
                break;
              }
              q = old;
            }
            if (!sm.prep_cnt) sm.prep_wait = 1u;  // lost the race for the last keys: they are in hand
          }
        }
        __syncwarp();
        if (lane == 0) sm.U = U;
      }
      // the table is full up to the cap: the spare slots belong to the stragglers; otherwise (queues
      // dry) every open task shares them breadth first, the reference's pass 2
      if (lane == 0) sm.B = (n_s && U >= cap) ? n_s : U;
    }
    __syncthreads();
    const unsigned U = sm.U;
    const unsigned prep_cnt = sm.prep_cnt, prep_wait = sm.prep_wait;
#ifndef DLB_AB_NO_PREP
    if (prep_cnt) {
      // ExpandA (sampling.hpp:42-56; one sponge per matrix polynomial, 32 streams per warp pass)
      // and the secret vectors (scheme.hpp:106-125; one warp per polynomial) of keys
      // [prep_k0, prep_k0 + prep_cnt) of the batch in ring slot prep_slot.  The stage buffers of
      // the round are free here and lend their shared memory.
      constexpr int KL = P::K * P::L, PV = P::L + 2 * P::K;
      const BatchView& v = sm.bv[sm.prep_slot];
      SignBatch* g = v.g;
      const unsigned k0 = sm.prep_k0, cnt = prep_cnt;
      const uint8_t* sks = g->prep_sks;
      const size_t stride = g->prep_stride;
      static_assert(sizeof(sm.u) >= sizeof(int32_t) * kSignWarps * 32 * kExpandAStageStride, "ExpandA staging fits the stage buffers");
      auto stage = reinterpret_cast<int32_t(*)[32][kExpandAStageStride]>(&sm.u);
      const unsigned send = (k0 + cnt) * KL;
      for (unsigned p0 = k0 * KL + (unsigned)warp * 32u; p0 < send; p0 += (unsigned)kSignThreads)
        expand_a_warp<P, false>(sks, stride, p0, send, const_cast<int32_t*>(v.A), stage[warp], lane);
      __syncthreads();
      for (unsigned id = k0 * PV + (unsigned)warp; id < (k0 + cnt) * PV; id += (unsigned)kSignWarps)
        sign_unpack_poly<P, false>(id, sks, stride, const_cast<int32_t*>(v.shat), &g->key_bad,
                                   sm.u.a.ws[warp].tile, sm.zs, lane);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(&g->prep_done, cnt);
      }
    }
#endif
    if (U == 0) {
      if (!prep_cnt && !prep_wait) break;
      // look again: the batch may be claimable now, or its last keys are being expanded by other
      // CTAs and its tasks follow shortly.  (Barrier: warp 0 rewrites the refill's shared words.)
      if (!prep_cnt) __nanosleep(2000);
      __syncthreads();
      continue;
    }
    const unsigned B = sm.B;

    // ---- S0: mu = H(tr || M), rho' = H(K || mu) of the tasks just claimed (scheme.hpp:240-248)
    if (sm.need_hash) {
      if ((unsigned)tid >= sm.Uold && (unsigned)tid < U) {
        const BatchView& v = sm.bv[sm.ubatch[tid]];
        const SignBatch* g = v.g;
        const uint64_t* msg_off = g->msg_off;
        if (msg_off) {
          const unsigned task = sm.utask[tid];
          const size_t kt = v.key_idx ? (size_t)ld_weak(v.key_idx + task) : (size_t)task * v.key_stride;
          const uint8_t* sk = g->sk_base + kt * S::SK;
          const uint64_t m0 = ld_weak(msg_off + task), m1 = ld_weak(msg_off + task + 1);
          uint64_t* rp_w = g->rp_w;
          hash_mu_task<Hashing<P>::MLDSA, false>(
              reinterpret_cast<const uint64_t*>(sk + 64), reinterpret_cast<const uint64_t*>(sk + 32),
              g->pfx, g->plen, g->msgs + m0, (size_t)(m1 - m0), g->mu_w + (size_t)task * 8,
              rp_w ? rp_w + (size_t)task * 8 : nullptr);
        }
      }
      __syncthreads();
    }

    // ---- schedule (scheduler.hpp:58-92): pass 1 = slot u runs open task u's next nonce; pass 2 =
    // the slots behind the table run further nonces, breadth first over the first B tasks --------
    // Depth 0 (pass 1) always runs.  Speculative depths (pass 2) only use the first a.slots
    // slots and only exist when the queues could not fill the table, because the refill above
    // comes first.
    {
      // slots [0, U): depth 0 of every open task; slot U + j: task j mod B at depth 1 + j div B
      const unsigned j = (unsigned)tid >= U ? (unsigned)tid - U : 0u;
      const unsigned u = (unsigned)tid < U ? (unsigned)tid : j % B;
      const unsigned depth = (unsigned)tid < U ? 0u : 1u + j / B;
      const unsigned bi = sm.ubatch[u];
      const BatchView& v = sm.bv[bi];
      const unsigned att = sm.unext[u] + depth;
      const bool boosted = B != U;  // spare slots reserved for stragglers, not the kernel's pass-2 budget
      const bool on = (depth == 0 || (boosted ? depth <= min(a.boost_depth, v.spec_depth)
                                              : ((unsigned)tid < a.slots && depth <= v.spec_depth))) &&
                      att <= v.max_attempt;
      const unsigned task = sm.utask[u];
      sm.slot_task[tid] = on ? task : kNoSlot;
      sm.slot_attempt[tid] = att;
      sm.slot_batch[tid] = (uint8_t)bi;
      sm.slot_valid[tid] = 0;
      if (tid == 0) sm.cursor2 = sm.cursor4 = 0;
      // per-batch counters, one atomic per warp and batch
      const unsigned grp = __match_any_sync(0xffffffffu, on ? bi : 0xFFu);
      const unsigned specm = __ballot_sync(0xffffffffu, on && depth > 0);
      if (on && lane == __ffs(grp) - 1) {
        atomicAdd(&v.g->attempts, (unsigned long long)__popc(grp));
        const unsigned ns = __popc(grp & specm);
        if (ns) atomicAdd(&v.g->speculative, (unsigned long long)ns);
      }
      const unsigned hi = __reduce_max_sync(0xffffffffu, on ? (unsigned)tid + 1u : 0u);
      if (lane == 0 && hi) atomicMax(&sm.span, hi);
      if (a.alog && on) {  // Assignment{slot, task, attempt, kappa} (scheduler.hpp:14-19)
        const unsigned long long idx = atomicAdd(&a.log->alog_count, 1ull);
        if (idx < a.alog_cap) {
          const unsigned k0 = v.kappa0 ? ld_weak(v.kappa0 + task) : 0u;
          reinterpret_cast<uint4*>(a.alog)[idx] =
              make_uint4((unsigned)cta * kSignThreads + tid, task, att, k0 + att * P::L);
        }
      }
      const unsigned n_on = __syncthreads_count(on);
      const unsigned n_spec = __syncthreads_count(on && depth > 0);
      if (warp == 0) {  // a round counts for every batch present; idle slots go to the oldest
        const bool present = sm.bcnt[lane] > 0;
        const unsigned pm = __ballot_sync(0xffffffffu, present);
        if (present) {
          atomicAdd(&sm.bv[lane].g->rounds, 1ull);
          if (lane == __ffs(pm) - 1 && a.slots > n_on)
            atomicAdd(&sm.bv[lane].g->idle_slots, (unsigned long long)(a.slots - n_on));
        }
      }
      if (tid == 0) {
        sm.rounds += 1;
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
    // towards 5.  Active slots lie in [0, span); items are laid out polynomial-major so
    // the lanes of a warp share j.  With all 128 slots active this is thread t -> slot t,
    // j = 0 .. L-1.
    {
      const unsigned span = sm.span;
#pragma unroll 1
      for (unsigned item = tid; item < span * P::L; item += kSignThreads) {
        const unsigned slot = item % span, j = item / span;
        const unsigned task = sm.slot_task[slot];
        if (task == kNoSlot) continue;
        const BatchView& v = sm.bv[sm.slot_batch[slot]];
        const unsigned k0 = v.kappa0 ? ld_weak(v.kappa0 + task) : 0u;
        const unsigned kappa = k0 + sm.slot_attempt[slot] * P::L;
        expand_mask_stream<P, false>(v.rho_prime + (size_t)task * 8, kappa + j,
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
    auto key_of = [&](int s) -> size_t {  // key table index of the task in slot s
      const BatchView& v = sm.bv[sm.slot_batch[s]];
      return v.key_idx ? (size_t)ld_weak(v.key_idx + sm.slot_task[s])
                       : (size_t)sm.slot_task[s] * v.key_stride;
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
        stage_w<P>(sm.u.a.ws[warp], pp, sm.zs, sm.nzs, lane, ybytes + (size_t)s * Z::Y_SLOT,
                   nx < kSignThreads ? ybytes + (size_t)nx * Z::Y_SLOT : nullptr,
                   sm.bv[sm.slot_batch[s]].A + key_of(s) * (P::K * P::L * kN),
                   wbuf + (size_t)s * Z::W_SLOT, w1buf + (size_t)s * S::W1_ALL);
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
            sm.bv[sm.slot_batch[tid]].mu + (size_t)my_task * 8,
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
        const BatchView& v = sm.bv[sm.slot_batch[s]];
        const bool direct = (unsigned)s < U && !v.stage_out;  // depth 0: the task's next unresolved nonce
        const int rej = stage_finish<P, DBG>(
            sm.u.a.ws[warp], pp, par, sm.zs, sm.nzs, lane, ybytes + (size_t)s * Z::Y_SLOT,
            wbuf + (size_t)s * Z::W_SLOT, nx < kSignThreads ? c8buf + (size_t)nx * kN : nullptr,
            ctbuf + s * CTW, v.shat + key_of(s) * ((P::L + 2 * P::K) * kN),
            direct ? v.sigs + (size_t)sm.slot_task[s] * S::SIG : staging + (size_t)s * Z::SIG_PAD, direct,
            DBG ? v.g->bounds : nullptr);
        if (lane == 0) {
          sm.slot_valid[s] = rej == 0 ? 1 : 0;
          // RejectStage of the reference (scheme.hpp:34): 0 z, 1 r0, 2 c t0, 3 hint weight; 255 accepted
          if (DBG && v.g->dbg_stage) v.g->dbg_stage[sm.slot_task[s]] = rej ? (uint8_t)(rej - 1) : (uint8_t)255;
        }
        s = nx;
        par ^= 1;
      }
      cp_async_wait<0>();
    }
    __syncthreads();

    // ---- commit: smallest valid attempt per task wins (scheduler.hpp:97-136) --------
    bool keep = false;
    unsigned my_u_task = 0, my_u_next = 0, my_u_batch = 0;
    if ((unsigned)tid < U) {
      const unsigned task = sm.utask[tid];
      unsigned next = sm.unext[tid];
      const unsigned bi = sm.ubatch[tid];
      const BatchView& v = sm.bv[bi];
      int win = -1;
      unsigned ran = 0;
      for (unsigned s = tid; s < (unsigned)kSignThreads; s = s < U ? U + s : s + B) {
        if (s >= U && (unsigned)tid >= B) break;  // only the first B tasks own slots behind the table
        if (sm.slot_task[s] == kNoSlot) break;
        ++ran;
        if (sm.slot_valid[s]) {
          win = (int)s;
          break;
        }
      }
      const SignBatch* g = v.g;
      if (uint8_t* dbg_ct = g->dbg_ctilde) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(ctbuf + tid * CTW);
        uint32_t* dst = reinterpret_cast<uint32_t*>(dbg_ct + (size_t)task * Hashing<P>::CT);
        for (int w = 0; w < 2 * CTW; ++w) dst[w] = src[w];
      }
      if (win >= 0) {
        const unsigned ordinal = sm.slot_attempt[win] + 1;
        if (uint32_t* ao = g->attempts_out) ao[task] = ordinal;
        if (uint8_t* fo = g->failed_out) fo[task] = 0;
        atomicAdd(&v.g->accepted_sum, (unsigned long long)ordinal);
      } else {
        next += ran;
        if (next > v.max_attempt || a.single_round) {
          win = -2;  // nonce space exhausted (scheduler.hpp:122-128)
          if (uint32_t* ao = g->attempts_out) ao[task] = 0;
          if (uint8_t* fo = g->failed_out) fo[task] = 1;
          atomicAdd(&v.g->failed, 1ull);
        }
      }
      sm.winner[tid] = win;
      keep = win == -1;
      if (!keep) atomicAdd(&sm.bfin[bi], 1u);
      my_u_task = task;
      my_u_next = next;
      my_u_batch = bi;
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
      // copy winners' staged signatures out before the table is overwritten; a failed task's
      // signature is all zero like the reference's (batch.hpp:128-131 leaves the default array)
#pragma unroll 1
      for (unsigned u = warp; u < U; u += kSignWarps) {
        const int win = sm.winner[u];
        // open, or a depth-0 winner that S4 wrote in place
        if (win == -1 || (win == (int)u && !sm.bv[sm.ubatch[u]].stage_out)) continue;
        const uint8_t* src = staging + (size_t)(win < 0 ? 0 : win) * Z::SIG_PAD;
        uint8_t* dst = sm.bv[sm.ubatch[u]].sigs + (size_t)sm.utask[u] * S::SIG;
        // word-granular, coalesced copy to a destination of any alignment (sig_bytes is
        // odd at levels 3/5): the destination may be pinned host memory, where 128-byte
        // write bursts matter
        const unsigned head = (4u - (unsigned)(reinterpret_cast<uintptr_t>(dst) & 3)) & 3u;
        const unsigned nwords = (S::SIG - head) / 4;
        uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + head);
        const unsigned done = head + 4 * nwords;
        if (win < 0) {
          if (lane < (int)head) dst[lane] = 0;
          for (unsigned w = lane; w < nwords; w += 32) d32[w] = 0;
          if (lane < (int)(S::SIG - done)) dst[done + lane] = 0;
          continue;
        }
        if (lane < (int)head) dst[lane] = src[lane];
        const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);  // staging is 16-byte aligned
        for (unsigned w = lane; w < nwords; w += 32)
          d32[w] = head ? __funnelshift_r(s32[w], s32[w + 1], 8 * head) : s32[w];
        if (lane < (int)(S::SIG - done)) dst[done + lane] = src[done + lane];
      }
      __syncthreads();
      if (keep) {
        sm.utask[pos] = my_u_task;
        sm.unext[pos] = my_u_next;
        sm.ubatch[pos] = (uint8_t)my_u_batch;
      }
      // per-batch completion: everything this CTA wrote for the finished tasks is made
      // visible system-wide before `done` moves; whoever completes the batch raises its flag
      if (tid < kRing && sm.bfin[tid]) {
        const unsigned f = sm.bfin[tid];
        sm.bfin[tid] = 0;
        sm.bcnt[tid] -= f;
        const BatchView& v = sm.bv[tid];
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        atomicMin(&v.g->t_first_exit, now);
        __threadfence_system();
        const unsigned old = atomicAdd(&v.g->done, f);
        if (old + f == v.n) {
          atomicMax(&v.g->t_last_exit, now);
          __threadfence_system();
          *v.g->host_flag = v.ticket1;
        }
      }
      if (tid == 0) {
        if (a.trace) {  // RoundTrace of this CTA's round (scheduler.hpp:21-28)
          const unsigned long long idx = atomicAdd(&a.log->trace_count, 1ull);
          if (idx < a.trace_cap) {
            uint4* rec = reinterpret_cast<uint4*>(a.trace + idx * 8);
            rec[0] = make_uint4(blockIdx.x, sm.rounds - 1u, U, sm.r_on);
            rec[1] = make_uint4(sm.r_spec, a.slots > sm.r_on ? a.slots - sm.r_on : 0u, U - total, a.ticket);
          }
        }
        sm.U = total;
      }
      __syncthreads();
    }
  }
}

// ---- host side ---------------------------------------------------------------------
//
// Submission and completion are separate (dlb_sign_submit / dlb_sign_wait); the synchronous
// entry points are submit + wait.  A submission enqueues its inputs, the descriptor body and
// the gate word that publishes the batch on the publication stream, and the batch's own scheduler
// kernel on a stream lane.  Per-key precomputation: a shared key comes from the cross-call cache
// (a miss runs the two one-warp-CTA kernels once); key tables and per-task keys are expanded by
// the scheduler CTAs themselves (SignBatch::prep_*), because no other kernel can become resident
// beside a scheduler grid: 4 CTAs x 128 threads x 128 registers fill the register file.

namespace {

// Stream lane (and scratch set) for the scheduler kernel of a ticket: the lowest lane whose last
// kernel has finished -- synchronous callers only ever touch lane 0 -- else round robin.
inline int pick_lane(dlb_ctx* c, unsigned ticket) {
  for (int l = 0; l < kLanes; ++l)
    if (!c->lane_used[l] || cudaEventQuery(c->lane_done[l]) == cudaSuccess) return l;
  return (int)(ticket % kLanes);
}

int sign_state_init(dlb_ctx* c) {
  if (c->sign_ready) return 0;
  DLB_CUDA_CHECK(cudaMalloc(&c->d_ring, kRing * sizeof(SignBatch)));
  DLB_CUDA_CHECK(cudaMemset(c->d_ring, 0, kRing * sizeof(SignBatch)));
  DLB_CUDA_CHECK(cudaMalloc(&c->d_log, sizeof(SignLog)));
  DLB_CUDA_CHECK(cudaMemset(c->d_log, 0, sizeof(SignLog)));
  DLB_CUDA_CHECK(cudaHostAlloc(&c->h_ring, kRing * sizeof(SignBatch), cudaHostAllocDefault));
  memset(c->h_ring, 0, kRing * sizeof(SignBatch));
  DLB_CUDA_CHECK(cudaHostAlloc(&c->h_flags, kRing * sizeof(unsigned), cudaHostAllocMapped));
  memset((void*)c->h_flags, 0, kRing * sizeof(unsigned));
  DLB_CUDA_CHECK(cudaHostGetDevicePointer((void**)&c->d_flags, (void*)c->h_flags, 0));
  for (int l = 0; l < kLanes; ++l)
    DLB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->sign_lane[l], cudaStreamNonBlocking));
  for (int l = 0; l < kLanes; ++l)
    DLB_CUDA_CHECK(cudaEventCreateWithFlags(&c->lane_done[l], cudaEventDisableTiming));
  DLB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->sign_pub, cudaStreamNonBlocking));
  DLB_CUDA_CHECK(cudaEventCreateWithFlags(&c->sign_pubd, cudaEventDisableTiming));
  for (int r = 0; r < kRing; ++r) {
    DLB_CUDA_CHECK(cudaEventCreate(&c->sign_evs[r]));
    DLB_CUDA_CHECK(cudaEventCreate(&c->sign_ev0[r]));
    DLB_CUDA_CHECK(cudaEventCreate(&c->sign_ev1[r]));
    DLB_CUDA_CHECK(cudaEventCreateWithFlags(&c->sign_cpy[r], cudaEventDisableTiming));
  }
  DLB_CUDA_CHECK(cudaEventCreateWithFlags(&c->sign_dep, cudaEventDisableTiming));
  c->sign_ready = true;
  return 0;
}

template <class P, bool DBG>
int sign_kernel_config(dlb_ctx* c, int* occ_out, size_t* smem_out) {
  static_assert(sizeof(SignSmem<P>) <= 56 * 1024, "four CTAs per SM");
  const int li = level_index(P::LEVEL) * 2 + (DBG ? 1 : 0);
  if (!c->sign_occ[li]) {
    const size_t smem_bytes = sizeof(SignSmem<P>) + c->knob_sign_pad_smem;
    DLB_CUDA_CHECK(cudaFuncSetAttribute(k_sign_persistent<P, DBG>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
    int occ = 0;
    DLB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sign_persistent<P, DBG>,
                                                                 kSignThreads, smem_bytes));
    // Registers are per SM sub-partition: four resident CTAs (16 warps x 120 registers) leave
    // 1,024 registers in each -- no room for a single warp of any Keccak kernel, so the
    // precompute kernels of the NEXT batch could not start before CTAs of this one exit.  Three
    // resident CTAs per SM cost ~1 % of the scheduler's throughput (occupancy is not its
    // limiter, profiles/r01_summary.md section 3) and leave a quarter of every SM to them.
    if (c->knob_sign_occ && occ > (int)c->knob_sign_occ) occ = (int)c->knob_sign_occ;
    c->sign_occ[li] = occ < 1 ? 1 : occ;
    c->sign_smem[li] = smem_bytes;
    // One L1 / shared-memory split for the scheduler kernel and the precompute kernels that must
    // run beside its resident grid: a kernel preferring another split waits until the SM has
    // drained (profiles/r01_summary.md, negative results), which would delay the publication of
    // the next batch to the tail of this one.  Smallest split that holds the resident CTAs.
    const size_t need = (size_t)c->sign_occ[li] * (smem_bytes + 1024);
    int pct = (int)((need * 100 + 228 * 1024 - 1) / (228 * 1024));
    if (pct > 100) pct = 100;
    c->sign_carveout[li] = pct;
    prefer_carveout(k_sign_persistent<P, DBG>, pct);
    prefer_carveout(k_expand_a<P, 1>, pct);
    prefer_carveout(k_sign_unpack<P, 1>, pct);
  }
  *occ_out = c->sign_occ[li];
  *smem_out = c->sign_smem[li];
  return 0;
}

// eta range check of the packed secret vectors (packing.hpp:79-86) on the host
template <class P>
bool sk_eta_ok(const uint8_t* sk) {
  const uint8_t* p = sk + Sizes<P>::SK_S1;
  const size_t fields = (size_t)(P::K + P::L) * kN;
  uint64_t acc = 0;
  unsigned nbits = 0;
  size_t seen = 0;
  while (seen < fields) {
    acc |= (uint64_t)(*p++) << nbits;
    nbits += 8;
    while (nbits >= (unsigned)P::ETA_BITS && seen < fields) {
      if ((acc & ((1u << P::ETA_BITS) - 1)) > 2u * P::ETA) return false;
      acc >>= P::ETA_BITS;
      nbits -= P::ETA_BITS;
      ++seen;
    }
  }
  return true;
}

inline uint64_t fnv1a(const uint8_t* p, size_t n) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

// Finds or builds the cache entry of a shared key (host bytes hk, device copy dsk); the per-key
// kernels of a miss run on `st`.
// Returns nullptr when the cache is off or full of entries that batches in flight may use.
template <class P>
KeyCacheEntry* key_cache_get(dlb_ctx* c, const uint8_t* hk, const uint8_t* dsk, cudaStream_t st, int* rc) {
  using S = Sizes<P>;
  constexpr int KL = P::K * P::L, PV = P::L + 2 * P::K;
  *rc = 0;
  if (!c->knob_key_cache) return nullptr;
  const uint64_t h = fnv1a(hk, S::SK);
  for (auto& e : c->key_cache)
    if (e.level == P::LEVEL && e.hash == h && memcmp(e.sk.data(), hk, S::SK) == 0) {
      e.last_use = ++c->key_cache_clock;
      ++c->key_cache_hits;
      cudaStreamWaitEvent(st, e.ready, 0);
      return &e;
    }
  ++c->key_cache_misses;
  KeyCacheEntry* e = nullptr;
  if (c->key_cache.size() < c->knob_key_cache) {
    c->key_cache.emplace_back();
    e = &c->key_cache.back();
  } else {
    for (int r = 0; r < kRing; ++r)
      if (c->tickets[r].active) return nullptr;  // an entry may be in use: sign uncached this time
    for (auto& x : c->key_cache)
      if (!e || x.last_use < e->last_use) e = &x;
  }
  if (!e->A) {  // entries are sized for the largest parameter set and reused across levels
    constexpr size_t kMaxKL = 8 * 7, kMaxPV = 7 + 2 * 8;
    if (cudaMalloc(&e->A, kMaxKL * kN * 4) != cudaSuccess || cudaMalloc(&e->shat, kMaxPV * kN * 4) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ready, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      if (e->A) cudaFree(e->A);
      if (e->shat) cudaFree(e->shat);
      c->key_cache.pop_back();
      *rc = DLB_E_NOMEM;
      return nullptr;
    }
  }
  e->level = P::LEVEL;
  e->hash = h;
  e->sk.assign(hk, hk + S::SK);
  e->last_use = ++c->key_cache_clock;
  unsigned* bad;
  *rc = dalloc(c, "s.kbad", 1, &bad);
  if (*rc != 0) return nullptr;
  k_expand_a<P, 1><<<cdiv(KL, 32), 32, 0, st>>>(dsk, 0, (unsigned)KL, e->A);
  k_sign_unpack<P, 1><<<(unsigned)PV, 32, 0, st>>>(1u, dsk, 0, e->shat, bad);  // range already checked
  cudaEventRecord(e->ready, st);
  c->launches += 2;
  return e;
}

}  // namespace

// Everything that publishes a batch (input copies, descriptor, the kernels of a key-cache miss,
// gate) goes through one publication stream that never holds a scheduler kernel, so it cannot
// queue up behind a running one; the scheduler kernel of the ticket then goes to its lane.
int sign_reserve(dlb_ctx* c, unsigned* ticket, cudaStream_t* pub) {
  DLB_TRY(sign_state_init(c));
  const unsigned t = c->next_ticket;
  if (c->tickets[t % kRing].active) return DLB_E_BUSY;  // kRing batches in flight: wait for the oldest first
  // The ring slot of a completed ticket may be rewritten while scheduler CTAs that once served it
  // are still resident: their view of the slot is tagged with the old ticket, and a claim is a
  // compare-and-swap against the slot's (ticket + 1 : next task) word, so it can only succeed
  // against the batch the view was loaded for.
  *ticket = t;
  *pub = c->sign_pub;
  cudaStream_t* lane = pub;
  int set = 0;
  while (set < kRing - 1 && c->set_busy[set]) ++set;  // at most kRing - 1 others are in flight
  c->cur_set = set;
  // inputs produced on the caller's stream (the *_dev entry points) are ordered before the lane's work
  DLB_CUDA_CHECK(cudaEventRecord(c->sign_dep, c->s()));
  DLB_CUDA_CHECK(cudaStreamWaitEvent(*lane, c->sign_dep, 0));
  return 0;
}

template <class P, bool DBG>
static int sign_submit_t(dlb_ctx* c, unsigned ticket, const SignIo& io) {
  using S = Sizes<P>;
  using Z = SignSizes<P>;
  constexpr int KL = P::K * P::L, PV = P::L + 2 * P::K;
  const size_t n = io.n;
  if (n == 0 || n > 0x7fffffffu) return DLB_E_ARG;
  if (io.d_key_idx && (io.n_keys == 0 || io.sk_stride == 0)) return DLB_E_ARG;
  const int slot = (int)(ticket % kRing), ln = pick_lane(c, ticket);
  cudaStream_t st = c->sign_pub, lane = c->sign_lane[ln];
  // distinct keys to precompute: the key table, one key per task, or one shared key
  const size_t nk = io.d_key_idx ? io.n_keys : (io.sk_stride ? n : 1);

  PhaseProf prof(c->knob_submit_prof);
  int32_t *A = nullptr, *shat = nullptr;
  uint64_t *mu, *rp;
  // a shared key is looked up in (or added to) the cross-call cache: a hit needs no per-key kernels
  bool cached = false;
  if (nk == 1 && !io.single_round) {
    std::vector<uint8_t> tmp;
    const uint8_t* hk = io.h_sks;
    if (!hk && c->knob_key_cache) {  // device-resident key: fetch its bytes for the lookup
      tmp.resize(S::SK);
      DLB_CUDA_CHECK(cudaMemcpyAsync(tmp.data(), io.d_sks, S::SK, cudaMemcpyDeviceToHost, c->s()));
      DLB_CUDA_CHECK(cudaStreamSynchronize(c->s()));
      hk = tmp.data();
    }
    if (hk) {
      if (!sk_eta_ok<P>(hk)) return DLB_E_KEY;  // packing.hpp:79-86: nothing is signed
      int rc = 0;
      if (KeyCacheEntry* e = key_cache_get<P>(c, hk, io.d_sks, st, &rc)) {
        A = e->A;
        shat = e->shat;
        cached = true;
      } else if (rc != 0) {
        return rc;
      }
    }
  }
  if (!cached) {
    DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "s.A"), nk * KL * kN, &A));
    DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "s.shat"), nk * PV * kN, &shat));
  }
  DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "s.mu"), n * 8, &mu));
  DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "s.rp"), n * 8, &rp));

  // grid: resident CTAs of the persistent kernel
  int occ = 0;
  size_t smem_bytes = 0;
  prof.mark(" arenas");
  DLB_TRY((sign_kernel_config<P, DBG>(c, &occ, &smem_bytes)));
  prof.mark(" config");
  const size_t grid_max = (size_t)c->sm_count * occ;
  // Psi = resident attempt slots (BatchConfig::psi).  Default (measured, profiles/
  // r01_summary.md): nine slots per task -- the speculation depth cap plus one -- while that
  // fits one warp's worth of slots per CTA (batches up to ~2,000 tasks: latency is what
  // matters there and the unluckiest task should advance nine nonces per round), about three
  // per task up to the machine's capacity, every resident slot beyond.  A Psi below the
  // machine's capacity is spread over as many CTAs as there are tasks (up to the resident
  // maximum), each using fewer of its 128 slots: the warp-per-slot stages of a round then
  // take proportionally less time.
  size_t want_slots = io.psi;
  if (!want_slots) {
    if (!io.speculate) want_slots = n;
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
  if (io.single_round) {
    slots_per = kSignThreads;
    tcap = kSignThreads;
    grid = (n + kSignThreads - 1) / kSignThreads;
  }

  // ---- descriptor body (everything but the gate), then the precomputation it points at
  SignBatch& h = c->h_ring[slot];
  memset(&h, 0, sizeof h);
  h.n = (unsigned)n;
  h.tcap = (unsigned)tcap;
  h.max_attempt = (65535u - (P::L - 1)) / P::L;
  if (c->dbg_max_attempt && c->dbg_max_attempt < h.max_attempt) h.max_attempt = c->dbg_max_attempt;
  // Deepest speculative attempt a task may run in one round.  Filling every idle slot
  // (the reference's pass 2) wastes work once few tasks remain: attempt d is only needed
  // with probability (1-p)^d.  Measured on B200 (profiles/r01_summary.md): cap 8 gives the
  // best batch-10k latency and batch-100k throughput; speculate > 1 sets the cap explicitly.
  h.spec_depth = io.single_round || !io.speculate ? 0u
                 : (io.speculate > 1 ? (unsigned)io.speculate : c->knob_spec_depth);
  h.key_stride = io.sk_stride ? 1u : 0u;
  h.level = P::LEVEL;
  h.exclusive = (io.single_round || DBG) ? 1u : 0u;
  h.ticket1 = ticket + 1u;
  h.head = (unsigned long long)(ticket + 1u) << 32;  // queue word: ticket + 1 : next unclaimed task
  h.mu = io.d_mu_in ? io.d_mu_in : mu;
  h.rho_prime = io.d_rho_prime ? reinterpret_cast<const uint64_t*>(io.d_rho_prime) : rp;
  h.kappa0 = io.d_kappa0;
  h.A = A;
  h.shat = shat;
  h.key_idx = io.d_key_idx;
  h.sigs = io.d_sigs;
  h.attempts_out = io.d_attempts;
  h.failed_out = io.d_failed;
  h.dbg_ctilde = io.d_dbg_ct;
  h.dbg_stage = io.d_dbg_stage;
  for (int i = 0; i < 3; ++i) h.bounds[i] = io.bounds[i];
  if (!io.d_mu_in) {  // digests are computed by the scheduler when it claims a task
    h.sk_base = io.d_sks;
    h.msgs = io.d_msgs;
    h.msg_off = io.d_msg_off;
    if (Hashing<P>::MLDSA) DLB_TRY(mldsa_prefix(c, st, &h.pfx, &h.plen));
    h.mu_w = mu;
    h.rp_w = io.d_rho_prime ? nullptr : rp;
  }
  h.host_flag = c->d_flags + slot;
  h.stage_out = io.host_out && c->knob_host_stage ? 1u : 0u;
  if (!cached) {
    h.prep_sks = io.d_sks;
    h.prep_stride = (unsigned)io.sk_stride;
    h.prep_n = (unsigned)nk;
    h.prep_q = (unsigned long long)(ticket + 1u) << 32;
  }
  h.t_first_start = h.t_first_exit = ~0ull;
  h.gate = ticket + 1u;
  SignBatch* g = c->d_ring + slot;
  c->h_flags[slot] = 0;
  cudaEventRecord(c->sign_evs[slot], st);
  DLB_CUDA_CHECK(cudaMemcpyAsync(g, &h, offsetof(SignBatch, gate), cudaMemcpyHostToDevice, st));

  prof.mark(" body copy");
  // per-key precomputation (scheme.hpp:106-125), unless the shared key came from the cache: done
  // by the scheduler CTAs themselves (prep_* in the descriptor), nothing to launch
  prof.mark(" prep launches");
  // publish: running scheduler kernels of earlier tickets may start claiming tasks now
  DLB_CUDA_CHECK(cudaMemcpyAsync(&g->gate, &h.gate, sizeof(unsigned), cudaMemcpyHostToDevice, st));

  prof.mark(" gate copy");
  SignArgs a;
  memset(&a, 0, sizeof a);
  a.ring = c->d_ring;
  a.ticket = ticket;
  a.window = h.exclusive ? 1u : (unsigned)kRing;
  a.slots = (unsigned)slots_per;
  a.single_round = io.single_round;
  a.boost_thr = io.single_round ? 0u : c->knob_boost_thr;
  a.boost_depth = c->knob_boost_depth ? c->knob_boost_depth : 1u;
  a.log = c->d_log;
  if (c->trace_cap && !io.single_round) {
    DLB_TRY(dalloc(c, "s.trace", c->trace_cap * 8, &a.trace));
    a.trace_cap = (unsigned)(c->trace_cap > 0xFFFFFFFFu ? 0xFFFFFFFFu : c->trace_cap);
  }
  if (c->alog_cap && !io.single_round) {
    DLB_TRY(dalloc(c, "s.alog", c->alog_cap * 4, &a.alog));
    a.alog_cap = (unsigned)(c->alog_cap > 0xFFFFFFFFu ? 0xFFFFFFFFu : c->alog_cap);
  }
  if (a.trace || a.alog) DLB_CUDA_CHECK(cudaMemsetAsync(c->d_log, 0, sizeof(SignLog), st));
  // One scratch set per lane, sized for the full resident grid so it never moves under a
  // running kernel of the same lane.  All lanes are sized together: growing an arena frees the
  // old one, which waits for every kernel on the device, so a lane left at a smaller parameter
  // set's size would stall a later submission in the middle of a flow (which lane a ticket gets
  // depends on when earlier kernels retire).  This way the first ticket of a larger set pays once.
  const size_t slots = grid_max * kSignThreads;
  for (int l = 0; l < kLanes; ++l) {
    uint8_t* yb;
    int32_t* wb;
    uint8_t *w1b, *stg;
    int8_t* c8b;
    uint64_t* ctb;
    DLB_TRY(dalloc(c, c->lane_name(l, "s.y"), slots * Z::Y_SLOT + 16, &yb));
    DLB_TRY(dalloc(c, c->lane_name(l, "s.w"), slots * Z::W_SLOT, &wb));
    DLB_TRY(dalloc(c, c->lane_name(l, "s.w1"), slots * S::W1_ALL, &w1b));
    DLB_TRY(dalloc(c, c->lane_name(l, "s.ct"), slots * Hashing<P>::CTW, &ctb));
    DLB_TRY(dalloc(c, c->lane_name(l, "s.c8"), slots * kN, &c8b));
    DLB_TRY(dalloc(c, c->lane_name(l, "s.stage"), slots * Z::SIG_PAD, &stg));
    if (l == ln) {
      a.ybytes = yb;
      a.wbuf = wb;
      a.w1buf = w1b;
      a.ctbuf = ctb;
      a.c8buf = c8b;
      a.staging = stg;
    }
  }
  prof.mark(" scratch");
  DLB_CUDA_CHECK(cudaEventRecord(c->sign_pubd, st));
  DLB_CUDA_CHECK(cudaStreamWaitEvent(lane, c->sign_pubd, 0));
  cudaEventRecord(c->sign_ev0[slot], lane);
  k_sign_persistent<P, DBG><<<(unsigned)grid, kSignThreads, smem_bytes, lane>>>(a);
  cudaEventRecord(c->sign_ev1[slot], lane);
  cudaEventRecord(c->lane_done[ln], lane);
  c->lane_used[ln] = true;
  c->launches += 1;
  DLB_LAUNCH_CHECK();
  prof.mark(" launch");

  SignTicket& tk = c->tickets[slot];
  tk = SignTicket{};
  tk.active = true;
  tk.ticket = ticket;
  tk.level = P::LEVEL;
  tk.n = n;
  tk.sig_bytes = S::SIG;
  tk.had_trace = a.trace != nullptr;
  tk.had_alog = a.alog != nullptr;
  tk.set = c->cur_set;
  c->set_busy[tk.set] = true;
  c->next_ticket = ticket + 1u;
  return 0;
}

template <class P>
int sign_submit(dlb_ctx* c, unsigned ticket, const SignIo& io) {
  return io.dbg_bounds ? sign_submit_t<P, true>(c, ticket, io) : sign_submit_t<P, false>(c, ticket, io);
}

// Queues the device -> host copies of a completed batch's results (those not written in place)
// on the copy-out stream; sign_cpy[slot] follows them.
static int sign_copy_out(dlb_ctx* c, int slot) {
  SignTicket& tk = c->tickets[slot];
  if (tk.copy_issued) return 0;
  cudaStream_t co = c->copy_out;
  if (tk.h_sigs) DLB_CUDA_CHECK(cudaMemcpyAsync(tk.h_sigs, tk.d_sigs, tk.n * tk.sig_bytes, cudaMemcpyDeviceToHost, co));
  if (tk.h_att) DLB_CUDA_CHECK(cudaMemcpyAsync(tk.h_att, tk.d_att, tk.n * 4, cudaMemcpyDeviceToHost, co));
  if (tk.h_failed) DLB_CUDA_CHECK(cudaMemcpyAsync(tk.h_failed, tk.d_failed, tk.n, cudaMemcpyDeviceToHost, co));
  DLB_CUDA_CHECK(cudaEventRecord(c->sign_cpy[slot], co));
  tk.copy_issued = true;
  return 0;
}

// Blocks until the batch of `ticket` is complete (its flag in mapped host memory), then
// fetches its counters.  drain = also wait for the batch's own scheduler kernel to exit
// (the synchronous entry points: kernel time is reported and nothing is left running).
int sign_wait(dlb_ctx* c, unsigned ticket, dlb_sign_stats* stats, bool drain) {
  const int slot = (int)(ticket % kRing);
  SignTicket& tk = c->tickets[slot];
  if (!c->sign_ready || !tk.active || tk.ticket != ticket) return DLB_E_ARG;
  struct Release {  // the ticket and its arena set are free again however the wait ends
    dlb_ctx* c;
    SignTicket& tk;
    ~Release() {
      tk.active = false;
      c->set_busy[tk.set] = false;
    }
  } release{c, tk};
  volatile unsigned* flag = c->h_flags + slot;
  unsigned spins = 0;
  while (*flag != ticket + 1u) {
    if ((++spins & 0x3FF) == 0) {
      // safety net: if every lane has drained and the flag is still down, something faulted
      bool idle = true;
      for (int l = 0; l <= kLanes && idle; ++l) {
        const cudaError_t e = cudaStreamQuery(l < kLanes ? c->sign_lane[l] : c->sign_pub);
        if (e == cudaErrorNotReady) idle = false;
        else if (e != cudaSuccess) return -1000 - (int)e;
      }
      if (idle && *flag != ticket + 1u) {
        SignBatch hq;  // what the device thinks of the batch, for the bug report
        if (cudaMemcpy(&hq, c->d_ring + slot, sizeof hq, cudaMemcpyDeviceToHost) == cudaSuccess)
          fprintf(stderr, "dilithium-b200: ticket %u never completed: n %u queue %u:%u done %u gate %u failed %llu\n",
                  ticket, hq.n, (unsigned)(hq.head >> 32), (unsigned)hq.head, hq.done, hq.gate, hq.failed);
        return DLB_E_INTERNAL;
      }
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  if (drain) {
    DLB_CUDA_CHECK(cudaEventSynchronize(c->sign_ev1[slot]));
    cudaEventElapsedTime(&c->last_main_ms, c->sign_ev0[slot], c->sign_ev1[slot]);
    cudaEventSynchronize(c->sign_evs[slot]);
    cudaEventElapsedTime(&c->last_ms, c->sign_evs[slot], c->sign_ev1[slot]);
  }
  SignBatch hq;
  DLB_TRY(sign_copy_out(c, slot));
  // Other batches that have completed meanwhile: queue their result copies behind this one now, so
  // the copy engine works through them while the caller handles this batch (only when the copies
  // are asynchronous; a pageable destination would block here).
  for (unsigned k = 1; k < (unsigned)kRing; ++k) {
    const int s2 = (int)((ticket + k) % kRing);
    const SignTicket& t2 = c->tickets[s2];
    if (t2.active && t2.host_pinned && !t2.copy_issued && c->h_flags[s2] == t2.ticket + 1u)
      DLB_TRY(sign_copy_out(c, s2));
  }
  DLB_CUDA_CHECK(cudaEventSynchronize(c->sign_cpy[slot]));
  DLB_CUDA_CHECK(cudaMemcpyAsync(&hq, c->d_ring + slot, sizeof hq, cudaMemcpyDeviceToHost, c->copy_stats));
  SignLog hl{};
  if (tk.had_trace || tk.had_alog)
    DLB_CUDA_CHECK(cudaMemcpyAsync(&hl, c->d_log, sizeof hl, cudaMemcpyDeviceToHost, c->copy_stats));
  DLB_CUDA_CHECK(cudaStreamSynchronize(c->copy_stats));
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
  if (tk.had_trace) c->trace_count = hl.trace_count;
  if (tk.had_alog) c->alog_count = hl.alog_count;
  if (hq.key_bad) {  // no signature is produced for a malformed key (scheme.hpp:271)
    if (tk.zero_host) memset(tk.zero_host, 0, tk.n * tk.sig_bytes);
    if (tk.zero_dev) cudaMemset(tk.zero_dev, 0, tk.n * tk.sig_bytes);
    return DLB_E_KEY;
  }
  return 0;
}

#define DLB_INST(LV) template int sign_submit<Params<LV>>(dlb_ctx*, unsigned, const SignIo&);
DLB_INST(2)
DLB_INST(3)
DLB_INST(5)
DLB_INST(44)
DLB_INST(65)
DLB_INST(87)

}  // namespace dlb

using namespace dlb;

// sign_attempt<P> (scheme.hpp:225-230) / detail::sign_attempt_bounded<P> (:133-219) for n
// independent (key, mu, rho', kappa) tuples: one scheduler round with one attempt per task; z
// and hints are decoded back from the staged signature.  bounds == nullptr runs the production
// kernel; otherwise the DBG instantiation with the three norm bounds injected, which also
// reports the reject stage in the reference's check order.
static int dbg_sign_attempt(dlb_ctx* c, int level, size_t n, const uint8_t* sks, size_t sk_stride,
                            const uint8_t* mus, const uint8_t* rho_primes, const uint32_t* kappas,
                            const int32_t* bounds, uint8_t* accepted, uint8_t* stage, uint8_t* c_tilde,
                            int32_t* z, int32_t* hints) {
  if (!c || !sks || !mus || !rho_primes || !kappas || !accepted || !c_tilde || !z || !hints)
    return DLB_E_ARG;
  if (n == 0) return 0;
  // chknorm refuses bounds above (q-1)/8 (rounding.hpp:65); the device check has the same domain
  if (bounds)
    for (int i = 0; i < 3; ++i)
      if (bounds[i] < 0 || bounds[i] > (kQ - 1) / 8) return DLB_E_ARG;
  cudaSetDevice(c->device);
  auto run = [&](auto p) -> int {
    using P = decltype(p);
    using S = Sizes<P>;
    const size_t nk = sk_stride ? n : 1;
    uint8_t *dsk, *dsig, *dfail, *dct, *drp, *dstage;
    uint64_t* dmu;
    uint32_t *dk, *datt;
    DLB_TRY(dalloc(c, "dbg.sk", nk * S::SK, &dsk));
    DLB_TRY(dalloc(c, "dbg.a", n * 8, &dmu));
    DLB_TRY(dalloc(c, "dbg.b", n * 64, &drp));
    DLB_TRY(dalloc(c, "dbg.c", n, &dk));
    DLB_TRY(dalloc(c, "dbg.sig", n * S::SIG + 8, &dsig));
    DLB_TRY(dalloc(c, "dbg.att", n, &datt));
    DLB_TRY(dalloc(c, "dbg.fail", n, &dfail));
    DLB_TRY(dalloc(c, "dbg.d", n * Hashing<P>::CT, &dct));
    DLB_TRY(dalloc(c, "dbg.stage", n, &dstage));
    unsigned t;
    cudaStream_t st;
    DLB_TRY(sign_reserve(c, &t, &st));
    DLB_CUDA_CHECK(cudaMemcpyAsync(dsk, sks, nk * S::SK, cudaMemcpyHostToDevice, st));
    DLB_CUDA_CHECK(cudaMemcpyAsync(dmu, mus, n * 64, cudaMemcpyHostToDevice, st));
    DLB_CUDA_CHECK(cudaMemcpyAsync(drp, rho_primes, n * 64, cudaMemcpyHostToDevice, st));
    DLB_CUDA_CHECK(cudaMemcpyAsync(dk, kappas, n * 4, cudaMemcpyHostToDevice, st));
    DLB_CUDA_CHECK(cudaMemsetAsync(dsig, 0, n * S::SIG, st));
    DLB_CUDA_CHECK(cudaMemsetAsync(dstage, 0xFF, n, st));
    SignIo io;
    io.n = n;
    io.d_sks = dsk;
    io.sk_stride = sk_stride;
    io.d_mu_in = dmu;
    io.d_rho_prime = drp;
    io.d_kappa0 = dk;
    io.speculate = 0;
    io.single_round = 1;
    io.d_sigs = dsig;
    io.d_attempts = datt;
    io.d_failed = dfail;
    io.d_dbg_ct = dct;
    if (bounds) {
      io.dbg_bounds = true;
      io.d_dbg_stage = dstage;
      for (int i = 0; i < 3; ++i) io.bounds[i] = bounds[i];
    }
    const int src = sign_submit<P>(c, t, io);
    if (src != 0) {
      cudaStreamSynchronize(st);
      return src;
    }
    const int wrc = sign_wait(c, t, nullptr, true);
    if (wrc != 0 && wrc != DLB_E_KEY) return wrc;
    uint8_t* hsig = new uint8_t[n * S::SIG];
    uint8_t* hfail = new uint8_t[n];
    cudaMemcpyAsync(hsig, dsig, n * S::SIG, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hfail, dfail, n, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(c_tilde, dct, n * Hashing<P>::CT, cudaMemcpyDeviceToHost, st);
    if (stage) cudaMemcpyAsync(stage, dstage, n, cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
      memset(z, 0, n * P::L * kN * 4);
      memset(hints, 0, n * P::K * kN * 4);
      for (size_t t2 = 0; t2 < n; ++t2) {
        accepted[t2] = hfail[t2] ? 0 : 1;
        if (!accepted[t2]) continue;
        const uint8_t* sg = hsig + t2 * S::SIG;
        for (int j = 0; j < P::L; ++j)
          for (int m = 0; m < kN; ++m) {
            const size_t bit = (size_t)m * P::Z_BITS;
            uint32_t raw = 0;
            for (int b = 0; b < P::Z_BITS; ++b)
              raw |= (uint32_t)((sg[S::SIG_Z + j * S::Z_POLY + ((bit + b) >> 3)] >> ((bit + b) & 7)) & 1) << b;
            z[(t2 * P::L + j) * kN + m] = P::GAMMA1 - (int32_t)raw;
          }
        const uint8_t* h = sg + S::SIG_Z + P::L * S::Z_POLY;
        unsigned prev = 0;
        for (int i = 0; i < P::K; ++i) {
          const unsigned cnt = h[P::OMEGA + i];
          for (unsigned k = prev; k < cnt && k < (unsigned)P::OMEGA; ++k)
            hints[(t2 * P::K + i) * kN + h[k]] = 1;
          prev = cnt;
        }
      }
    }
    delete[] hsig;
    delete[] hfail;
    if (e != cudaSuccess) return -1000 - (int)e;
    return wrc;
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

extern "C" int dlb_dbg_sign_attempt(dlb_ctx* c, int level, size_t n, const uint8_t* sks,
                                    size_t sk_stride, const uint8_t* mus, const uint8_t* rho_primes,
                                    const uint32_t* kappas, uint8_t* accepted, uint8_t* c_tilde,
                                    int32_t* z, int32_t* hints) {
  return dbg_sign_attempt(c, level, n, sks, sk_stride, mus, rho_primes, kappas, nullptr, accepted, nullptr,
                          c_tilde, z, hints);
}

extern "C" int dlb_dbg_sign_attempt_bounded(dlb_ctx* c, int level, size_t n, const uint8_t* sks,
                                            size_t sk_stride, const uint8_t* mus,
                                            const uint8_t* rho_primes, const uint32_t* kappas,
                                            int32_t z_bound, int32_t r0_bound, int32_t vt_bound,
                                            uint8_t* accepted, uint8_t* stage, uint8_t* c_tilde,
                                            int32_t* z, int32_t* hints) {
  if (!stage) return DLB_E_ARG;
  const int32_t bounds[3] = {z_bound, r0_bound, vt_bound};
  return dbg_sign_attempt(c, level, n, sks, sk_stride, mus, rho_primes, kappas, bounds, accepted, stage,
                          c_tilde, z, hints);
}
