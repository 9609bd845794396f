// engine.cuh -- host-side context shared by the translation units of libdilithium_b200.
//
// Plays the role of the reference's MemoryPool + WorkerPool (memory_pool.hpp:25-100,
// thread_pool.hpp) for the GPU: device arenas that are allocated once and grown on
// demand, pinned host staging, streams and events.  Nothing here is per-call.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <map>
#include <string>
#include <vector>

#include "../../include/dilithium_b200.h"
#include "common.cuh"
#include "sign_queue.cuh"

namespace dlb {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
};

// host-side record of a submitted signing batch (ring slot = ticket % kRing)
struct SignTicket {
  bool active = false;
  unsigned ticket = 0;
  int level = 0;
  size_t n = 0, sig_bytes = 0;
  bool had_trace = false, had_alog = false;
  int set = 0;  // arena set held until the wait
  // results still to be copied to the caller at wait time (null = already in place)
  uint8_t* h_sigs = nullptr;
  const uint8_t* d_sigs = nullptr;
  uint32_t* h_att = nullptr;
  const uint32_t* d_att = nullptr;
  uint8_t* h_failed = nullptr;
  const uint8_t* d_failed = nullptr;
  // the caller's signature buffer, cleared when the key turns out malformed
  uint8_t* zero_host = nullptr;
  uint8_t* zero_dev = nullptr;
  bool copy_issued = false;  // the result copies are already queued on copy_out (sign_cpy[slot] follows them)
  bool host_pinned = false;  // the caller's result buffers are page-locked: the copies are asynchronous
};

// Per-key signing state kept across calls (SignPrecomp, scheme.hpp:26-32,106-125): the expanded
// matrix and the transformed secret vectors of a shared key, in device allocations that are never
// rewritten while the entry lives.  A batch signed under a cached key needs no per-key kernels.
struct KeyCacheEntry {
  int level = 0;
  uint64_t hash = 0;
  std::vector<uint8_t> sk;   // the packed key the entry was built from (compared on a hit)
  int32_t* A = nullptr;
  int32_t* shat = nullptr;
  cudaEvent_t ready = nullptr;  // precomputation finished (recorded on the lane that built it)
  unsigned long long last_use = 0;
};

// what a signing submission passes down; device pointers unless noted
struct SignIo {
  size_t n = 0;
  const uint8_t* d_sks = nullptr;
  const uint8_t* h_sks = nullptr;         // nullable: host copy of the keys (shared key: cache lookup)
  size_t sk_stride = 0, n_keys = 0;
  bool host_out = false;  // d_sigs is mapped host memory
  const uint32_t* d_key_idx = nullptr;
  const uint8_t* d_msgs = nullptr;
  const uint64_t* d_msg_off = nullptr;
  const uint64_t* d_mu_in = nullptr;      // stage tests: mu supplied (then d_rho_prime is rho' itself)
  const uint8_t* d_rho_prime = nullptr;   // nullable: n * 64 override
  const uint32_t* d_kappa0 = nullptr;     // stage tests: first nonce per task
  size_t psi = 0;
  int speculate = 1, single_round = 0;
  uint8_t* d_sigs = nullptr;
  uint32_t* d_attempts = nullptr;
  uint8_t* d_failed = nullptr;
  uint8_t* d_dbg_ct = nullptr;
  uint8_t* d_dbg_stage = nullptr;
  bool dbg_bounds = false;                // run the DBG kernel with the bounds below
  int32_t bounds[3] = {0, 0, 0};
};

inline int level_index(int level) {
  switch (level) {
    case 2: return 0;
    case 3: return 1;
    case 5: return 2;
    case 44: return 3;
    case 65: return 4;
    default: return 5;
  }
}

}  // namespace dlb

struct dlb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;      // engine-owned compute stream
  cudaStream_t copy_in = nullptr;     // H2D stream
  cudaStream_t copy_out = nullptr;    // D2H stream
  cudaStream_t copy_stats = nullptr;  // D2H of a finished batch's counters (never behind a bulk copy)
  cudaStream_t ext = nullptr;         // caller's stream for *_dev calls (optional)
  cudaStream_t lane_s[2] = {};        // two compute lanes: consecutive chunks overlap
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};  // chunk pipeline hand-offs
  float last_ms = 0.f, last_main_ms = 0.f;  // whole call / dominant kernel only
  unsigned launches = 0;
  int sm_count = 148;
  size_t max_batch_hint = 0;     // dlb_create's sizing hint: arenas of the first call are sized for it
  size_t trace_cap = 0;          // per-round scheduler trace (dlb_set_trace); 0 = off
  unsigned long long trace_count = 0;  // records the last sign call produced
  // FIPS 204 message prefix 0 || |ctx| || ctx (2..257 bytes) for the ML-DSA levels: host copy
  // and its device mirror; the default is the empty context string
  uint8_t mldsa_pfx[288] = {0, 0};       // + an 11-byte hash OID in the pre-hash variant (HashML-DSA)
  unsigned mldsa_plen = 2;
  uint8_t* d_mldsa_pfx = nullptr;
  bool mldsa_pfx_dirty = true;
  std::map<std::string, dlb::DevBuf> dev;
  std::map<std::string, dlb::HostBuf> pinned;

  // ---- signing scheduler: batches in flight (sign.cu) --------------------------------
  bool sign_ready = false;
  dlb::SignBatch* d_ring = nullptr;      // kRing descriptors in device memory
  dlb::SignBatch* h_ring = nullptr;      // pinned staging of the same
  volatile unsigned* h_flags = nullptr;  // mapped pinned completion flags, one per ring slot
  unsigned* d_flags = nullptr;           // their device alias
  dlb::SignLog* d_log = nullptr;
  cudaStream_t sign_lane[dlb::kLanes] = {};
  cudaEvent_t lane_done[dlb::kLanes] = {};  // last scheduler kernel of the lane finished
  bool lane_used[dlb::kLanes] = {};
  cudaStream_t sign_pub = nullptr;       // publication stream: copies and per-key kernels, never a scheduler kernel
  cudaEvent_t sign_pubd = nullptr;       // batch published (the lane's kernel launch waits for it)
  // per ring slot: start of the batch's device work, start / end of its scheduler kernel
  cudaEvent_t sign_evs[dlb::kRing] = {}, sign_ev0[dlb::kRing] = {}, sign_ev1[dlb::kRing] = {}, sign_cpy[dlb::kRing] = {},
              sign_dep = nullptr;
  dlb::SignTicket tickets[dlb::kRing];
  unsigned next_ticket = 0;
  // input / output / per-batch arenas come in sets; a ticket holds the lowest free set from
  // submission to wait, so a pipeline of depth d only ever touches (and warms) d sets
  bool set_busy[dlb::kRing] = {};
  int cur_set = 0;                       // set reserved for the submission in progress
  int sign_occ[12] = {};                 // resident CTAs per SM of k_sign_persistent<level, DBG>
  size_t sign_smem[12] = {};
  int sign_carveout[12] = {};            // their L1 / shared split (percent of 228 KB)
  size_t alog_cap = 0;                   // executed-attempt log (dlb_set_assignment_log); 0 = off
  unsigned long long alog_count = 0;
  std::vector<dlb::KeyCacheEntry> key_cache;
  unsigned long long key_cache_clock = 0, key_cache_hits = 0, key_cache_misses = 0;
  size_t knob_key_cache = 32;            // entries; 0 disables (DLB_KEY_CACHE)
  bool knob_host_stage = false;          // signatures for a pinned caller buffer leave the kernel as whole rows from
                                         // the staging buffer instead of field by field (DLB_HOST_STAGE)
  size_t knob_zero_copy_max = ~(size_t)0; // signatures go straight into a pinned caller buffer up to this many
                                         // bytes per batch, through device memory + a copy at wait time above
                                         // (DLB_ZERO_COPY_MAX; in place is faster at every size measured,
                                         // profiles/r02_summary.md)
  unsigned dbg_max_attempt = 0;          // stage tests: smaller nonce space (0 = the scheme's)
  // tuning knobs, read from the environment once at dlb_create (profiles/: the sweeps)
  unsigned knob_spec_depth = 8;
  // straggler boost (DLB_BOOST_THR failed attempts, 0 = off; DLB_BOOST_DEPTH extra nonces per round).
  // Off by default: measured 54 -> 42 ms batch latency in a deep pipeline for -0.6 % throughput
  // (profiles/r02_summary.md section 2)
  unsigned knob_boost_thr = 0, knob_boost_depth = 4;
  size_t knob_chunk = 65536;      // keygen / verify device chunk (tasks)
  size_t knob_pipe_chunk = 8192;  // host transfer pipeline chunk (tasks)
  size_t knob_sign_pad_smem = 0;  // occupancy experiments
  int knob_carveout = -1;
  bool knob_submit_prof = false;  // DLB_SUBMIT_PROF: host-side phase times of every submission on stderr
  unsigned knob_sign_occ = 0;     // resident scheduler CTAs per SM (DLB_SIGN_OCC; 0 = what fits)

  cudaStream_t s() const { return ext ? ext : stream; }
  const char* slot_name(int slot, const char* what) {
    snprintf(name_buf, sizeof name_buf, "r%02d.%s", slot, what);
    return name_buf;
  }
  const char* lane_name(int lane, const char* what) {
    snprintf(name_buf, sizeof name_buf, "l%d.%s", lane, what);
    return name_buf;
  }
  char name_buf[48] = {};

  // 256-byte aligned device arena slot (memory_pool.hpp:27 kArenaAlign), grown geometrically
  int dbuf(const char* name, size_t bytes, void** out) {
    dlb::DevBuf& b = dev[name];
    if (b.cap < bytes) {
      if (b.p) {
        cudaStreamSynchronize(s());
        cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
      }
      size_t want = bytes + bytes / 4 + 256;
      cudaError_t e = cudaMalloc(&b.p, want);
      if (e != cudaSuccess) {
        cudaGetLastError();
        e = cudaMalloc(&b.p, bytes + 256);
        if (e != cudaSuccess) {
          cudaGetLastError();
          return DLB_E_NOMEM;
        }
        want = bytes + 256;
      }
      b.cap = want;
    }
    *out = b.p;
    return 0;
  }

  int hbuf(const char* name, size_t bytes, void** out) {
    dlb::HostBuf& b = pinned[name];
    if (b.cap < bytes) {
      if (b.p) cudaFreeHost(b.p);
      b.p = nullptr;
      b.cap = 0;
      const size_t want = bytes + bytes / 4 + 256;
      if (cudaHostAlloc(&b.p, want, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return DLB_E_NOMEM;
      }
      b.cap = want;
    }
    *out = b.p;
    return 0;
  }
};

namespace dlb {

// host-side phase timer for the submission path (DLB_SUBMIT_PROF=1 at dlb_create: prints to stderr)
struct PhaseProf {
  bool on;
  double t0;
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
  }
  explicit PhaseProf(bool enabled) : on(enabled), t0(on ? now() : 0) {}
  void mark(const char* what) {
    if (!on) return;
    const double t = now();
    fprintf(stderr, "[submit] %-16s %.3f ms\n", what, t - t0);
    t0 = t;
  }
};

template <class T>
inline int dalloc(dlb_ctx* c, const char* name, size_t count, T** out) {
  void* p = nullptr;
  const int rc = c->dbuf(name, count * sizeof(T), &p);
  *out = static_cast<T*>(p);
  return rc;
}

inline unsigned cdiv(size_t a, size_t b) { return (unsigned)((a + b - 1) / b); }

// device mirror of the ML-DSA message prefix, refreshed on `st` when the context string changed
inline int mldsa_prefix(dlb_ctx* c, cudaStream_t st, const uint8_t** d_pfx, unsigned* plen) {
  if (!c->d_mldsa_pfx) {
    const int rc = dalloc(c, "mldsa.pfx", sizeof c->mldsa_pfx, &c->d_mldsa_pfx);
    if (rc != 0) return rc;
    c->mldsa_pfx_dirty = true;
  }
  if (c->mldsa_pfx_dirty) {
    if (cudaMemcpyAsync(c->d_mldsa_pfx, c->mldsa_pfx, sizeof c->mldsa_pfx, cudaMemcpyHostToDevice, st) !=
        cudaSuccess)
      return -1000 - (int)cudaGetLastError();
    cudaStreamSynchronize(st);  // the host copy may change again right after this call
    c->mldsa_pfx_dirty = false;
  }
  *d_pfx = c->d_mldsa_pfx;
  *plen = c->mldsa_plen;
  return 0;
}

// One L1 / shared-memory split for every kernel of a pipeline.  The split is a per-SM
// setting that cannot change under resident CTAs: a kernel that prefers another split than
// the one an SM is running waits until that SM (measured: the whole previous grid) has
// drained, which serialises kernels that should overlap -- the chunk lanes of keygen /
// verify, or two engine contexts (scripts/ubench/overlap.cu).  percent = share of the
// 256 KB given to shared memory (cudaSharedmemCarveoutMaxShared = 100).
template <class K>
inline void prefer_carveout(K kernel, int percent) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, percent);
}
inline int pipeline_carveout(const dlb_ctx* c) { return c->knob_carveout; }  // -1: the driver's per-kernel choice

#define DLB_TRY(x)            \
  do {                        \
    const int rc_ = (x);      \
    if (rc_ != 0) return rc_; \
  } while (0)

#define DLB_LAUNCH_CHECK()                                   \
  do {                                                       \
    const cudaError_t e_ = cudaGetLastError();               \
    if (e_ != cudaSuccess) return -1000 - (int)e_;           \
  } while (0)

// per-level device-resident implementations (keygen.cu / verify.cu / sign.cu)
template <class P>
int keygen_dev(dlb_ctx* c, size_t n, const uint8_t* d_zetas, uint8_t* d_pks, uint8_t* d_sks);
// d_key_idx == nullptr: stride 0 = one shared key, else task t uses key t; d_key_idx != nullptr:
// a table of n_keys keys (stride apart), task t uses key d_key_idx[t].
template <class P>
int verify_dev(dlb_ctx* c, size_t n, const uint8_t* d_pks, size_t pk_stride, size_t n_keys,
               const uint32_t* d_key_idx, const uint8_t* d_msgs, const uint64_t* d_msg_off,
               const uint8_t* d_sigs, uint8_t* d_flags, bool keys_expanded = false);
// signing: reserve a ticket (and learn its stream lane, for the caller's input copies), enqueue
// the batch, later wait for it (sign.cu)
int sign_reserve(dlb_ctx* c, unsigned* ticket, cudaStream_t* lane);
template <class P>
int sign_submit(dlb_ctx* c, unsigned ticket, const SignIo& io);
int sign_wait(dlb_ctx* c, unsigned ticket, dlb_sign_stats* stats, bool drain);

}  // namespace dlb
