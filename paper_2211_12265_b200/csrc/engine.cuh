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
#include <map>
#include <string>

#include "../../include/dilithium_b200.h"
#include "common.cuh"

namespace dlb {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
};

}  // namespace dlb

struct dlb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;      // engine-owned compute stream
  cudaStream_t copy_in = nullptr;     // H2D stream
  cudaStream_t copy_out = nullptr;    // D2H stream
  cudaStream_t ext = nullptr;         // caller's stream for *_dev calls (optional)
  cudaStream_t lane_s[2] = {};        // two compute lanes: consecutive chunks overlap
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  cudaEvent_t ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};  // chunk pipeline hand-offs
  float last_ms = 0.f, last_main_ms = 0.f;  // whole call / dominant kernel only
  unsigned launches = 0;
  int sm_count = 148;
  size_t trace_cap = 0;          // per-round scheduler trace (dlb_set_trace); 0 = off
  unsigned long long trace_count = 0;  // records the last sign call produced
  // FIPS 204 message prefix 0 || |ctx| || ctx (2..257 bytes) for the ML-DSA levels: host copy
  // and its device mirror; the default is the empty context string
  uint8_t mldsa_pfx[264] = {0, 0};
  unsigned mldsa_plen = 2;
  uint8_t* d_mldsa_pfx = nullptr;
  bool mldsa_pfx_dirty = true;
  std::map<std::string, dlb::DevBuf> dev;
  std::map<std::string, dlb::HostBuf> pinned;

  cudaStream_t s() const { return ext ? ext : stream; }

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
inline int pipeline_carveout() {
  static const int v = [] {
    const char* e = getenv("DLB_CARVEOUT");  // experiments: -1 leaves the driver's per-kernel choice
    return e ? atoi(e) : -1;
  }();
  return v;
}

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
               const uint8_t* d_sigs, uint8_t* d_flags);
template <class P>
int sign_dev(dlb_ctx* c, size_t n, const uint8_t* d_sks, size_t sk_stride, size_t n_keys,
             const uint32_t* d_key_idx, const uint8_t* d_msgs, const uint64_t* d_msg_off,
             const uint8_t* d_rho_prime, size_t psi, int speculate, uint8_t* d_sigs,
             uint32_t* d_attempts, uint8_t* d_failed, dlb_sign_stats* stats);

}  // namespace dlb
