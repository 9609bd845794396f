// engine.cu -- C ABI (include/dilithium_b200.h): context, host<->device marshalling,
// level dispatch, and the stage-level entry points used by the device parity tests.
#include <sched.h>

#include "engine.cuh"
#include "ntt.cuh"
#include "samplers.cuh"

using namespace dlb;

namespace {

template <class Fn>
int with_level(int level, Fn&& fn) {
  switch (level) {
    case 2: return fn(Params<2>{});
    case 3: return fn(Params<3>{});
    case 5: return fn(Params<5>{});
    case 44: return fn(Params<44>{});  // ML-DSA-44 / 65 / 87 (FIPS 204)
    case 65: return fn(Params<65>{});
    case 87: return fn(Params<87>{});
    default: return DLB_E_LEVEL;
  }
}

struct LevelSizes {
  size_t pk, sk, sig;
  int k, l;
};

bool level_sizes(int level, LevelSizes* o) {
  return with_level(level, [&](auto p) {
           using P = decltype(p);
           *o = {Sizes<P>::PK, Sizes<P>::SK, Sizes<P>::SIG, P::K, P::L};
           return 0;
         }) == 0;
}

struct Timed {
  dlb_ctx* c;
  explicit Timed(dlb_ctx* ctx) : c(ctx) {
    c->launches = 0;
    cudaEventRecord(c->ev0, c->s());
  }
  int finish() {
    cudaEventRecord(c->ev1, c->s());
    const cudaError_t e = cudaStreamSynchronize(c->s());
    if (e != cudaSuccess) return -1000 - (int)e;
    cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1);
    return 0;
  }
};

int h2d(dlb_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return 0;
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->s());
  return e == cudaSuccess ? 0 : -1000 - (int)e;
}

int d2h(dlb_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return 0;
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->s());
  return e == cudaSuccess ? 0 : -1000 - (int)e;
}

int sync(dlb_ctx* c) {
  const cudaError_t e = cudaStreamSynchronize(c->s());
  return e == cudaSuccess ? 0 : -1000 - (int)e;
}

// ---- stage-level kernels (parity tests) ------------------------------------------

__global__ void k_dbg_keccak(unsigned n, uint64_t* states) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint64_t s[25];
#pragma unroll
  for (int i = 0; i < 25; ++i) s[i] = states[(size_t)t * 25 + i];
  keccak_f1600(s);
#pragma unroll
  for (int i = 0; i < 25; ++i) states[(size_t)t * 25 + i] = s[i];
}

__global__ void k_dbg_shake256(unsigned n, const uint8_t* msgs, const uint64_t* off, uint64_t* out) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint64_t s[25];
  keccak_clear(s);
  const uint8_t* m = msgs + off[t];
  const size_t len = (size_t)(off[t + 1] - off[t]);
  const size_t nblocks = len / kRate256 + 1;
  for (size_t blk = 0; blk < nblocks; ++blk) {
#pragma unroll
    for (int w = 0; w < kWords256; ++w) s[w] ^= padded_word(m, len, blk * kRate256 + 8 * w);
    if (blk == nblocks - 1) s[kWords256 - 1] ^= 0x8000000000000000ull;
    keccak_f1600(s);
  }
#pragma unroll
  for (int w = 0; w < 8; ++w) out[(size_t)t * 8 + w] = s[w];
}

template <class P, int WARPS>
__global__ void k_dbg_expand_mask(unsigned n, const uint64_t* rho_primes, const uint32_t* kappas,
                                  uint8_t* ybytes) {
  const unsigned p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n * P::L) return;
  const unsigned a = p / P::L, j = p % P::L;
  expand_mask_stream<P>(rho_primes + (size_t)a * 8, kappas[a] + j,
                        ybytes + (size_t)p * Sizes<P>::Z_POLY);
}

template <class P>
__global__ void k_dbg_unpack_mask(unsigned n_polys, const uint8_t* ybytes, int32_t* out) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_polys * kN) return;
  const unsigned p = i / kN, cidx = i % kN;
  out[i] = P::GAMMA1 - (int32_t)load_bits(ybytes + (size_t)p * Sizes<P>::Z_POLY,
                                           cidx * P::Z_BITS, P::Z_BITS);
}

__global__ void k_dbg_ntt(unsigned n, int32_t* polys, int inverse) {
  __shared__ __align__(16) int2 zs[256], nzs[256];
  __shared__ __align__(16) int32_t tiles[4][kTileWords];
  load_twiddles(zs, nzs);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned t = blockIdx.x * 4 + warp;
  if (t >= n) return;
  int32_t* a = polys + (size_t)t * kN;
  int32_t r[8];
  if (!inverse) {
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = a[lane + 32 * i];
    ntt_fwd(r, tiles[warp], zs, lane);
#pragma unroll
    for (int m = 0; m < 8; ++m) a[8 * lane + m] = freeze(r[m]);
  } else {
    // the inverse carries an extra factor R (see ntt.cuh); undo it for the value test
#pragma unroll
    for (int m = 0; m < 8; ++m) r[m] = inverse == 2 ? a[8 * lane + m] : center(a[8 * lane + m]);
    ntt_inv(r, tiles[warp], nzs, lane);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[lane + 32 * i] = freeze(mont_mul(r[i], 1));
  }
}

// rounding.hpp:13-59 on the device, one value per thread: Power2Round, Decompose and
// UseHint with hint 0 / 1, for the exhaustive value test over [0, q)
template <int GAMMA2>
__global__ void k_dbg_rounding(unsigned n, int32_t first, int32_t* p2r_hi, int32_t* p2r_lo,
                               int32_t* dec_hi, int32_t* dec_lo, int32_t* use0, int32_t* use1) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t a = first + (int32_t)i;
  power2round(a, p2r_hi[i], p2r_lo[i]);
  dec_hi[i] = decompose<GAMMA2>(a, dec_lo[i]);
  use0[i] = use_hint<GAMMA2>(0, a);
  use1[i] = use_hint<GAMMA2>(1, a);
}

}  // namespace

extern "C" {

const char* dlb_version(void) { return "dilithium-b200 0.1 (sm_100a)"; }

static int create_resources(dlb_ctx* c) {
  DLB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  DLB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy_in, cudaStreamNonBlocking));
  DLB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking));
  DLB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy_stats, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) {
    DLB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->lane_s[b], cudaStreamNonBlocking));
    DLB_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_join[b], cudaEventDisableTiming));
  }
  DLB_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  DLB_CUDA_CHECK(cudaEventCreate(&c->ev0));
  DLB_CUDA_CHECK(cudaEventCreate(&c->ev1));
  for (int b = 0; b < 2; ++b) {
    DLB_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_in[b], cudaEventDisableTiming));
    DLB_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_comp[b], cudaEventDisableTiming));
    DLB_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_out[b], cudaEventDisableTiming));
  }
  return 0;
}

int dlb_create(dlb_ctx** out, int device, size_t max_batch) {
  if (!out) return DLB_E_ARG;
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess) return -1000 - (int)e;
  if (device < 0 || device >= count) return DLB_E_ARG;
  DLB_CUDA_CHECK(cudaSetDevice(device));
  dlb_ctx* c = new dlb_ctx();
  c->device = device;
  c->max_batch_hint = max_batch;
  // tuning knobs for the sweeps recorded in profiles/: read once, here
  if (const char* v = getenv("DLB_SPEC_DEPTH")) c->knob_spec_depth = (unsigned)atoi(v);
  if (const char* v = getenv("DLB_CHUNK")) c->knob_chunk = (size_t)atol(v);
  if (const char* v = getenv("DLB_PIPE_CHUNK")) c->knob_pipe_chunk = (size_t)atol(v);
  if (const char* v = getenv("DLB_SIGN_PAD_SMEM")) c->knob_sign_pad_smem = (size_t)atol(v);
  if (const char* v = getenv("DLB_CARVEOUT")) c->knob_carveout = atoi(v);
  if (const char* v = getenv("DLB_BOOST_THR")) c->knob_boost_thr = (unsigned)atoi(v);
  if (const char* v = getenv("DLB_BOOST_DEPTH")) c->knob_boost_depth = (unsigned)atoi(v);
  if (c->knob_boost_depth < 1 || c->knob_boost_depth > 8) c->knob_boost_depth = 4;
  if (const char* v = getenv("DLB_SIGN_OCC")) c->knob_sign_occ = (unsigned)atoi(v);
  c->knob_submit_prof = getenv("DLB_SUBMIT_PROF") != nullptr;
  if (const char* v = getenv("DLB_KEY_CACHE")) c->knob_key_cache = (size_t)atol(v);
  if (const char* v = getenv("DLB_HOST_STAGE")) c->knob_host_stage = atoi(v) != 0;
  if (const char* v = getenv("DLB_ZERO_COPY_MAX")) c->knob_zero_copy_max = (size_t)atoll(v);
  const int rc = create_resources(c);
  if (rc != 0) {
    dlb_destroy(c);  // tolerates the handles that were never created
    return rc;
  }
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  // max_batch > 0: the caller knows its batch size -- build the signing state (ring, lanes, flags)
  // and the size-dependent I/O arenas of the first arena set now instead of inside the first call
  if (max_batch) {
    unsigned t;
    cudaStream_t pub;
    int rc2 = sign_reserve(c, &t, &pub);  // creates the state; the ticket itself is not consumed
    void* p = nullptr;
    if (rc2 == 0) rc2 = c->dbuf(c->slot_name(0, "io.off"), (max_batch + 1) * 8, &p);
    if (rc2 == 0) rc2 = c->dbuf(c->slot_name(0, "io.att"), max_batch * 4, &p);
    if (rc2 == 0) rc2 = c->dbuf(c->slot_name(0, "io.fail"), max_batch, &p);
    if (rc2 == 0) rc2 = c->dbuf(c->slot_name(0, "s.mu"), max_batch * 64, &p);
    if (rc2 == 0) rc2 = c->dbuf(c->slot_name(0, "s.rp"), max_batch * 64, &p);
    if (rc2 != 0) {
      dlb_destroy(c);
      return rc2;
    }
  }
  *out = c;
  return 0;
}

void dlb_destroy(dlb_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  // secret material (keys, their transforms, rho', masks) lives in these arenas: wipe before release
  for (auto& kv : c->dev)
    if (kv.second.p) {
      cudaMemset(kv.second.p, 0, kv.second.cap);
      cudaFree(kv.second.p);
    }
  for (auto& kv : c->pinned)
    if (kv.second.p) {
      memset(kv.second.p, 0, kv.second.cap);
      cudaFreeHost(kv.second.p);
    }
  for (auto& e : c->key_cache) {
    if (e.A) {
      cudaMemset(e.A, 0, 8 * 7 * kN * 4);
      cudaFree(e.A);
    }
    if (e.shat) {
      cudaMemset(e.shat, 0, (7 + 2 * 8) * kN * 4);
      cudaFree(e.shat);
    }
    if (e.ready) cudaEventDestroy(e.ready);
    if (!e.sk.empty()) memset(e.sk.data(), 0, e.sk.size());
  }
  if (c->sign_ready) {
    cudaFree(c->d_ring);
    cudaFree(c->d_log);
    cudaFreeHost(c->h_ring);
    cudaFreeHost((void*)c->h_flags);
    for (int l = 0; l < kLanes; ++l) {
      if (c->sign_lane[l]) cudaStreamDestroy(c->sign_lane[l]);
      if (c->lane_done[l]) cudaEventDestroy(c->lane_done[l]);
    }
    for (int r = 0; r < kRing; ++r) {
      if (c->sign_evs[r]) cudaEventDestroy(c->sign_evs[r]);
      if (c->sign_ev0[r]) cudaEventDestroy(c->sign_ev0[r]);
      if (c->sign_ev1[r]) cudaEventDestroy(c->sign_ev1[r]);
      if (c->sign_cpy[r]) cudaEventDestroy(c->sign_cpy[r]);
    }
    if (c->sign_dep) cudaEventDestroy(c->sign_dep);
    if (c->sign_pubd) cudaEventDestroy(c->sign_pubd);
    if (c->sign_pub) cudaStreamDestroy(c->sign_pub);
  }
  auto ev = [](cudaEvent_t e) {
    if (e) cudaEventDestroy(e);
  };
  auto st = [](cudaStream_t s) {
    if (s) cudaStreamDestroy(s);
  };
  ev(c->ev0);
  ev(c->ev1);
  for (int b = 0; b < 2; ++b) {
    ev(c->ev_in[b]);
    ev(c->ev_comp[b]);
    ev(c->ev_out[b]);
    ev(c->ev_join[b]);
    st(c->lane_s[b]);
  }
  ev(c->ev_fork);
  st(c->stream);
  st(c->copy_in);
  st(c->copy_out);
  st(c->copy_stats);
  delete c;
}

float dlb_last_kernel_ms(const dlb_ctx* c) { return c ? c->last_ms : 0.f; }
float dlb_last_main_kernel_ms(const dlb_ctx* c) { return c ? c->last_main_ms : 0.f; }
unsigned dlb_last_launches(const dlb_ctx* c) { return c ? c->launches : 0; }

int dlb_set_stream(dlb_ctx* c, void* cuda_stream) {
  if (!c) return DLB_E_ARG;
  c->ext = static_cast<cudaStream_t>(cuda_stream);
  return 0;
}

int dlb_set_trace(dlb_ctx* c, size_t cap) {
  if (!c || cap > (1u << 26)) return DLB_E_ARG;
  c->trace_cap = cap;
  c->trace_count = 0;
  return 0;
}

long long dlb_get_trace(dlb_ctx* c, dlb_round_trace* out, size_t max_records) {
  if (!c) return DLB_E_ARG;
  const unsigned long long have = c->trace_count < c->trace_cap ? c->trace_count : c->trace_cap;
  const size_t ncopy = have < max_records ? (size_t)have : max_records;
  if (ncopy && out) {
    auto it = c->dev.find("s.trace");
    if (it == c->dev.end() || !it->second.p) return DLB_E_ARG;
    cudaSetDevice(c->device);
    const cudaError_t e = cudaMemcpy(out, it->second.p, ncopy * sizeof(dlb_round_trace), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return -1000 - (int)e;
  }
  return (long long)c->trace_count;
}

int dlb_set_mldsa_context(dlb_ctx* c, const uint8_t* ctx_bytes, size_t len) {
  if (!c || len > 255 || (len && !ctx_bytes)) return DLB_E_ARG;  // FIPS 204: |ctx| <= 255
  for (int r = 0; r < kRing; ++r)  // batches in flight hash their tasks with the current string
    if (c->tickets[r].active) return DLB_E_BUSY;
  c->mldsa_pfx[0] = 0;
  c->mldsa_pfx[1] = (uint8_t)len;
  if (len) memcpy(c->mldsa_pfx + 2, ctx_bytes, len);
  c->mldsa_plen = 2 + (unsigned)len;
  c->mldsa_pfx_dirty = true;
  return 0;
}

int dlb_set_mldsa_prehash(dlb_ctx* c, const uint8_t* ctx_bytes, size_t len, const uint8_t* oid, size_t oid_len) {
  if (!c || len > 255 || (len && !ctx_bytes) || oid_len > 16 || (oid_len && !oid)) return DLB_E_ARG;
  if (oid_len == 0) return dlb_set_mldsa_context(c, ctx_bytes, len);
  for (int r = 0; r < kRing; ++r)
    if (c->tickets[r].active) return DLB_E_BUSY;
  c->mldsa_pfx[0] = 1;  // FIPS 204 Alg. 4 / 5: M' = 1 || |ctx| || ctx || OID || PH(M)
  c->mldsa_pfx[1] = (uint8_t)len;
  if (len) memcpy(c->mldsa_pfx + 2, ctx_bytes, len);
  memcpy(c->mldsa_pfx + 2 + len, oid, oid_len);
  c->mldsa_plen = 2 + (unsigned)len + (unsigned)oid_len;
  c->mldsa_pfx_dirty = true;
  return 0;
}

namespace {

// "/sys/bus/pci/devices/<domain:bus:dev.fn>/<leaf>" of a CUDA device, first line
bool pci_sysfs_line(int device, const char* leaf, char* out, size_t cap) {
  char id[32] = {};
  if (cudaDeviceGetPCIBusId(id, sizeof id, device) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  for (char* p = id; *p; ++p)
    if (*p >= 'A' && *p <= 'Z') *p = (char)(*p - 'A' + 'a');
  char path[128];
  snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/%s", id, leaf);
  FILE* f = fopen(path, "r");
  if (!f) return false;
  const bool ok = fgets(out, (int)cap, f) != nullptr;
  fclose(f);
  return ok;
}

}  // namespace

int dlb_device_numa_node(int device) {
  char line[64];
  if (!pci_sysfs_line(device, "numa_node", line, sizeof line)) return -1;
  return atoi(line);
}

int dlb_bind_thread_to_device(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return DLB_E_ARG;
  }
  if (device < 0 || device >= count) return DLB_E_ARG;
  char line[4096];
  if (!pci_sysfs_line(device, "local_cpulist", line, sizeof line)) return 1;
  cpu_set_t set;
  CPU_ZERO(&set);
  int n_set = 0;
  for (char* p = line; *p && *p != '\n';) {  // "0-15,32-47"
    char* end;
    const long a = strtol(p, &end, 10);
    if (end == p) break;
    long b = a;
    p = end;
    if (*p == '-') {
      b = strtol(p + 1, &end, 10);
      p = end;
    }
    for (long cpu = a; cpu <= b && cpu < CPU_SETSIZE; ++cpu) {
      CPU_SET((int)cpu, &set);
      ++n_set;
    }
    if (*p == ',') ++p;
  }
  if (n_set == 0) return 1;
  if (sched_setaffinity(0, sizeof set, &set) != 0) return 1;  // e.g. a cgroup that excludes those CPUs
  return 0;
}

void* dlb_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void dlb_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

// ---- device-resident ---------------------------------------------------------------

int dlb_keygen_batch_dev(dlb_ctx* c, int level, size_t n, const uint8_t* d_zetas, uint8_t* d_pks,
                         uint8_t* d_sks) {
  if (!c || (n && (!d_zetas || !d_pks || !d_sks))) return DLB_E_ARG;
  cudaSetDevice(c->device);
  Timed tm(c);
  DLB_TRY(with_level(level, [&](auto p) {
    return keygen_dev<decltype(p)>(c, n, d_zetas, d_pks, d_sks);
  }));
  return tm.finish();
}

int dlb_verify_batch_keyed_dev(dlb_ctx* c, int level, size_t n_keys, const uint8_t* d_pks, size_t n,
                               const uint32_t* d_key_idx, const uint8_t* d_msgs,
                               const uint64_t* d_msg_off, const uint8_t* d_sigs, uint8_t* d_flags) {
  LevelSizes ls;
  if (!c || (n && (!d_pks || !d_msg_off || !d_sigs || !d_flags || !d_key_idx || !n_keys))) return DLB_E_ARG;
  if (!level_sizes(level, &ls)) return DLB_E_LEVEL;
  cudaSetDevice(c->device);
  Timed tm(c);
  DLB_TRY(with_level(level, [&](auto p) {
    return verify_dev<decltype(p)>(c, n, d_pks, ls.pk, n_keys, d_key_idx, d_msgs, d_msg_off, d_sigs,
                                   d_flags);
  }));
  return tm.finish();
}

int dlb_verify_batch_dev(dlb_ctx* c, int level, size_t n, const uint8_t* d_pks, size_t pk_stride,
                         const uint8_t* d_msgs, const uint64_t* d_msg_off, const uint8_t* d_sigs,
                         uint8_t* d_flags) {
  if (!c || (n && (!d_pks || !d_msg_off || !d_sigs || !d_flags))) return DLB_E_ARG;
  cudaSetDevice(c->device);
  Timed tm(c);
  DLB_TRY(with_level(level, [&](auto p) {
    return verify_dev<decltype(p)>(c, n, d_pks, pk_stride, 0, nullptr, d_msgs, d_msg_off, d_sigs,
                                   d_flags);
  }));
  return tm.finish();
}

namespace {

// ticket handed to callers: internal ticket + 1; 0 = an empty batch (nothing to wait for)
int sign_submit_dev(dlb_ctx* c, int level, size_t n_keys, const uint8_t* d_sks, size_t sk_stride, size_t n,
                    const uint32_t* d_key_idx, const uint8_t* d_msgs, const uint64_t* d_msg_off,
                    const uint8_t* d_rho_prime, size_t psi, int speculate, uint8_t* d_sigs,
                    uint32_t* d_attempts, uint8_t* d_failed, uint64_t* ticket_out) {
  LevelSizes ls;
  if (!c || !ticket_out) return DLB_E_ARG;
  if (!level_sizes(level, &ls)) return DLB_E_LEVEL;
  *ticket_out = 0;
  if (n == 0) return 0;
  if (!d_sks || !d_msg_off || !d_sigs) return DLB_E_ARG;
  if (sk_stride != 0 && sk_stride != ls.sk) return DLB_E_ARG;
  cudaSetDevice(c->device);
  unsigned t;
  cudaStream_t st;
  DLB_TRY(sign_reserve(c, &t, &st));
  SignIo io;
  io.n = n;
  io.d_sks = d_sks;
  io.sk_stride = sk_stride;
  io.n_keys = n_keys;
  io.d_key_idx = d_key_idx;
  io.d_msgs = d_msgs;
  io.d_msg_off = d_msg_off;
  io.d_rho_prime = d_rho_prime;
  io.psi = psi;
  io.speculate = speculate;
  io.d_sigs = d_sigs;
  io.d_attempts = d_attempts;
  io.d_failed = d_failed;
  c->launches = 0;
  DLB_TRY(with_level(level, [&](auto p) { return sign_submit<decltype(p)>(c, t, io); }));
  c->tickets[t % kRing].zero_dev = d_sigs;
  *ticket_out = (uint64_t)t + 1;
  return 0;
}

int sign_wait_ticket(dlb_ctx* c, uint64_t ticket, dlb_sign_stats* stats, bool drain) {
  if (!c) return DLB_E_ARG;
  if (stats) memset(stats, 0, sizeof *stats);
  if (ticket == 0) return 0;
  cudaSetDevice(c->device);
  return sign_wait(c, (unsigned)(ticket - 1), stats, drain);
}

}  // namespace

int dlb_sign_submit_dev(dlb_ctx* c, int level, size_t n_keys, const uint8_t* d_sks, size_t sk_stride,
                        size_t n, const uint32_t* d_key_idx, const uint8_t* d_msgs,
                        const uint64_t* d_msg_off, const uint8_t* d_rho_prime, size_t psi, int speculate,
                        uint8_t* d_sigs, uint32_t* d_attempts, uint8_t* d_failed, uint64_t* ticket) {
  if (n && d_key_idx && !n_keys) return DLB_E_ARG;
  return sign_submit_dev(c, level, n_keys, d_sks, sk_stride, n, d_key_idx, d_msgs, d_msg_off, d_rho_prime,
                         psi, speculate, d_sigs, d_attempts, d_failed, ticket);
}

int dlb_sign_wait(dlb_ctx* c, uint64_t ticket, dlb_sign_stats* stats) {
  return sign_wait_ticket(c, ticket, stats, false);
}

int dlb_sign_batch_keyed_dev(dlb_ctx* c, int level, size_t n_keys, const uint8_t* d_sks, size_t n,
                             const uint32_t* d_key_idx, const uint8_t* d_msgs,
                             const uint64_t* d_msg_off, const uint8_t* d_rho_prime, size_t psi,
                             int speculate, uint8_t* d_sigs, uint32_t* d_attempts, uint8_t* d_failed,
                             dlb_sign_stats* stats) {
  LevelSizes ls;
  if (!c || (n && (!d_key_idx || !n_keys))) return DLB_E_ARG;
  if (!level_sizes(level, &ls)) return DLB_E_LEVEL;
  uint64_t t = 0;
  DLB_TRY(sign_submit_dev(c, level, n_keys, d_sks, ls.sk, n, d_key_idx, d_msgs, d_msg_off, d_rho_prime, psi,
                          speculate, d_sigs, d_attempts, d_failed, &t));
  return sign_wait_ticket(c, t, stats, true);
}

int dlb_sign_batch_dev(dlb_ctx* c, int level, size_t n, const uint8_t* d_sks, size_t sk_stride,
                       const uint8_t* d_msgs, const uint64_t* d_msg_off,
                       const uint8_t* d_rho_prime, size_t psi, int speculate, uint8_t* d_sigs,
                       uint32_t* d_attempts, uint8_t* d_failed, dlb_sign_stats* stats) {
  uint64_t t = 0;
  DLB_TRY(sign_submit_dev(c, level, 0, d_sks, sk_stride, n, nullptr, d_msgs, d_msg_off, d_rho_prime, psi,
                          speculate, d_sigs, d_attempts, d_failed, &t));
  return sign_wait_ticket(c, t, stats, true);
}

// ---- host-buffer API -----------------------------------------------------------------
//
// Transfers are hidden behind compute (the paper's multi-stream scheme):
//   keygen / verify  the batch is cut into chunks that flow through three streams --
//                    H2D of chunk c+1, kernels of chunk c and D2H of chunk c-1 run
//                    concurrently on double-buffered device arenas;
//   sign             one persistent kernel covers the whole batch; when the caller's
//                    signature buffer is pinned (dlb_host_alloc / cudaHostAlloc) the
//                    commit step stores finished signatures straight into it over PCIe
//                    while other tasks are still in the rejection loop, so no D2H copy
//                    remains after the kernel.  Pageable buffers fall back to one
//                    cudaMemcpy from a device arena.

namespace {

// (pipeline chunk cap: dlb_ctx::knob_pipe_chunk, 8192 tasks -- measured: finer chunks hide more of the PCIe time, +3 % at 100k)

// transfer/compute pipeline granularity: at least four chunks per batch so small batches
// (the batch-10k latency case) overlap their copies too
inline size_t pipe_chunk(const dlb_ctx* ctx, size_t n) {
  size_t c = (n + 3) / 4;
  if (c < 2048) c = 2048;
  const size_t cmax = ctx->knob_pipe_chunk;  // DLB_PIPE_CHUNK at dlb_create
  if (c > cmax) c = cmax;
  return c < n ? c : n;
}

// On an early error return of a host pipeline, copies and kernels that reference the caller's
// buffers may still be in flight on the engine's streams: drain them before the call returns.
struct DrainOnError {
  dlb_ctx* c;
  bool ok = false;
  explicit DrainOnError(dlb_ctx* ctx) : c(ctx) {}
  ~DrainOnError() {
    if (ok) return;
    cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->copy_in);
    cudaStreamSynchronize(c->copy_out);
    cudaGetLastError();
  }
};

struct OwnStream {  // host-buffer calls always run on the engine's own streams
  dlb_ctx* c;
  cudaStream_t saved;
  explicit OwnStream(dlb_ctx* ctx) : c(ctx), saved(ctx->ext) { c->ext = nullptr; }
  ~OwnStream() { c->ext = saved; }
};

// device-visible alias of a pinned host pointer, or nullptr for pageable memory
void* pinned_alias(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (at.type == cudaMemoryTypeHost && at.devicePointer) return at.devicePointer;
  return nullptr;
}

#define DLB_CU(x)                                  \
  do {                                             \
    const cudaError_t e_ = (x);                    \
    if (e_ != cudaSuccess) return -1000 - (int)e_; \
  } while (0)

}  // namespace

int dlb_keygen_batch(dlb_ctx* c, int level, size_t n, const uint8_t* zetas, uint8_t* pks,
                     uint8_t* sks) {
  LevelSizes ls;
  if (!c) return DLB_E_ARG;
  if (!level_sizes(level, &ls)) return DLB_E_LEVEL;
  if (n == 0) return 0;
  if (!zetas || !pks || !sks) return DLB_E_ARG;
  cudaSetDevice(c->device);
  OwnStream own(c);
  DrainOnError drain(c);
  cudaStream_t S = c->stream, CO = c->copy_out;
  const size_t chunk = pipe_chunk(c, n);
  uint8_t *dz, *dpk[2], *dsk[2];
  DLB_TRY(dalloc(c, "io.zeta", n * 32, &dz));
  DLB_TRY(dalloc(c, "io.pk0", chunk * ls.pk, &dpk[0]));
  DLB_TRY(dalloc(c, "io.pk1", chunk * ls.pk, &dpk[1]));
  DLB_TRY(dalloc(c, "io.sk0", chunk * ls.sk, &dsk[0]));
  DLB_TRY(dalloc(c, "io.sk1", chunk * ls.sk, &dsk[1]));
  c->launches = 0;
  DLB_CU(cudaEventRecord(c->ev0, S));
  DLB_CU(cudaMemcpyAsync(dz, zetas, n * 32, cudaMemcpyHostToDevice, S));
  size_t ci = 0;
  for (size_t lo = 0; lo < n; lo += chunk, ++ci) {
    const size_t cnt = n - lo < chunk ? n - lo : chunk;
    const int b = (int)(ci & 1);
    if (ci >= 2) DLB_CU(cudaStreamWaitEvent(S, c->ev_out[b], 0));  // arena b drained
    DLB_TRY(with_level(level, [&](auto p) {
      return keygen_dev<decltype(p)>(c, cnt, dz + lo * 32, dpk[b], dsk[b]);
    }));
    DLB_CU(cudaEventRecord(c->ev_comp[b], S));
    DLB_CU(cudaStreamWaitEvent(CO, c->ev_comp[b], 0));
    DLB_CU(cudaMemcpyAsync(pks + lo * ls.pk, dpk[b], cnt * ls.pk, cudaMemcpyDeviceToHost, CO));
    DLB_CU(cudaMemcpyAsync(sks + lo * ls.sk, dsk[b], cnt * ls.sk, cudaMemcpyDeviceToHost, CO));
    DLB_CU(cudaEventRecord(c->ev_out[b], CO));
  }
  DLB_CU(cudaEventRecord(c->ev1, S));
  DLB_CU(cudaStreamSynchronize(CO));
  DLB_CU(cudaStreamSynchronize(S));
  cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1);
  drain.ok = true;
  return 0;
}

namespace {

// range check of a key-index array (host side: an out-of-range index would read past the table)
bool key_idx_ok(const uint32_t* key_idx, size_t n, size_t n_keys) {
  for (size_t i = 0; i < n; ++i)
    if (key_idx[i] >= n_keys) return false;
  return true;
}

// offsets must be non-decreasing (task i uses msgs[off[i] .. off[i+1])) and msgs non-null when any byte is used
bool msg_off_ok(const uint8_t* msgs, const uint64_t* msg_off, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (msg_off[i + 1] < msg_off[i]) return false;
  return msg_off[n] == msg_off[0] || msgs != nullptr;
}

int verify_host(dlb_ctx* c, int level, size_t n, const uint8_t* pks, size_t pk_stride, size_t n_keys,
                const uint32_t* key_idx, const uint8_t* msgs, const uint64_t* msg_off,
                const uint8_t* sigs, uint8_t* flags) {
  LevelSizes ls;
  if (!c) return DLB_E_ARG;
  if (!level_sizes(level, &ls)) return DLB_E_LEVEL;
  if (n == 0) return 0;
  if (!pks || !msg_off || !sigs || !flags) return DLB_E_ARG;
  if (pk_stride != 0 && pk_stride != ls.pk) return DLB_E_ARG;
  if (key_idx && (n_keys == 0 || pk_stride == 0 || !key_idx_ok(key_idx, n, n_keys))) return DLB_E_ARG;
  if (msg_off[0] != 0 || !msg_off_ok(msgs, msg_off, n)) return DLB_E_ARG;
  cudaSetDevice(c->device);
  OwnStream own(c);
  DrainOnError drain(c);
  cudaStream_t S = c->stream, CI = c->copy_in;
  const size_t mbytes = msg_off[n];
  const size_t chunk = pipe_chunk(c, n);
  const bool keyed = key_idx != nullptr;
  const size_t pk_cap = keyed ? n_keys : (pk_stride ? chunk : 1);
  uint8_t *dpk[2], *dm, *dsig[2], *dfl;
  uint64_t* doff;
  uint32_t* dkidx = nullptr;
  if (keyed) DLB_TRY(dalloc(c, "io.kidx", n, &dkidx));
  DLB_TRY(dalloc(c, "io.pk0", pk_cap * ls.pk, &dpk[0]));
  DLB_TRY(dalloc(c, "io.pk1", pk_cap * ls.pk, &dpk[1]));
  DLB_TRY(dalloc(c, "io.msg", mbytes + 8, &dm));
  DLB_TRY(dalloc(c, "io.off", n + 1, &doff));
  DLB_TRY(dalloc(c, "io.sig0", chunk * ls.sig + 8, &dsig[0]));
  DLB_TRY(dalloc(c, "io.sig1", chunk * ls.sig + 8, &dsig[1]));
  DLB_TRY(dalloc(c, "io.flag", n, &dfl));
  c->launches = 0;
  DLB_CU(cudaEventRecord(c->ev0, S));
  if (mbytes) DLB_CU(cudaMemcpyAsync(dm, msgs, mbytes, cudaMemcpyHostToDevice, CI));
  DLB_CU(cudaMemcpyAsync(doff, msg_off, (n + 1) * 8, cudaMemcpyHostToDevice, CI));
  if (keyed) {
    DLB_CU(cudaMemcpyAsync(dpk[0], pks, n_keys * ls.pk, cudaMemcpyHostToDevice, CI));
    DLB_CU(cudaMemcpyAsync(dkidx, key_idx, n * 4, cudaMemcpyHostToDevice, CI));
  } else if (!pk_stride) {
    DLB_CU(cudaMemcpyAsync(dpk[0], pks, ls.pk, cudaMemcpyHostToDevice, CI));
  }
  size_t ci = 0;
  for (size_t lo = 0; lo < n; lo += chunk, ++ci) {
    const size_t cnt = n - lo < chunk ? n - lo : chunk;
    const int b = (int)(ci & 1);
    if (ci >= 2) DLB_CU(cudaStreamWaitEvent(CI, c->ev_comp[b], 0));  // arena b consumed
    DLB_CU(cudaMemcpyAsync(dsig[b], sigs + lo * ls.sig, cnt * ls.sig, cudaMemcpyHostToDevice, CI));
    if (pk_stride && !keyed)
      DLB_CU(cudaMemcpyAsync(dpk[b], pks + lo * ls.pk, cnt * ls.pk, cudaMemcpyHostToDevice, CI));
    DLB_CU(cudaEventRecord(c->ev_in[b], CI));
    DLB_CU(cudaStreamWaitEvent(S, c->ev_in[b], 0));
    DLB_TRY(with_level(level, [&](auto p) {
      // a shared key or a key table is expanded by the first chunk only (every distinct key once)
      return verify_dev<decltype(p)>(c, cnt, (pk_stride && !keyed) ? dpk[b] : dpk[0], pk_stride, n_keys,
                                     keyed ? dkidx + lo : nullptr, dm, doff + lo, dsig[b], dfl + lo,
                                     ci > 0 && (keyed || !pk_stride));
    }));
    DLB_CU(cudaEventRecord(c->ev_comp[b], S));
  }
  DLB_CU(cudaMemcpyAsync(flags, dfl, n, cudaMemcpyDeviceToHost, S));
  DLB_CU(cudaEventRecord(c->ev1, S));
  DLB_CU(cudaStreamSynchronize(S));
  cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1);
  drain.ok = true;
  return 0;
}

}  // namespace

int dlb_verify_batch(dlb_ctx* c, int level, size_t n, const uint8_t* pks, size_t pk_stride,
                     const uint8_t* msgs, const uint64_t* msg_off, const uint8_t* sigs,
                     uint8_t* flags) {
  return verify_host(c, level, n, pks, pk_stride, 0, nullptr, msgs, msg_off, sigs, flags);
}

int dlb_verify_batch_keyed(dlb_ctx* c, int level, size_t n_keys, const uint8_t* pks, size_t n,
                           const uint32_t* key_idx, const uint8_t* msgs, const uint64_t* msg_off,
                           const uint8_t* sigs, uint8_t* flags) {
  LevelSizes ls;
  if (!level_sizes(level, &ls)) return DLB_E_LEVEL;
  if (n && !key_idx) return DLB_E_ARG;
  return verify_host(c, level, n, pks, ls.pk, n_keys, key_idx, msgs, msg_off, sigs, flags);
}

namespace {

int sign_host_submit(dlb_ctx* c, int level, size_t n, const uint8_t* sks, size_t sk_stride, size_t n_keys,
                     const uint32_t* key_idx, const uint8_t* msgs, const uint64_t* msg_off,
                     const uint8_t* rho_prime, size_t psi, int speculate, uint8_t* sigs,
                     uint32_t* attempts, uint8_t* failed, uint64_t* ticket_out) {
  LevelSizes ls;
  if (!c || !ticket_out) return DLB_E_ARG;
  if (!level_sizes(level, &ls)) return DLB_E_LEVEL;
  *ticket_out = 0;
  if (n == 0) return 0;
  if (!sks || !msg_off || !sigs) return DLB_E_ARG;
  if (sk_stride != 0 && sk_stride != ls.sk) return DLB_E_ARG;
  if (key_idx && (n_keys == 0 || sk_stride == 0 || !key_idx_ok(key_idx, n, n_keys))) return DLB_E_ARG;
  if (msg_off[0] != 0 || !msg_off_ok(msgs, msg_off, n)) return DLB_E_ARG;
  cudaSetDevice(c->device);
  OwnStream own(c);
  PhaseProf prof(c->knob_submit_prof);
  unsigned t;
  cudaStream_t S;
  DLB_TRY(sign_reserve(c, &t, &S));
  prof.mark("reserve");
  const int slot = (int)(t % kRing);
  const size_t mbytes = msg_off[n];
  const size_t nk = key_idx ? n_keys : (sk_stride ? n : 1);
  uint8_t *dsk, *dm, *dsig, *dfail, *drp = nullptr;
  uint64_t* doff;
  uint32_t *datt, *dkidx = nullptr;
  if (key_idx) DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "io.kidx"), n, &dkidx));
  // Pinned result buffer: signatures are written in place by the kernel's commit step (no copy to
  // wait for).  DLB_ZERO_COPY_MAX sends batches above a size through device memory and a copy at
  // wait time instead; measured slower at every size (profiles/r02_summary.md), so off by default.
  uint8_t* const pinned_sigs = static_cast<uint8_t*>(pinned_alias(sigs));
  uint8_t* zero_copy = n * ls.sig <= c->knob_zero_copy_max ? pinned_sigs : nullptr;
  DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "io.sk"), nk * ls.sk, &dsk));
  DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "io.msg"), mbytes + 8, &dm));
  DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "io.off"), n + 1, &doff));
  if (!zero_copy) DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "io.sig"), n * ls.sig + 8, &dsig));
  else dsig = zero_copy;
  DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "io.att"), n, &datt));
  DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "io.fail"), n, &dfail));
  // Inputs go up with truly asynchronous copies: pageable memory is first copied into this ring
  // slot's pinned staging (a pageable cudaMemcpyAsync would wait for the lane's previous kernel
  // and stall the submitting thread); pinned caller buffers are used where they lie.
  auto upload = [&](const char* what, void* dst, const void* src, size_t bytes) -> int {
    if (!bytes) return 0;
    if (!pinned_alias(src)) {
      void* stage = nullptr;
      DLB_TRY(c->hbuf(c->slot_name(c->cur_set, what), bytes, &stage));
      memcpy(stage, src, bytes);
      src = stage;
    }
    DLB_CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S));
    return 0;
  };
  prof.mark("arenas");
  DLB_TRY(upload("h.sk", dsk, sks, nk * ls.sk));
  DLB_TRY(upload("h.msg", dm, msgs, mbytes));
  // the digest kernels read whole aligned words around the last message bytes (and mask them)
  DLB_CU(cudaMemsetAsync(dm + mbytes, 0, 8, S));
  DLB_TRY(upload("h.off", doff, msg_off, (n + 1) * 8));
  if (key_idx) DLB_TRY(upload("h.kidx", dkidx, key_idx, n * 4));
  if (rho_prime) {
    DLB_TRY(dalloc(c, c->slot_name(c->cur_set, "io.rp"), n * 64, &drp));
    DLB_TRY(upload("h.rp", drp, rho_prime, n * 64));
  }
  prof.mark("uploads");
  SignIo io;
  io.n = n;
  io.d_sks = dsk;
  io.h_sks = sks;
  io.sk_stride = sk_stride;
  io.n_keys = n_keys;
  io.d_key_idx = dkidx;
  io.d_msgs = dm;
  io.d_msg_off = doff;
  io.d_rho_prime = drp;
  io.psi = psi;
  io.speculate = speculate;
  io.d_sigs = dsig;
  io.host_out = zero_copy != nullptr;
  io.d_attempts = datt;
  io.d_failed = dfail;
  c->launches = 0;
  const int rc = with_level(level, [&](auto p) { return sign_submit<decltype(p)>(c, t, io); });
  prof.mark("sign_submit");
  if (rc != 0) {
    cudaStreamSynchronize(S);  // copies in flight read the caller's buffers
    return rc;
  }
  SignTicket& tk = c->tickets[slot];
  if (!zero_copy) {
    tk.h_sigs = sigs;
    tk.d_sigs = dsig;
  }
  if (attempts) {
    tk.h_att = attempts;
    tk.d_att = datt;
  }
  if (failed) {
    tk.h_failed = failed;
    tk.d_failed = dfail;
  }
  tk.zero_host = sigs;
  tk.host_pinned = pinned_sigs && (!attempts || pinned_alias(attempts)) && (!failed || pinned_alias(failed));
  *ticket_out = (uint64_t)t + 1;
  return 0;
}

}  // namespace

int dlb_sign_submit(dlb_ctx* c, int level, size_t n_keys, const uint8_t* sks, size_t sk_stride, size_t n,
                    const uint32_t* key_idx, const uint8_t* msgs, const uint64_t* msg_off,
                    const uint8_t* rho_prime, size_t psi, int speculate, uint8_t* sigs,
                    uint32_t* attempts, uint8_t* failed, uint64_t* ticket) {
  return sign_host_submit(c, level, n, sks, sk_stride, n_keys, key_idx, msgs, msg_off, rho_prime, psi,
                          speculate, sigs, attempts, failed, ticket);
}

int dlb_sign_batch(dlb_ctx* c, int level, size_t n, const uint8_t* sks, size_t sk_stride,
                   const uint8_t* msgs, const uint64_t* msg_off, const uint8_t* rho_prime,
                   size_t psi, int speculate, uint8_t* sigs, uint32_t* attempts, uint8_t* failed,
                   dlb_sign_stats* stats) {
  if (stats) memset(stats, 0, sizeof *stats);
  uint64_t t = 0;
  DLB_TRY(sign_host_submit(c, level, n, sks, sk_stride, 0, nullptr, msgs, msg_off, rho_prime, psi, speculate,
                           sigs, attempts, failed, &t));
  return sign_wait_ticket(c, t, stats, true);
}

int dlb_sign_batch_keyed(dlb_ctx* c, int level, size_t n_keys, const uint8_t* sks, size_t n,
                         const uint32_t* key_idx, const uint8_t* msgs, const uint64_t* msg_off,
                         const uint8_t* rho_prime, size_t psi, int speculate, uint8_t* sigs,
                         uint32_t* attempts, uint8_t* failed, dlb_sign_stats* stats) {
  LevelSizes ls;
  if (!level_sizes(level, &ls)) return DLB_E_LEVEL;
  if (n && !key_idx) return DLB_E_ARG;
  if (stats) memset(stats, 0, sizeof *stats);
  uint64_t t = 0;
  DLB_TRY(sign_host_submit(c, level, n, sks, ls.sk, n_keys, key_idx, msgs, msg_off, rho_prime, psi, speculate,
                           sigs, attempts, failed, &t));
  return sign_wait_ticket(c, t, stats, true);
}

int dlb_set_assignment_log(dlb_ctx* c, size_t cap) {
  if (!c || cap > (1u << 26)) return DLB_E_ARG;
  c->alog_cap = cap;
  c->alog_count = 0;
  return 0;
}

long long dlb_get_assignment_log(dlb_ctx* c, dlb_assignment* out, size_t max_records) {
  if (!c) return DLB_E_ARG;
  const unsigned long long have = c->alog_count < c->alog_cap ? c->alog_count : c->alog_cap;
  const size_t ncopy = have < max_records ? (size_t)have : max_records;
  if (ncopy && out) {
    auto it = c->dev.find("s.alog");
    if (it == c->dev.end() || !it->second.p) return DLB_E_ARG;
    cudaSetDevice(c->device);
    const cudaError_t e = cudaMemcpy(out, it->second.p, ncopy * sizeof(dlb_assignment), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return -1000 - (int)e;
  }
  return (long long)c->alog_count;
}

int dlb_dbg_set_max_attempt(dlb_ctx* c, unsigned max_attempt) {
  if (!c) return DLB_E_ARG;
  c->dbg_max_attempt = max_attempt;
  return 0;
}

// ---- stage-level entry points -----------------------------------------------------------

int dlb_dbg_keccak_f1600(dlb_ctx* c, size_t n, uint64_t* states) {
  if (!c || !states) return DLB_E_ARG;
  cudaSetDevice(c->device);
  uint64_t* d;
  DLB_TRY(dalloc(c, "dbg.a", n * 25, &d));
  DLB_TRY(h2d(c, d, states, n * 200));
  k_dbg_keccak<<<cdiv(n, 128), 128, 0, c->s()>>>((unsigned)n, d);
  DLB_LAUNCH_CHECK();
  DLB_TRY(d2h(c, states, d, n * 200));
  return sync(c);
}

int dlb_dbg_shake256(dlb_ctx* c, size_t n, const uint8_t* msgs, const uint64_t* msg_off,
                     uint8_t* out64) {
  if (!c || !msg_off || !out64) return DLB_E_ARG;
  cudaSetDevice(c->device);
  uint8_t* dm;
  uint64_t *doff, *dout;
  DLB_TRY(dalloc(c, "dbg.a", msg_off[n] + 8, &dm));
  DLB_TRY(dalloc(c, "dbg.b", n + 1, &doff));
  DLB_TRY(dalloc(c, "dbg.c", n * 8, &dout));
  DLB_TRY(h2d(c, dm, msgs, msg_off[n]));
  DLB_TRY(h2d(c, doff, msg_off, (n + 1) * 8));
  k_dbg_shake256<<<cdiv(n, 128), 128, 0, c->s()>>>((unsigned)n, dm, doff, dout);
  DLB_LAUNCH_CHECK();
  DLB_TRY(d2h(c, out64, dout, n * 64));
  return sync(c);
}

int dlb_dbg_expand_a(dlb_ctx* c, int level, size_t n_keys, const uint8_t* rhos, int32_t* out) {
  if (!c || !rhos || !out) return DLB_E_ARG;
  cudaSetDevice(c->device);
  return with_level(level, [&](auto p) {
    using P = decltype(p);
    const size_t streams = n_keys * P::K * P::L;
    uint8_t* dr;
    int32_t* dout;
    DLB_TRY(dalloc(c, "dbg.a", n_keys * 32, &dr));
    DLB_TRY(dalloc(c, "dbg.b", streams * kN, &dout));
    DLB_TRY(h2d(c, dr, rhos, n_keys * 32));
    k_expand_a<P, 4><<<cdiv(streams, 128), 128, 0, c->s()>>>(dr, 32, (unsigned)streams, dout);
    DLB_LAUNCH_CHECK();
    DLB_TRY(d2h(c, out, dout, streams * kN * 4));
    return sync(c);
  });
}

int dlb_dbg_expand_s(dlb_ctx* c, int level, size_t n, const uint8_t* rho_primes, int8_t* out) {
  if (!c || !rho_primes || !out) return DLB_E_ARG;
  cudaSetDevice(c->device);
  return with_level(level, [&](auto p) {
    using P = decltype(p);
    const size_t streams = n * (P::K + P::L);
    uint8_t* dr;
    int8_t* dout;
    DLB_TRY(dalloc(c, "dbg.a", n * 64, &dr));
    DLB_TRY(dalloc(c, "dbg.b", streams * kN, &dout));
    DLB_TRY(h2d(c, dr, rho_primes, n * 64));
    k_expand_s<P, 4><<<cdiv(streams, 128), 128, 0, c->s()>>>(dr, 64, (unsigned)streams, dout);
    DLB_LAUNCH_CHECK();
    DLB_TRY(d2h(c, out, dout, streams * kN));
    return sync(c);
  });
}

int dlb_dbg_expand_mask(dlb_ctx* c, int level, size_t n, const uint8_t* rho_primes,
                        const uint32_t* kappas, int32_t* out) {
  if (!c || !rho_primes || !kappas || !out) return DLB_E_ARG;
  cudaSetDevice(c->device);
  return with_level(level, [&](auto p) {
    using P = decltype(p);
    const size_t polys = n * P::L;
    uint64_t* dr;
    uint32_t* dk;
    uint8_t* dy;
    int32_t* dout;
    DLB_TRY(dalloc(c, "dbg.a", n * 8, &dr));
    DLB_TRY(dalloc(c, "dbg.b", n, &dk));
    DLB_TRY(dalloc(c, "dbg.c", polys * Sizes<P>::Z_POLY + 8, &dy));
    DLB_TRY(dalloc(c, "dbg.d", polys * kN, &dout));
    DLB_TRY(h2d(c, dr, rho_primes, n * 64));
    DLB_TRY(h2d(c, dk, kappas, n * 4));
    k_dbg_expand_mask<P, 4><<<cdiv(polys, 128), 128, 0, c->s()>>>((unsigned)n, dr, dk, dy);
    k_dbg_unpack_mask<P><<<cdiv(polys * kN, 256), 256, 0, c->s()>>>((unsigned)polys, dy, dout);
    DLB_LAUNCH_CHECK();
    DLB_TRY(d2h(c, out, dout, polys * kN * 4));
    return sync(c);
  });
}

int dlb_dbg_sample_in_ball(dlb_ctx* c, int level, size_t n, const uint8_t* c_tildes, int8_t* out) {
  if (!c || !c_tildes || !out) return DLB_E_ARG;
  cudaSetDevice(c->device);
  return with_level(level, [&](auto p) {
    using P = decltype(p);
    uint8_t* dc;
    int8_t* dout;
    constexpr size_t CT = Hashing<P>::CT;  // 32 bytes, or lambda/4 at the FIPS 204 levels
    DLB_TRY(dalloc(c, "dbg.a", n * CT, &dc));
    DLB_TRY(dalloc(c, "dbg.b", n * kN, &dout));
    DLB_TRY(h2d(c, dc, c_tildes, n * CT));
    k_sample_in_ball<P, 4><<<cdiv(n, 128), 128, 0, c->s()>>>(dc, CT, (unsigned)n, dout);
    DLB_LAUNCH_CHECK();
    DLB_TRY(d2h(c, out, dout, n * kN));
    return sync(c);
  });
}

int dlb_dbg_rounding(dlb_ctx* c, int gamma2_divisor, int32_t first, size_t n, int32_t* out6) {
  if (!c || !out6 || (gamma2_divisor != 88 && gamma2_divisor != 32)) return DLB_E_ARG;
  cudaSetDevice(c->device);
  int32_t* d;
  DLB_TRY(dalloc(c, "dbg.a", 6 * n, &d));
  if (gamma2_divisor == 88)
    k_dbg_rounding<(kQ - 1) / 88><<<cdiv(n, 256), 256, 0, c->s()>>>((unsigned)n, first, d, d + n, d + 2 * n,
                                                                    d + 3 * n, d + 4 * n, d + 5 * n);
  else
    k_dbg_rounding<(kQ - 1) / 32><<<cdiv(n, 256), 256, 0, c->s()>>>((unsigned)n, first, d, d + n, d + 2 * n,
                                                                    d + 3 * n, d + 4 * n, d + 5 * n);
  DLB_LAUNCH_CHECK();
  DLB_TRY(d2h(c, out6, d, 6 * n * 4));
  return sync(c);
}

int dlb_dbg_ntt(dlb_ctx* c, size_t n, int32_t* polys, int inverse) {
  if (!c || !polys) return DLB_E_ARG;
  cudaSetDevice(c->device);
  int32_t* d;
  DLB_TRY(dalloc(c, "dbg.a", n * kN, &d));
  DLB_TRY(h2d(c, d, polys, n * kN * 4));
  k_dbg_ntt<<<cdiv(n, 4), 128, 0, c->s()>>>((unsigned)n, d, inverse);
  DLB_LAUNCH_CHECK();
  DLB_TRY(d2h(c, polys, d, n * kN * 4));
  return sync(c);
}

}  // extern "C"
