// verify.cu -- batched verification pipeline (scheme.hpp:277-318, batch.hpp:148-156).
//
// Stage kernels over a chunk of tasks, intermediates in the device arena:
//   k_expand_a        n_keys*K*L sponges  -> A            (sampling.hpp:42-56)
//   k_hash_tr         n_keys sponges      -> tr           (scheme.hpp:287)
//   k_hash_mu         n sponges           -> mu           (scheme.hpp:288)
//   k_sample_in_ball  n sponges           -> c            (sampling.hpp:97-120)
//   k_verify_arith    one warp per task   -> w1', pre_ok  (scheme.hpp:284-309)
//   k_verify_final    n sponges           -> flags        (scheme.hpp:311-317)
#include "engine.cuh"
#include "samplers.cuh"
#include "verify_keygen.cuh"

namespace dlb {

template <class P>
__global__ void k_verify_final(unsigned n, const uint64_t* __restrict__ mu,
                               const uint8_t* __restrict__ w1buf, const uint8_t* __restrict__ sig,
                               size_t sig_stride, const uint8_t* __restrict__ pre_ok,
                               uint8_t* __restrict__ flags) {
  using S = Sizes<P>;
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  constexpr int CTW = Hashing<P>::CTW;
  uint64_t ct[CTW];
  hash_ctilde_stream<S::W1_ALL, true, CTW>(
      mu + (size_t)t * 8, reinterpret_cast<const uint64_t*>(w1buf + (size_t)t * S::W1_ALL), ct);
  const uint8_t* ts = sig + (size_t)t * sig_stride;
  bool eq = true;
#pragma unroll
  for (int w = 0; w < CTW; ++w) eq = eq && (load_u64_unaligned(ts + 8 * w) == ct[w]);
  flags[t] = (eq && pre_ok[t]) ? 1 : 0;
}

// device chunk: dlb_ctx::knob_chunk = 65536 tasks -- measured: 16k -> 64k tasks per chunk = +7..15 %

// Chunks alternate between two compute lanes (streams forked from / joined to the
// caller's stream): the sponge-per-task kernels of one chunk (tr, mu, challenge, final
// hash -- one thread per task, too few warps to fill 148 SMs on their own) overlap the
// wide ExpandA / arithmetic kernels of the neighbouring chunk.
//
// Keys: pk_stride == 0 -> one public key for the whole batch; d_key_idx != nullptr -> a
// table of n_keys public keys (pk_stride apart) and task t verifies under key
// d_key_idx[t] (every distinct key is expanded once, before the chunks); otherwise task
// t uses the key at d_pks + t * pk_stride and keys are expanded chunk by chunk.
template <class P>
int verify_dev(dlb_ctx* c, size_t n, const uint8_t* d_pks, size_t pk_stride, size_t n_keys,
               const uint32_t* d_key_idx, const uint8_t* d_msgs, const uint64_t* d_msg_off,
               const uint8_t* d_sigs, uint8_t* d_flags, bool keys_expanded) {
  using S = Sizes<P>;
  constexpr int KL = P::K * P::L;
  constexpr int HW = 4;  // warps per CTA for the sponge kernels
  if (n == 0) return 0;
  cudaStream_t main = c->s();
  const bool keyed = d_key_idx != nullptr;
  if (keyed && (n_keys == 0 || pk_stride == 0)) return DLB_E_ARG;
  const bool shared_key = pk_stride == 0 || keyed;  // keys expanded once, before the fork
  if (!keyed) n_keys = 1;
  size_t chunk = (n + 1) / 2;
  if (chunk < 2048) chunk = 2048;
  const size_t cmax = c->knob_chunk;  // DLB_CHUNK at dlb_create for experiments
  if (chunk > cmax) chunk = cmax;
  if (chunk > n) chunk = n;
  const size_t keys_cap = shared_key ? n_keys : chunk;

  // The one-sponge-per-task stages (tr, mu, challenge, final hash) run once over the whole call:
  // a chunk's worth of tasks is too few warps for 148 SMs.  Only ExpandA and the arithmetic,
  // whose scratch is the expanded matrix (16-56 KB per key), are chunked over two lanes.
  int32_t* A[2];
  uint8_t *tr, *w1buf, *pre_ok;
  uint64_t* mu;
  int8_t* c8;
  const size_t n_tr = shared_key ? n_keys : n;
  DLB_TRY(dalloc(c, "v.A0", keys_cap * KL * kN, &A[0]));
  if (shared_key) A[1] = A[0];  // one expanded key (table) serves both lanes
  else DLB_TRY(dalloc(c, "v.A1", keys_cap * KL * kN, &A[1]));
  DLB_TRY(dalloc(c, "v.tr", n_tr * Hashing<P>::TR, &tr));
  DLB_TRY(dalloc(c, "v.mu", n * 8, &mu));
  DLB_TRY(dalloc(c, "v.c8", n * kN, &c8));
  DLB_TRY(dalloc(c, "v.w1", n * S::W1_ALL, &w1buf));
  DLB_TRY(dalloc(c, "v.ok", n, &pre_ok));
  if (const int co = pipeline_carveout(c); co >= 0) {
    prefer_carveout(k_expand_a<P, HW>, co);
    prefer_carveout(k_hash_tr, co);
    prefer_carveout(k_hash_mu<Hashing<P>::MLDSA>, co);
    prefer_carveout(k_sample_in_ball<P, HW>, co);
    prefer_carveout(k_verify_arith<P, 4>, co);
    prefer_carveout(k_verify_final<P>, co);
  }
  const uint8_t* pfx = nullptr;
  unsigned plen = 0;
  if (Hashing<P>::MLDSA) DLB_TRY(mldsa_prefix(c, main, &pfx, &plen));
  // (keys_expanded: a previous call of the same host-side batch already expanded this key
  // table into the context's arenas -- the host pipeline calls once per transfer chunk)
  if (shared_key && !keys_expanded) {
    k_expand_a<P, HW><<<cdiv(n_keys * KL, HW * 32), HW * 32, 0, main>>>(d_pks, pk_stride,
                                                                        (unsigned)(n_keys * KL), A[0]);
    c->launches += 1;
  }
  if (!(shared_key && keys_expanded)) {
    k_hash_tr<<<cdiv(n_tr, 128), 128, 0, main>>>(d_pks, pk_stride, S::PK, (unsigned)n_tr, tr,
                                                 Hashing<P>::TR, Hashing<P>::TRW);
    c->launches += 1;
  }
  const size_t key_step = keyed ? 1 : (shared_key ? 0 : 1);  // 0: every task uses key 0
  k_hash_mu<Hashing<P>::MLDSA><<<cdiv(n, 128), 128, 0, main>>>(
      tr, key_step * Hashing<P>::TR, nullptr, 0, d_key_idx, pfx, plen, d_msgs, d_msg_off, (unsigned)n, mu,
      nullptr);
  k_sample_in_ball<P, HW><<<cdiv(n, HW * 32), HW * 32, 0, main>>>(d_sigs, S::SIG, (unsigned)n, c8);
  c->launches += 2;
  DLB_CUDA_CHECK(cudaEventRecord(c->ev_fork, main));
  DLB_CUDA_CHECK(cudaStreamWaitEvent(c->lane_s[0], c->ev_fork, 0));
  DLB_CUDA_CHECK(cudaStreamWaitEvent(c->lane_s[1], c->ev_fork, 0));
  size_t ci = 0;
  for (size_t lo = 0; lo < n; lo += chunk, ++ci) {
    const size_t cnt = n - lo < chunk ? n - lo : chunk;
    const int b = (int)(ci & 1);
    cudaStream_t st = c->lane_s[b];
    const uint8_t* pks = keyed ? d_pks : d_pks + lo * pk_stride;
    const uint32_t* kidx = keyed ? d_key_idx + lo : nullptr;
    const uint8_t* sigs = d_sigs + lo * S::SIG;
    if (!shared_key) {
      k_expand_a<P, HW><<<cdiv(cnt * KL, HW * 32), HW * 32, 0, st>>>(pks, pk_stride,
                                                                     (unsigned)(cnt * KL), A[b]);
      c->launches += 1;
    }
    k_verify_arith<P, 4><<<cdiv(cnt, 4), 128, 0, st>>>(
        (unsigned)cnt, pks, pk_stride, sigs, S::SIG, A[b], key_step * (size_t)KL * kN, kidx, c8 + lo * kN,
        w1buf + lo * S::W1_ALL, pre_ok + lo);
    c->launches += 1;
    DLB_LAUNCH_CHECK();
  }
  for (int b = 0; b < 2; ++b) {
    DLB_CUDA_CHECK(cudaEventRecord(c->ev_join[b], c->lane_s[b]));
    DLB_CUDA_CHECK(cudaStreamWaitEvent(main, c->ev_join[b], 0));
  }
  k_verify_final<P><<<cdiv(n, 128), 128, 0, main>>>((unsigned)n, mu, w1buf, d_sigs, S::SIG, pre_ok, d_flags);
  c->launches += 1;
  DLB_LAUNCH_CHECK();
  return 0;
}

#define DLB_INST(LV)                                                                          \
  template int verify_dev<Params<LV>>(dlb_ctx*, size_t, const uint8_t*, size_t, size_t,       \
                                      const uint32_t*, const uint8_t*, const uint64_t*,       \
                                      const uint8_t*, uint8_t*, bool);
DLB_INST(2)
DLB_INST(3)
DLB_INST(5)
DLB_INST(44)
DLB_INST(65)
DLB_INST(87)
#undef DLB_INST

}  // namespace dlb
