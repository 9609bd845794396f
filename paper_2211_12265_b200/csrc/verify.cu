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
  uint64_t ct[4];
  hash_ctilde_stream<S::W1_ALL>(mu + (size_t)t * 8,
                                reinterpret_cast<const uint64_t*>(w1buf + (size_t)t * S::W1_ALL), ct);
  const uint8_t* ts = sig + (size_t)t * sig_stride;
  bool eq = true;
#pragma unroll
  for (int w = 0; w < 4; ++w) eq = eq && (load_u64_unaligned(ts + 8 * w) == ct[w]);
  flags[t] = (eq && pre_ok[t]) ? 1 : 0;
}

constexpr size_t kVerifyChunk = 16384;

template <class P>
int verify_dev(dlb_ctx* c, size_t n, const uint8_t* d_pks, size_t pk_stride, const uint8_t* d_msgs,
               const uint64_t* d_msg_off, const uint8_t* d_sigs, uint8_t* d_flags) {
  using S = Sizes<P>;
  constexpr int KL = P::K * P::L;
  constexpr int HW = 4;  // warps per CTA for the sponge kernels
  if (n == 0) return 0;
  cudaStream_t st = c->s();
  const bool shared_key = pk_stride == 0;
  const size_t chunk = n < kVerifyChunk ? n : kVerifyChunk;
  const size_t keys_cap = shared_key ? 1 : chunk;

  int32_t* A;
  uint8_t *tr, *w1buf, *pre_ok;
  uint64_t* mu;
  int8_t* c8;
  DLB_TRY(dalloc(c, "v.A", keys_cap * KL * kN, &A));
  DLB_TRY(dalloc(c, "v.tr", keys_cap * 32, &tr));
  DLB_TRY(dalloc(c, "v.mu", chunk * 8, &mu));
  DLB_TRY(dalloc(c, "v.c8", chunk * kN, &c8));
  DLB_TRY(dalloc(c, "v.w1", chunk * S::W1_ALL, &w1buf));
  DLB_TRY(dalloc(c, "v.ok", chunk, &pre_ok));

  for (size_t lo = 0; lo < n; lo += chunk) {
    const size_t cnt = n - lo < chunk ? n - lo : chunk;
    const uint8_t* pks = d_pks + lo * pk_stride;
    const uint8_t* sigs = d_sigs + lo * S::SIG;
    if (!shared_key || lo == 0) {
      const size_t nk = shared_key ? 1 : cnt;
      k_expand_a<P, HW><<<cdiv(nk * KL, HW * 32), HW * 32, 0, st>>>(pks, pk_stride, (unsigned)(nk * KL), A);
      k_hash_tr<<<cdiv(nk, 128), 128, 0, st>>>(pks, pk_stride, S::PK, (unsigned)nk, tr, 32);
      c->launches += 2;
    }
    k_hash_mu<<<cdiv(cnt, 128), 128, 0, st>>>(tr, shared_key ? 0 : 32, nullptr, 0, d_msgs,
                                              d_msg_off + lo, (unsigned)cnt, mu, nullptr);
    k_sample_in_ball<P, HW><<<cdiv(cnt, HW * 32), HW * 32, 0, st>>>(sigs, S::SIG, (unsigned)cnt, c8);
    k_verify_arith<P, 4><<<cdiv(cnt, 4), 128, 0, st>>>(
        (unsigned)cnt, pks, pk_stride, sigs, S::SIG, A, shared_key ? 0 : (size_t)KL * kN, c8, w1buf,
        pre_ok);
    k_verify_final<P><<<cdiv(cnt, 128), 128, 0, st>>>((unsigned)cnt, mu, w1buf, sigs, S::SIG, pre_ok,
                                                      d_flags + lo);
    c->launches += 4;
    DLB_LAUNCH_CHECK();
  }
  return 0;
}

template int verify_dev<Params<2>>(dlb_ctx*, size_t, const uint8_t*, size_t, const uint8_t*,
                                   const uint64_t*, const uint8_t*, uint8_t*);
template int verify_dev<Params<3>>(dlb_ctx*, size_t, const uint8_t*, size_t, const uint8_t*,
                                   const uint64_t*, const uint8_t*, uint8_t*);
template int verify_dev<Params<5>>(dlb_ctx*, size_t, const uint8_t*, size_t, const uint8_t*,
                                   const uint64_t*, const uint8_t*, uint8_t*);

}  // namespace dlb
