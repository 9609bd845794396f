// keygen.cu -- batched key generation pipeline (scheme.hpp:68-104, batch.hpp:159-166).
//
//   k_keygen_seed   n sponges            zeta -> rho | rho' | K     (scheme.hpp:70-76)
//   k_expand_s      n*(L+K) sponges      -> s1, s2 (int8)           (sampling.hpp:61-79)
//   k_expand_a      n*K*L sponges        -> A                       (sampling.hpp:42-56)
//   k_keygen_arith  one warp per task    -> pk, sk (minus tr)       (scheme.hpp:84-101,103)
//   k_hash_tr       n sponges            pk -> tr into sk           (scheme.hpp:102)
#include "engine.cuh"
#include "samplers.cuh"
#include "verify_keygen.cuh"

namespace dlb {

// device chunk: dlb_ctx::knob_chunk = 65536 tasks -- measured: 16k -> 64k tasks per chunk = +7 % (one-sponge-per-task kernels fill more SMs)

// Chunks alternate between two compute lanes so the one-thread-per-task hashes of one
// chunk overlap the wide sampler / arithmetic kernels of the next (see verify.cu).
// The one-sponge-per-task kernels (seed expansion, tr) run once over the whole call so they
// bring enough warps to fill 148 SMs; only the stages whose scratch is large (the expanded
// matrix, 16-56 KB per key) are cut into chunks, which alternate between two compute lanes so
// the arithmetic of one chunk overlaps the samplers of the next.
template <class P>
int keygen_dev(dlb_ctx* c, size_t n, const uint8_t* d_zetas, uint8_t* d_pks, uint8_t* d_sks) {
  using S = Sizes<P>;
  constexpr int KL = P::K * P::L, PV = P::K + P::L;
  constexpr int HW = 4;
  if (n == 0) return 0;
  cudaStream_t main = c->s();
  size_t chunk = (n + 1) / 2;
  if (chunk < 2048) chunk = 2048;
  const size_t cmax = c->knob_chunk;  // DLB_CHUNK at dlb_create for experiments
  if (chunk > cmax) chunk = cmax;
  if (chunk > n) chunk = n;
  uint64_t* seeds;
  int8_t* s8[2];
  int32_t* A[2];
  const char* nm[2][2] = {{"g.s80", "g.A0"}, {"g.s81", "g.A1"}};
  DLB_TRY(dalloc(c, "g.seeds", n * 16, &seeds));
  for (int b = 0; b < 2; ++b) {
    DLB_TRY(dalloc(c, nm[b][0], chunk * PV * kN, &s8[b]));
    DLB_TRY(dalloc(c, nm[b][1], chunk * KL * kN, &A[b]));
  }
  if (const int co = pipeline_carveout(c); co >= 0) {
    prefer_carveout(k_keygen_seed, co);
    prefer_carveout(k_expand_s<P, HW>, co);
    prefer_carveout(k_expand_a<P, HW>, co);
    prefer_carveout(k_keygen_arith<P, 4>, co);
    prefer_carveout(k_hash_tr, co);
  }
  k_keygen_seed<<<cdiv(n, 128), 128, 0, main>>>(
      d_zetas, (unsigned)n, seeds,
      Hashing<P>::MLDSA ? ((unsigned)P::K | ((unsigned)P::L << 8) | (1u << 16)) : 0u);
  c->launches += 1;
  DLB_CUDA_CHECK(cudaEventRecord(c->ev_fork, main));
  DLB_CUDA_CHECK(cudaStreamWaitEvent(c->lane_s[0], c->ev_fork, 0));
  DLB_CUDA_CHECK(cudaStreamWaitEvent(c->lane_s[1], c->ev_fork, 0));
  size_t ci = 0;
  for (size_t lo = 0; lo < n; lo += chunk, ++ci) {
    const size_t cnt = n - lo < chunk ? n - lo : chunk;
    const int b = (int)(ci & 1);
    cudaStream_t st = c->lane_s[b];
    const uint8_t* seedb = reinterpret_cast<const uint8_t*>(seeds + lo * 16);
    uint8_t* pks = d_pks + lo * S::PK;
    uint8_t* sks = d_sks + lo * S::SK;
    k_expand_s<P, HW><<<cdiv(cnt * PV, HW * 32), HW * 32, 0, st>>>(seedb + 32, 128,
                                                                    (unsigned)(cnt * PV), s8[b]);
    k_expand_a<P, HW><<<cdiv(cnt * KL, HW * 32), HW * 32, 0, st>>>(seedb, 128, (unsigned)(cnt * KL),
                                                                    A[b]);
    k_keygen_arith<P, 4><<<cdiv(cnt, 4), 128, 0, st>>>((unsigned)cnt, seedb, s8[b], A[b], pks, sks);
    c->launches += 3;
    DLB_LAUNCH_CHECK();
  }
  for (int b = 0; b < 2; ++b) {
    DLB_CUDA_CHECK(cudaEventRecord(c->ev_join[b], c->lane_s[b]));
    DLB_CUDA_CHECK(cudaStreamWaitEvent(main, c->ev_join[b], 0));
  }
  k_hash_tr<<<cdiv(n, 128), 128, 0, main>>>(d_pks, S::PK, S::PK, (unsigned)n, d_sks + 64, S::SK,
                                            Hashing<P>::TRW);
  c->launches += 1;
  DLB_LAUNCH_CHECK();
  return 0;
}

template int keygen_dev<Params<2>>(dlb_ctx*, size_t, const uint8_t*, uint8_t*, uint8_t*);
template int keygen_dev<Params<3>>(dlb_ctx*, size_t, const uint8_t*, uint8_t*, uint8_t*);
template int keygen_dev<Params<5>>(dlb_ctx*, size_t, const uint8_t*, uint8_t*, uint8_t*);
template int keygen_dev<Params<44>>(dlb_ctx*, size_t, const uint8_t*, uint8_t*, uint8_t*);
template int keygen_dev<Params<65>>(dlb_ctx*, size_t, const uint8_t*, uint8_t*, uint8_t*);
template int keygen_dev<Params<87>>(dlb_ctx*, size_t, const uint8_t*, uint8_t*, uint8_t*);

}  // namespace dlb
