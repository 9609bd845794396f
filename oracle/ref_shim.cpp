// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile with
//   g++ -std=c++20 -O2 -I/root/reference/proj/include
// from the sources where they lie (nothing from the reference is copied into this
// repo); the output goes to oracle/_ref/libdilithium_ref.so, which is git-ignored
// but travels to the GPU box.  Used to (1) pin oracle/dilithium_oracle.c,
// (2) serve as the second checker in the GPU parity tests and (3) be timed as the
// CPU baseline (bench.py cpu_baseline.kind = "reference", and --impl reference).
// The product never loads it.
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "dilithium/dilithium.hpp"

using namespace dilithium;

namespace {

template <class Fn>
int dispatch(int level, Fn&& fn) {
  int rc = -1;
  bool ok = with_params(level, [&](auto tag) { rc = fn(tag); });
  return ok ? rc : -1;
}

}  // namespace

extern "C" {

int ref_hw_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

void ref_keccak_f1600(uint64_t* s) {
  keccak::State st;
  std::memcpy(st.data(), s, 200);
  keccak::permute(st);
  std::memcpy(s, st.data(), 200);
}

void ref_shake128(uint8_t* out, size_t outlen, const uint8_t* in, size_t inlen) {
  keccak::shake128(std::span<uint8_t>(out, outlen), std::span<const uint8_t>(in, inlen));
}

void ref_shake256(uint8_t* out, size_t outlen, const uint8_t* in, size_t inlen) {
  keccak::shake256(std::span<uint8_t>(out, outlen), std::span<const uint8_t>(in, inlen));
}

void ref_expand_a(int32_t* out, const uint8_t* rho, unsigned i, unsigned j) {
  auto p = expand_a(std::span<const uint8_t, 32>(rho, 32), i, j);
  std::memcpy(out, p.c.data(), 1024);
}

void ref_expand_s(int32_t* out, const uint8_t* rho_prime, unsigned nonce, int eta) {
  auto p = expand_s(std::span<const uint8_t, 64>(rho_prime, 64), static_cast<uint16_t>(nonce), eta);
  std::memcpy(out, p.c.data(), 1024);
}

void ref_expand_mask(int32_t* out, const uint8_t* rho_prime, unsigned nonce, int gamma1,
                     int z_bits) {
  auto p = expand_mask(std::span<const uint8_t, 64>(rho_prime, 64), static_cast<uint16_t>(nonce),
                       gamma1, static_cast<size_t>(z_bits));
  std::memcpy(out, p.c.data(), 1024);
}

void ref_sample_in_ball(int32_t* out, const uint8_t* c_tilde, int tau) {
  auto p = sample_in_ball(std::span<const uint8_t, 32>(c_tilde, 32), tau);
  std::memcpy(out, p.c.data(), 1024);
}

// raw (unreduced) forward transform and the typed (centered) inverse
void ref_ntt(int32_t* a) { ntt_inplace(std::span<int32_t, 256>(a, 256)); }

void ref_intt(int32_t* a) {
  NttPoly f;
  std::memcpy(f.c.data(), a, 1024);
  NormalPoly g = intt(f);
  std::memcpy(a, g.c.data(), 1024);
}

void ref_power2round(int32_t a, int32_t* a1, int32_t* a0) {
  auto [x, y] = power2round(a);
  *a1 = x;
  *a0 = y;
}

void ref_decompose(int32_t r, int32_t gamma2, int32_t* r1, int32_t* r0) {
  auto [x, y] = decompose(r, gamma2);
  *r1 = x;
  *r0 = y;
}

int ref_make_hint(int32_t z, int32_t r, int32_t gamma2) { return make_hint(z, r, gamma2); }
int32_t ref_use_hint(int h, int32_t r, int32_t gamma2) { return use_hint(h, r, gamma2); }

int ref_keygen(int level, const uint8_t* zeta, uint8_t* pk, uint8_t* sk) {
  return dispatch(level, [&](auto tag) {
    constexpr Params P = decltype(tag)::value;
    auto [p, s] = keygen<P>(std::span<const uint8_t, 32>(zeta, 32));
    std::memcpy(pk, p.data(), p.size());
    std::memcpy(sk, s.data(), s.size());
    return 0;
  });
}

int ref_sign(int level, const uint8_t* sk, const uint8_t* msg, size_t msglen,
             const uint8_t* rho_prime_override, uint8_t* sig, uint32_t* attempts) {
  return dispatch(level, [&](auto tag) {
    constexpr Params P = decltype(tag)::value;
    auto pre = make_precomp<P>(std::span<const uint8_t>(sk, P.sk_bytes()));
    if (!pre) return -1;
    CrhArray rp;
    if (rho_prime_override) std::memcpy(rp.data(), rho_prime_override, 64);
    try {
      auto out = sign_with_precomp<P>(*pre, std::span<const uint8_t>(msg, msglen),
                                      rho_prime_override ? &rp : nullptr);
      std::memcpy(sig, out.sig.data(), out.sig.size());
      if (attempts) *attempts = out.attempts;
    } catch (const std::exception&) {
      return -2;
    }
    return 0;
  });
}

int ref_verify(int level, const uint8_t* pk, size_t pklen, const uint8_t* msg, size_t msglen,
               const uint8_t* sig, size_t siglen) {
  return dispatch(level, [&](auto tag) {
    constexpr Params P = decltype(tag)::value;
    return verify<P>(std::span<const uint8_t>(pk, pklen), std::span<const uint8_t>(msg, msglen),
                     std::span<const uint8_t>(sig, siglen))
               ? 1
               : 0;
  });
}

int ref_sign_attempt(int level, const uint8_t* sk, const uint8_t* mu, const uint8_t* rho_prime,
                     uint32_t kappa, int* stage, uint8_t* c_tilde, int32_t* z, int32_t* hints) {
  return dispatch(level, [&](auto tag) {
    constexpr Params P = decltype(tag)::value;
    auto pre = make_precomp<P>(std::span<const uint8_t>(sk, P.sk_bytes()));
    if (!pre) return -1;
    auto r = sign_attempt<P>(*pre, std::span<const uint8_t, 64>(mu, 64),
                             std::span<const uint8_t, 64>(rho_prime, 64), kappa);
    if (stage) *stage = static_cast<int>(r.stage);
    std::memcpy(c_tilde, r.c_tilde.data(), 32);
    for (size_t j = 0; j < P.l; ++j) std::memcpy(z + 256 * j, r.z.p[j].c.data(), 1024);
    for (size_t i = 0; i < P.k; ++i) std::memcpy(hints + 256 * i, r.hints.p[i].c.data(), 1024);
    return r.accepted ? 1 : 0;
  });
}

int ref_sign_attempt_bounded(int level, const uint8_t* sk, const uint8_t* mu, const uint8_t* rho_prime,
                             uint32_t kappa, int32_t z_bound, int32_t r0_bound, int32_t vt_bound,
                             int* stage, uint8_t* c_tilde, int32_t* z, int32_t* hints) {
  return dispatch(level, [&](auto tag) {
    constexpr Params P = decltype(tag)::value;
    auto pre = make_precomp<P>(std::span<const uint8_t>(sk, P.sk_bytes()));
    if (!pre) return -1;
    auto r = detail::sign_attempt_bounded<P>(*pre, std::span<const uint8_t, 64>(mu, 64),
                                             std::span<const uint8_t, 64>(rho_prime, 64), kappa, z_bound,
                                             r0_bound, vt_bound);
    if (stage) *stage = static_cast<int>(r.stage);
    std::memcpy(c_tilde, r.c_tilde.data(), 32);
    for (size_t j = 0; j < P.l; ++j) std::memcpy(z + 256 * j, r.z.p[j].c.data(), 1024);
    for (size_t i = 0; i < P.k; ++i) std::memcpy(hints + 256 * i, r.hints.p[i].c.data(), 1024);
    return r.accepted ? 1 : 0;
  });
}

int ref_batch_keygen(int level, size_t n, const uint8_t* zetas, uint8_t* pks, uint8_t* sks,
                     size_t workers) {
  return dispatch(level, [&](auto tag) {
    constexpr Params P = decltype(tag)::value;
    std::vector<SeedArray> z(n);
    for (size_t i = 0; i < n; ++i) std::memcpy(z[i].data(), zetas + 32 * i, 32);
    auto out = batch_keygen<P>(std::span<const SeedArray>(z), workers);
    for (size_t i = 0; i < n; ++i) {
      std::memcpy(pks + i * P.pk_bytes(), out[i].first.data(), P.pk_bytes());
      std::memcpy(sks + i * P.sk_bytes(), out[i].second.data(), P.sk_bytes());
    }
    return 0;
  });
}

struct ref_sign_stats {
  uint64_t rounds, attempts, speculative, idle_slot_rounds, accepted_attempt_sum, failed;
};

// sk_stride == 0: one shared key; otherwise one key per task (precomp built per distinct task)
int ref_batch_sign(int level, size_t n, const uint8_t* sks, size_t sk_stride, const uint8_t* msgs,
                   const uint64_t* msg_off, size_t psi, size_t workers, int speculate,
                   uint8_t* sigs, ref_sign_stats* stats) {
  return dispatch(level, [&](auto tag) {
    constexpr Params P = decltype(tag)::value;
    const size_t nkeys = sk_stride == 0 ? 1 : n;
    std::vector<SignPrecomp<P>> pre;
    pre.reserve(nkeys);
    for (size_t i = 0; i < nkeys; ++i) {
      auto p = make_precomp<P>(std::span<const uint8_t>(sks + i * sk_stride, P.sk_bytes()));
      if (!p) return -1;
      pre.push_back(std::move(*p));
    }
    std::vector<SignJob<P>> jobs(n);
    for (size_t i = 0; i < n; ++i) {
      jobs[i].key = &pre[sk_stride == 0 ? 0 : i];
      jobs[i].message = std::span<const uint8_t>(msgs + msg_off[i], msg_off[i + 1] - msg_off[i]);
    }
    BatchConfig cfg;
    cfg.psi = psi;
    cfg.workers = workers;
    cfg.speculate = speculate != 0;
    BatchStats st;
    auto out = batch_sign<P>(std::span<const SignJob<P>>(jobs), cfg, &st);
    for (size_t i = 0; i < n; ++i) std::memcpy(sigs + i * P.sig_bytes(), out[i].data(), P.sig_bytes());
    if (stats) {
      stats->rounds = st.rounds;
      stats->attempts = st.attempts;
      stats->speculative = st.speculative;
      stats->idle_slot_rounds = st.idle_slot_rounds;
      stats->accepted_attempt_sum = st.accepted_attempt_sum;
      stats->failed = st.failed_tasks.size();
    }
    return 0;
  });
}

int ref_batch_verify(int level, size_t n, const uint8_t* pks, size_t pk_stride,
                     const uint8_t* msgs, const uint64_t* msg_off, const uint8_t* sigs,
                     size_t sig_stride, size_t workers, uint8_t* flags) {
  return dispatch(level, [&](auto tag) {
    constexpr Params P = decltype(tag)::value;
    std::vector<VerifyJob<P>> jobs(n);
    for (size_t i = 0; i < n; ++i) {
      jobs[i].pk = std::span<const uint8_t>(pks + i * pk_stride, P.pk_bytes());
      jobs[i].message = std::span<const uint8_t>(msgs + msg_off[i], msg_off[i + 1] - msg_off[i]);
      jobs[i].sig = std::span<const uint8_t>(sigs + i * sig_stride, P.sig_bytes());
    }
    auto f = batch_verify<P>(std::span<const VerifyJob<P>>(jobs), workers);
    std::memcpy(flags, f.data(), n);
    return 0;
  });
}

// NonceScheduler driven by an externally supplied validity oracle: replays the
// reference's schedule/commit on a table valid[task][attempt] (attempt < depth) and
// returns per-task accepted attempt (-1 failed) -- used to pin the device scheduler's
// commit rule (scheduler.hpp:58-136).
int ref_scheduler_replay(size_t phi, size_t psi, uint32_t ell, int speculate,
                         const uint8_t* valid, size_t depth, int64_t* accepted,
                         uint64_t* attempts_executed) {
  NonceScheduler s(phi, psi, ell, speculate != 0);
  std::vector<uint8_t> v;
  while (!s.finished()) {
    const auto& a = s.schedule_round();
    v.assign(a.size(), 0);
    for (size_t i = 0; i < a.size(); ++i)
      v[i] = a[i].attempt < depth ? valid[a[i].task * depth + a[i].attempt] : 1;
    s.commit_round(v, [](size_t, size_t) {}, [](size_t) {});
  }
  for (size_t t = 0; t < phi; ++t) accepted[t] = s.accepted_attempt(t);
  if (attempts_executed) *attempts_executed = s.attempts_executed();
  return 0;
}

}  // extern "C"
