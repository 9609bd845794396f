// api.hpp -- C++ host shim over the C ABI (dilithium_b200.h) with the reference's API
// surface for the batched hot path, so call sites written against
// proj/include/dilithium/{scheme,batch}.hpp compile after switching the namespace:
//
//   dilithium::keygen<P>(zeta)                 scheme.hpp:68-69    -> dilithium::b200::keygen<P>
//   dilithium::make_precomp<P>(sk)             scheme.hpp:106-107  -> b200::make_precomp<P>
//   dilithium::sign_with_precomp<P>(pre,msg,rho')   :253-255       -> b200::sign_with_precomp<P>
//   dilithium::sign<P>(sk,msg)                 scheme.hpp:268-269  -> b200::sign<P>
//   dilithium::verify<P>(pk,msg,sig)           scheme.hpp:277-279  -> b200::verify<P>
//   dilithium::batch_sign<P>(jobs,cfg,stats)   batch.hpp:53-55     -> b200::batch_sign<P>
//   dilithium::batch_verify<P>(jobs,workers)   batch.hpp:148-149   -> b200::batch_verify<P>
//   dilithium::batch_keygen<P>(zetas,workers)  batch.hpp:159-161   -> b200::batch_keygen<P>
//
// Same argument meaning and error behaviour: sign throws std::invalid_argument on a
// malformed key (scheme.hpp:271), make_precomp returns nullopt (packing.hpp:217,79-86),
// verify never throws and rejects wrong lengths (scheme.hpp:280-283), batch_sign reports
// per-task failures in BatchStats::failed_tasks (batch.hpp:128-131).  `workers` is
// accepted and ignored (the GPU grid replaces the worker pool); cfg.psi = resident
// attempt slots; cfg.speculate honoured.  Header-only, C++20, links libdilithium_b200.so.
#pragma once
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <unordered_map>
#include <vector>

#include "../dilithium_b200.h"

namespace dilithium::b200 {

inline constexpr size_t kSeedBytes = 32;
inline constexpr size_t kCrhBytes = 64;

struct Params {
  int level;
  size_t k, l;
  int eta;
  size_t eta_bits, z_bits, omega;
  size_t tr_bytes = 32, ctilde_bytes = 32;  // 64 and lambda/4 for the FIPS 204 sets
  constexpr size_t pk_bytes() const { return 32 + k * 320; }
  constexpr size_t sk_bytes() const { return 64 + tr_bytes + (k + l) * 32 * eta_bits + k * 416; }
  constexpr size_t sig_bytes() const { return ctilde_bytes + l * 32 * z_bits + omega + k; }
  friend constexpr bool operator==(const Params&, const Params&) = default;
};

inline constexpr Params kDilithium2{2, 4, 4, 2, 3, 18, 80};
inline constexpr Params kDilithium3{3, 6, 5, 4, 4, 20, 55};
inline constexpr Params kDilithium5{5, 8, 7, 2, 3, 20, 75};
// FIPS 204 parameter sets (not in the reference, which declares them a non-goal): the same
// engine with the standard's hashing conventions; deterministic signing, empty context.
inline constexpr Params kMLDSA44{44, 4, 4, 2, 3, 18, 80, 64, 32};
inline constexpr Params kMLDSA65{65, 6, 5, 4, 4, 20, 55, 64, 48};
inline constexpr Params kMLDSA87{87, 8, 7, 2, 3, 20, 75, 64, 64};
static_assert(kMLDSA44.sk_bytes() == 2560 && kMLDSA44.sig_bytes() == 2420);
static_assert(kMLDSA65.sk_bytes() == 4032 && kMLDSA65.sig_bytes() == 3309);
static_assert(kMLDSA87.sk_bytes() == 4896 && kMLDSA87.sig_bytes() == 4627);
static_assert(kDilithium2.pk_bytes() == 1312 && kDilithium2.sk_bytes() == 2528 && kDilithium2.sig_bytes() == 2420);
static_assert(kDilithium3.pk_bytes() == 1952 && kDilithium3.sk_bytes() == 4000 && kDilithium3.sig_bytes() == 3293);
static_assert(kDilithium5.pk_bytes() == 2592 && kDilithium5.sk_bytes() == 4864 && kDilithium5.sig_bytes() == 4595);

template <Params P> using PkBytes = std::array<uint8_t, P.pk_bytes()>;
template <Params P> using SkBytes = std::array<uint8_t, P.sk_bytes()>;
template <Params P> using SigBytes = std::array<uint8_t, P.sig_bytes()>;
using SeedArray = std::array<uint8_t, kSeedBytes>;
using CrhArray = std::array<uint8_t, kCrhBytes>;

// One engine per GPU, created on first use (device 0) or explicitly.
class Engine {
 public:
  explicit Engine(int device = 0) {
    const int rc = dlb_create(&ctx_, device, 0);
    if (rc != 0) throw std::runtime_error("dlb_create failed (no CUDA device?): " + std::to_string(rc));
  }
  ~Engine() { dlb_destroy(ctx_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  dlb_ctx* ctx() const { return ctx_; }
  // FIPS 204 context string (<= 255 bytes) for the ML-DSA parameter sets; sticky, default empty
  void set_mldsa_context(std::span<const uint8_t> context) {
    check_rc(dlb_set_mldsa_context(ctx_, context.data(), context.size()));
  }
  static Engine& instance() {
    static Engine e(0);
    return e;
  }

 private:
  static void check_rc(int rc) {
    if (rc != 0) throw std::invalid_argument("dlb_set_mldsa_context: status " + std::to_string(rc));
  }
  dlb_ctx* ctx_ = nullptr;
};

inline void check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string(what) + " failed: status " + std::to_string(rc));
}

// Per-key signing state.  On the GPU the transformed key lives in device memory for
// the duration of a batch call; the host object keeps the validated packed key.
template <Params P>
struct SignPrecomp {
  SkBytes<P> sk{};
  SeedArray rho{}, key{};
  std::array<uint8_t, P.tr_bytes> tr{};
};

// scheme.hpp:106-125 + the eta range check of packing.hpp:79-86
template <Params P>
std::optional<SignPrecomp<P>> make_precomp(std::span<const uint8_t> sk_bytes) {
  if (sk_bytes.size() != P.sk_bytes()) return std::nullopt;
  const size_t n_eta = (P.k + P.l) * 256;
  uint64_t acc = 0;
  unsigned nbits = 0;
  size_t seen = 0, pos = 64 + P.tr_bytes;
  while (seen < n_eta) {
    acc |= static_cast<uint64_t>(sk_bytes[pos++]) << nbits;
    nbits += 8;
    while (nbits >= P.eta_bits && seen < n_eta) {
      if ((acc & ((1u << P.eta_bits) - 1)) > 2u * static_cast<unsigned>(P.eta)) return std::nullopt;
      acc >>= P.eta_bits;
      nbits -= static_cast<unsigned>(P.eta_bits);
      ++seen;
    }
  }
  SignPrecomp<P> pre;
  std::memcpy(pre.sk.data(), sk_bytes.data(), P.sk_bytes());
  std::memcpy(pre.rho.data(), sk_bytes.data(), 32);
  std::memcpy(pre.key.data(), sk_bytes.data() + 32, 32);
  std::memcpy(pre.tr.data(), sk_bytes.data() + 64, P.tr_bytes);
  return pre;
}

// scheduler.hpp:21-28.  The device scheduler runs one round loop per CTA, so a record is one
// round of one CTA (`stream`); the remaining fields are RoundTrace's, restricted to that CTA.
struct RoundTrace {
  uint64_t round;
  size_t unfinished, assigned, speculative, idle_slots, newly_done;
  size_t stream = 0;
};

struct BatchConfig {  // batch.hpp:23-29
  size_t psi = 0;
  size_t workers = 1;
  bool speculate = true;
  std::function<void(const RoundTrace&)> trace;  // called once per logged round after the batch
  size_t trace_capacity = 1 << 20;               // records kept per call when `trace` is set
};

struct BatchStats {  // batch.hpp:31-38
  uint64_t rounds = 0, attempts = 0, speculative = 0, idle_slot_rounds = 0, accepted_attempt_sum = 0;
  std::vector<size_t> failed_tasks;
};

template <Params P>
struct SignJob {
  const SignPrecomp<P>* key = nullptr;
  std::span<const uint8_t> message;
};

template <Params P>
struct VerifyJob {
  std::span<const uint8_t> pk, message, sig;
};

template <Params P>
struct SignOutput {
  SigBytes<P> sig;
  uint32_t attempts;
};

namespace detail {
template <class Jobs>
void flatten_messages(const Jobs& jobs, std::vector<uint8_t>& flat, std::vector<uint64_t>& off) {
  off.assign(jobs.size() + 1, 0);
  for (size_t i = 0; i < jobs.size(); ++i) off[i + 1] = off[i] + jobs[i].message.size();
  flat.resize(off.back() + 8);
  for (size_t i = 0; i < jobs.size(); ++i)
    if (!jobs[i].message.empty())
      std::memcpy(flat.data() + off[i], jobs[i].message.data(), jobs[i].message.size());
}
}  // namespace detail

// batch.hpp:159-166
template <Params P>
std::vector<std::pair<PkBytes<P>, SkBytes<P>>> batch_keygen(std::span<const SeedArray> zetas,
                                                            size_t /*workers*/ = 1,
                                                            Engine& eng = Engine::instance()) {
  const size_t n = zetas.size();
  std::vector<std::pair<PkBytes<P>, SkBytes<P>>> out(n);
  if (n == 0) return out;
  std::vector<uint8_t> pks(n * P.pk_bytes()), sks(n * P.sk_bytes());
  check(dlb_keygen_batch(eng.ctx(), P.level, n, zetas.data()->data(), pks.data(), sks.data()),
        "dlb_keygen_batch");
  for (size_t i = 0; i < n; ++i) {
    std::memcpy(out[i].first.data(), pks.data() + i * P.pk_bytes(), P.pk_bytes());
    std::memcpy(out[i].second.data(), sks.data() + i * P.sk_bytes(), P.sk_bytes());
  }
  return out;
}

// batch.hpp:53-137
template <Params P>
std::vector<SigBytes<P>> batch_sign(std::span<const SignJob<P>> jobs, const BatchConfig& cfg = {},
                                    BatchStats* stats = nullptr, Engine& eng = Engine::instance(),
                                    const CrhArray* rho_prime_override = nullptr,
                                    std::vector<uint32_t>* attempts_out = nullptr) {
  const size_t n = jobs.size();
  std::vector<SigBytes<P>> out(n);
  if (n == 0) return out;
  // SignJob.key is a non-owning pointer and jobs may share keys (batch.hpp:41-44): collect the
  // distinct keys once so the device precomputes each of them once, not once per task
  std::unordered_map<const SignPrecomp<P>*, uint32_t> key_of;
  std::vector<const SignPrecomp<P>*> keys;
  std::vector<uint32_t> key_idx(n);
  for (size_t i = 0; i < n; ++i) {
    auto [it, fresh] = key_of.try_emplace(jobs[i].key, static_cast<uint32_t>(keys.size()));
    if (fresh) keys.push_back(jobs[i].key);
    key_idx[i] = it->second;
  }
  const bool shared = keys.size() == 1;
  std::vector<uint8_t> sks;
  const uint8_t* skp = jobs[0].key->sk.data();
  if (!shared) {
    sks.resize(keys.size() * P.sk_bytes());
    for (size_t k = 0; k < keys.size(); ++k)
      std::memcpy(sks.data() + k * P.sk_bytes(), keys[k]->sk.data(), P.sk_bytes());
    skp = sks.data();
  }
  std::vector<uint8_t> flat;
  std::vector<uint64_t> off;
  detail::flatten_messages(jobs, flat, off);
  std::vector<uint32_t> att(n);
  std::vector<uint8_t> failed(n);
  dlb_sign_stats st{};
  static_assert(sizeof(SigBytes<P>) == P.sig_bytes());
  const uint8_t* rp = rho_prime_override ? rho_prime_override->data() : nullptr;
  if (cfg.trace) check(dlb_set_trace(eng.ctx(), cfg.trace_capacity), "dlb_set_trace");
  const int rc =
      shared ? dlb_sign_batch(eng.ctx(), P.level, n, skp, 0, flat.data(), off.data(), rp, cfg.psi,
                              cfg.speculate ? 1 : 0, out[0].data(), att.data(), failed.data(), &st)
             : dlb_sign_batch_keyed(eng.ctx(), P.level, keys.size(), skp, n, key_idx.data(), flat.data(),
                                    off.data(), rp, cfg.psi, cfg.speculate ? 1 : 0, out[0].data(),
                                    att.data(), failed.data(), &st);
  if (cfg.trace) {
    std::vector<dlb_round_trace> recs(cfg.trace_capacity);
    const long long total = rc == 0 ? dlb_get_trace(eng.ctx(), recs.data(), recs.size()) : 0;
    dlb_set_trace(eng.ctx(), 0);
    const size_t have = total < 0 ? 0 : std::min<size_t>(static_cast<size_t>(total), recs.size());
    std::sort(recs.begin(), recs.begin() + have, [](const dlb_round_trace& a, const dlb_round_trace& b) {
      return a.stream != b.stream ? a.stream < b.stream : a.round < b.round;
    });
    for (size_t i = 0; i < have; ++i)
      cfg.trace(RoundTrace{recs[i].round, recs[i].unfinished, recs[i].assigned, recs[i].speculative,
                           recs[i].idle_slots, recs[i].newly_done, recs[i].stream});
  }
  if (rc == DLB_E_KEY) throw std::invalid_argument("batch_sign: malformed secret key");
  check(rc, "dlb_sign_batch");
  if (stats) {
    stats->rounds = st.rounds;
    stats->attempts = st.attempts;
    stats->speculative = st.speculative;
    stats->idle_slot_rounds = st.idle_slot_rounds;
    stats->accepted_attempt_sum = st.accepted_attempt_sum;
    stats->failed_tasks.clear();
    for (size_t i = 0; i < n; ++i)
      if (failed[i]) stats->failed_tasks.push_back(i);
  }
  if (attempts_out) *attempts_out = att;
  return out;
}

// batch.hpp:148-156; wrong-length pk/sig reject host-side (scheme.hpp:280-283)
template <Params P>
std::vector<uint8_t> batch_verify(std::span<const VerifyJob<P>> jobs, size_t /*workers*/ = 1,
                                  Engine& eng = Engine::instance()) {
  const size_t n = jobs.size();
  std::vector<uint8_t> flags(n, 0);
  std::vector<size_t> live;
  for (size_t i = 0; i < n; ++i)
    if (jobs[i].pk.size() == P.pk_bytes() && jobs[i].sig.size() == P.sig_bytes()) live.push_back(i);
  if (live.empty()) return flags;
  const size_t m = live.size();
  // jobs that point at the same public key bytes share one expanded key on the device
  std::unordered_map<const uint8_t*, uint32_t> key_of;
  std::vector<const uint8_t*> keys;
  std::vector<uint32_t> key_idx(m);
  for (size_t a = 0; a < m; ++a) {
    const uint8_t* pkp = jobs[live[a]].pk.data();
    auto [it, fresh] = key_of.try_emplace(pkp, static_cast<uint32_t>(keys.size()));
    if (fresh) keys.push_back(pkp);
    key_idx[a] = it->second;
  }
  std::vector<uint8_t> pks(keys.size() * P.pk_bytes()), sigs(m * P.sig_bytes() + 8), flat, f(m);
  for (size_t k = 0; k < keys.size(); ++k) std::memcpy(pks.data() + k * P.pk_bytes(), keys[k], P.pk_bytes());
  std::vector<uint64_t> off(m + 1, 0);
  for (size_t a = 0; a < m; ++a) off[a + 1] = off[a] + jobs[live[a]].message.size();
  flat.resize(off.back() + 8);
  for (size_t a = 0; a < m; ++a) {
    const auto& j = jobs[live[a]];
    std::memcpy(sigs.data() + a * P.sig_bytes(), j.sig.data(), P.sig_bytes());
    if (!j.message.empty()) std::memcpy(flat.data() + off[a], j.message.data(), j.message.size());
  }
  if (keys.size() == 1)
    check(dlb_verify_batch(eng.ctx(), P.level, m, pks.data(), 0, flat.data(), off.data(), sigs.data(),
                           f.data()),
          "dlb_verify_batch");
  else
    check(dlb_verify_batch_keyed(eng.ctx(), P.level, keys.size(), pks.data(), m, key_idx.data(),
                                 flat.data(), off.data(), sigs.data(), f.data()),
          "dlb_verify_batch_keyed");
  for (size_t a = 0; a < m; ++a) flags[live[a]] = f[a];
  return flags;
}

// ---- single-task forms: batches of one ------------------------------------------------

template <Params P>
std::pair<PkBytes<P>, SkBytes<P>> keygen(std::span<const uint8_t, kSeedBytes> zeta,
                                         Engine& eng = Engine::instance()) {
  SeedArray z;
  std::memcpy(z.data(), zeta.data(), 32);
  return batch_keygen<P>(std::span<const SeedArray>(&z, 1), 1, eng)[0];
}

template <Params P>
SignOutput<P> sign_with_precomp(const SignPrecomp<P>& pre, std::span<const uint8_t> msg,
                                const CrhArray* rho_prime_override = nullptr,
                                Engine& eng = Engine::instance()) {
  SignJob<P> job{&pre, msg};
  BatchStats st;
  std::vector<uint32_t> att;
  auto sigs = batch_sign<P>(std::span<const SignJob<P>>(&job, 1), {}, &st, eng, rho_prime_override, &att);
  if (!st.failed_tasks.empty()) throw std::runtime_error("sign: rejection loop did not terminate");
  return {sigs[0], att[0]};
}

template <Params P>
SigBytes<P> sign(std::span<const uint8_t> sk_bytes, std::span<const uint8_t> msg,
                 Engine& eng = Engine::instance()) {
  auto pre = make_precomp<P>(sk_bytes);
  if (!pre) throw std::invalid_argument("sign: malformed secret key");
  return sign_with_precomp<P>(*pre, msg, nullptr, eng).sig;
}

template <Params P>
bool verify(std::span<const uint8_t> pk_bytes, std::span<const uint8_t> msg,
            std::span<const uint8_t> sig_bytes, Engine& eng = Engine::instance()) {
  VerifyJob<P> job{pk_bytes, msg, sig_bytes};
  try {
    return batch_verify<P>(std::span<const VerifyJob<P>>(&job, 1), 1, eng)[0] != 0;
  } catch (...) {
    return false;  // verify never throws (scheme.hpp:277-318 is fail-closed)
  }
}

// ---- several GPUs of one box ------------------------------------------------------------
// The path has no exchange step: a batch is cut into contiguous ranges lo = n*g/G,
// hi = n*(g+1)/G exactly like the reference tool's multi-engine mode
// (tools/dilithium_cli.cpp:319-339), one Engine and one host thread per device, results
// land in order.  No collective, no NCCL.  (Listing a device twice gives two contexts on
// that GPU -- used by the tests, which see a single GPU.)
class ShardedEngine {
 public:
  explicit ShardedEngine(const std::vector<int>& devices) {
    for (int d : devices) engines_.push_back(std::make_unique<Engine>(d));
    if (engines_.empty()) throw std::invalid_argument("ShardedEngine: no devices");
  }
  size_t size() const { return engines_.size(); }

  template <Params P>
  std::vector<std::pair<PkBytes<P>, SkBytes<P>>> batch_keygen(std::span<const SeedArray> zetas) {
    std::vector<std::pair<PkBytes<P>, SkBytes<P>>> out(zetas.size());
    run(zetas.size(), [&](Engine& e, size_t lo, size_t hi) {
      auto part = b200::batch_keygen<P>(zetas.subspan(lo, hi - lo), 1, e);
      std::move(part.begin(), part.end(), out.begin() + lo);
    });
    return out;
  }

  template <Params P>
  std::vector<SigBytes<P>> batch_sign(std::span<const SignJob<P>> jobs, const BatchConfig& cfg = {},
                                      BatchStats* stats = nullptr) {
    std::vector<SigBytes<P>> out(jobs.size());
    std::vector<BatchStats> part_stats(engines_.size());
    std::vector<size_t> los(engines_.size(), 0);
    run(jobs.size(), [&](Engine& e, size_t lo, size_t hi) {
      const size_t g = index_of(e);
      los[g] = lo;
      auto part = b200::batch_sign<P>(jobs.subspan(lo, hi - lo), cfg, &part_stats[g], e);
      std::copy(part.begin(), part.end(), out.begin() + lo);
    });
    if (stats) {
      *stats = BatchStats{};
      for (size_t g = 0; g < engines_.size(); ++g) {
        const BatchStats& s = part_stats[g];
        stats->rounds += s.rounds;
        stats->attempts += s.attempts;
        stats->speculative += s.speculative;
        stats->idle_slot_rounds += s.idle_slot_rounds;
        stats->accepted_attempt_sum += s.accepted_attempt_sum;
        for (size_t t : s.failed_tasks) stats->failed_tasks.push_back(los[g] + t);
      }
    }
    return out;
  }

  template <Params P>
  std::vector<uint8_t> batch_verify(std::span<const VerifyJob<P>> jobs) {
    std::vector<uint8_t> flags(jobs.size(), 0);
    run(jobs.size(), [&](Engine& e, size_t lo, size_t hi) {
      auto part = b200::batch_verify<P>(jobs.subspan(lo, hi - lo), 1, e);
      std::copy(part.begin(), part.end(), flags.begin() + lo);
    });
    return flags;
  }

 private:
  size_t index_of(const Engine& e) const {
    for (size_t g = 0; g < engines_.size(); ++g)
      if (engines_[g].get() == &e) return g;
    return 0;
  }
  // fork-join over the shards; the first exception is rethrown like WorkerPool::parallel_for
  template <class Fn>
  void run(size_t n, Fn&& fn) {
    const size_t G = engines_.size();
    std::vector<std::thread> threads;
    std::vector<std::exception_ptr> errs(G);
    for (size_t g = 0; g < G; ++g) {
      const size_t lo = n * g / G, hi = n * (g + 1) / G;
      if (hi == lo) continue;
      threads.emplace_back([&, g, lo, hi] {
        try {
          fn(*engines_[g], lo, hi);
        } catch (...) {
          errs[g] = std::current_exception();
        }
      });
    }
    for (auto& t : threads) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }
  std::vector<std::unique_ptr<Engine>> engines_;
};

}  // namespace dilithium::b200
