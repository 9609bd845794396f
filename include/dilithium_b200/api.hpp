// api.hpp -- C++ host shim over the C ABI (dilithium_b200.h) with the reference's API
// surface for the batched hot path, so call sites written against
// proj/include/dilithium/{params,scheme,scheduler,batch}.hpp compile after switching the namespace:
//
//   dilithium::Params, kDilithium2/3/5,        params.hpp:17-55    -> dilithium::b200::Params, ...
//     ParamsTag, with_params                   params.hpp:84-106   -> b200::ParamsTag, b200::with_params
//   dilithium::keygen<P>(zeta)                 scheme.hpp:68-69    -> b200::keygen<P>
//   dilithium::make_precomp<P>(sk)             scheme.hpp:106-107  -> b200::make_precomp<P>
//   dilithium::message_digest<P>, deterministic_rho_prime<P>   :240-248
//   dilithium::sign_attempt<P>, detail::sign_attempt_bounded<P>, AttemptResult, RejectStage
//                                              scheme.hpp:34-43,133-230
//   dilithium::sign_with_precomp<P>(pre,msg,rho')   :253-255       -> b200::sign_with_precomp<P>
//   dilithium::sign<P>(sk,msg)                 scheme.hpp:268-269  -> b200::sign<P>
//   dilithium::verify<P>(pk,msg,sig)           scheme.hpp:277-279  -> b200::verify<P>
//   dilithium::Assignment, RoundTrace          scheduler.hpp:14-28
//   dilithium::batch_sign<P>(jobs,cfg,stats)   batch.hpp:53-55     -> b200::batch_sign<P>
//   dilithium::batch_verify<P>(jobs,workers)   batch.hpp:148-149   -> b200::batch_verify<P>
//   dilithium::batch_keygen<P>(zetas,workers)  batch.hpp:159-161   -> b200::batch_keygen<P>
//
// Same argument meaning and error behaviour: sign throws std::invalid_argument on a
// malformed key (scheme.hpp:271), make_precomp returns nullopt (packing.hpp:217,79-86),
// verify never throws and rejects wrong lengths (scheme.hpp:280-283), batch_sign reports
// per-task failures in BatchStats::failed_tasks (batch.hpp:128-131).  `workers` is
// accepted and ignored (the GPU grid replaces the worker pool); cfg.psi = resident
// attempt slots; cfg.speculate honoured; cfg.trace / cfg.assignment_hook are replayed from
// device logs after the batch.  Header-only, C++20, links libdilithium_b200.so.
//
// Transfers: every batch call stages through pinned buffers the Engine owns (grown on demand,
// reused across calls).  batch_sign submits the batch as a few tickets in flight
// (dlb_sign_submit) whose signatures the device writes straight into the pinned staging; each
// finished part is appended to the result vector while the later parts are still signing.
#pragma once
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
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

#include <sys/mman.h>

#include "../dilithium_b200.h"

namespace dilithium::b200 {

inline constexpr int32_t kQ = 8380417;
inline constexpr size_t kN = 256;
inline constexpr int kD = 13;
inline constexpr size_t kSeedBytes = 32;
inline constexpr size_t kCrhBytes = 64;

// params.hpp:17-51 plus the two sizes that differ in the FIPS 204 sets
struct Params {
  int level;
  size_t k, l;
  int32_t eta, tau, beta, gamma1, gamma2;
  size_t omega, eta_bits, z_bits, w1_bits;
  size_t tr_bytes = 32, ctilde_bytes = 32;  // 64 and lambda/4 for the FIPS 204 sets

  constexpr int32_t alpha() const { return 2 * gamma2; }
  constexpr int32_t decomp_m() const { return (kQ - 1) / alpha(); }
  constexpr size_t poly_eta_bytes() const { return kN * eta_bits / 8; }
  constexpr size_t poly_z_bytes() const { return kN * z_bits / 8; }
  constexpr size_t poly_w1_bytes() const { return kN * w1_bits / 8; }
  static constexpr size_t poly_t1_bytes() { return kN * 10 / 8; }
  static constexpr size_t poly_t0_bytes() { return kN * kD / 8; }
  constexpr size_t pk_bytes() const { return kSeedBytes + k * poly_t1_bytes(); }
  constexpr size_t sk_bytes() const {
    return 2 * kSeedBytes + tr_bytes + (k + l) * poly_eta_bytes() + k * poly_t0_bytes();
  }
  constexpr size_t hint_bytes() const { return omega + k; }
  constexpr size_t sig_bytes() const { return ctilde_bytes + l * poly_z_bytes() + hint_bytes(); }
  friend constexpr bool operator==(const Params&, const Params&) = default;
};

inline constexpr Params kDilithium2{2, 4, 4, 2, 39, 78, 1 << 17, (kQ - 1) / 88, 80, 3, 18, 6};
inline constexpr Params kDilithium3{3, 6, 5, 4, 49, 196, 1 << 19, (kQ - 1) / 32, 55, 4, 20, 4};
inline constexpr Params kDilithium5{5, 8, 7, 2, 60, 120, 1 << 19, (kQ - 1) / 32, 75, 3, 20, 4};
// FIPS 204 parameter sets (not in the reference, which declares them a non-goal): the same
// engine with the standard's hashing conventions; deterministic signing, empty context.
inline constexpr Params kMLDSA44{44, 4, 4, 2, 39, 78, 1 << 17, (kQ - 1) / 88, 80, 3, 18, 6, 64, 32};
inline constexpr Params kMLDSA65{65, 6, 5, 4, 49, 196, 1 << 19, (kQ - 1) / 32, 55, 4, 20, 4, 64, 48};
inline constexpr Params kMLDSA87{87, 8, 7, 2, 60, 120, 1 << 19, (kQ - 1) / 32, 75, 3, 20, 4, 64, 64};
static_assert(kDilithium2.gamma2 == 95232 && kDilithium2.decomp_m() == 44);
static_assert(kDilithium3.gamma2 == 261888 && kDilithium3.decomp_m() == 16);
static_assert(kDilithium2.beta == kDilithium2.tau * kDilithium2.eta && kDilithium5.beta == 120);
static_assert(kMLDSA44.sk_bytes() == 2560 && kMLDSA44.sig_bytes() == 2420);
static_assert(kMLDSA65.sk_bytes() == 4032 && kMLDSA65.sig_bytes() == 3309);
static_assert(kMLDSA87.sk_bytes() == 4896 && kMLDSA87.sig_bytes() == 4627);
static_assert(kDilithium2.pk_bytes() == 1312 && kDilithium2.sk_bytes() == 2528 && kDilithium2.sig_bytes() == 2420);
static_assert(kDilithium3.pk_bytes() == 1952 && kDilithium3.sk_bytes() == 4000 && kDilithium3.sig_bytes() == 3293);
static_assert(kDilithium5.pk_bytes() == 2592 && kDilithium5.sk_bytes() == 4864 && kDilithium5.sig_bytes() == 4595);

// params.hpp:84-106
template <Params P>
struct ParamsTag {
  static constexpr Params value = P;
};

// Dispatches a runtime level to the matching compile-time parameter set; fn receives a
// ParamsTag; false for unsupported levels.  (44 / 65 / 87 select the FIPS 204 sets.)
template <class Fn>
bool with_params(int level, Fn&& fn) {
  switch (level) {
    case 2: fn(ParamsTag<kDilithium2>{}); return true;
    case 3: fn(ParamsTag<kDilithium3>{}); return true;
    case 5: fn(ParamsTag<kDilithium5>{}); return true;
    case 44: fn(ParamsTag<kMLDSA44>{}); return true;
    case 65: fn(ParamsTag<kMLDSA65>{}); return true;
    case 87: fn(ParamsTag<kMLDSA87>{}); return true;
    default: return false;
  }
}

template <Params P> using PkBytes = std::array<uint8_t, P.pk_bytes()>;
template <Params P> using SkBytes = std::array<uint8_t, P.sk_bytes()>;
template <Params P> using SigBytes = std::array<uint8_t, P.sig_bytes()>;
using SeedArray = std::array<uint8_t, kSeedBytes>;
using CrhArray = std::array<uint8_t, kCrhBytes>;

// DLB_SHIM_PROF=1 (read once per process): host-side phase times of the batch calls on stderr
inline bool shim_prof_enabled() {
  static const bool on = std::getenv("DLB_SHIM_PROF") != nullptr;
  return on;
}
struct ShimProf {
  bool on = shim_prof_enabled();
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[shim] %-18s %.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

inline void check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string(what) + " failed: status " + std::to_string(rc));
}

// Pinned host buffer owned by an Engine, grown geometrically, reused across calls.
class PinnedBuf {
 public:
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() { release(); }
  uint8_t* get(size_t bytes) {
    if (bytes > cap_) {
      release();
      const size_t want = bytes + bytes / 4 + 4096;
      p_ = static_cast<uint8_t*>(dlb_host_alloc(want));
      if (!p_) throw std::bad_alloc();
      cap_ = want;
    }
    return p_;
  }

 private:
  void release() {
    if (p_) {
      std::memset(p_, 0, cap_);  // may have held keys
      dlb_host_free(p_);
    }
    p_ = nullptr;
    cap_ = 0;
  }
  uint8_t* p_ = nullptr;
  size_t cap_ = 0;
};

// One engine per GPU, created on first use (device 0) or explicitly.  One host thread drives
// an engine at a time.
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
    const int rc = dlb_set_mldsa_context(ctx_, context.data(), context.size());
    if (rc != 0) throw std::invalid_argument("dlb_set_mldsa_context: status " + std::to_string(rc));
  }
  static Engine& instance() {
    static Engine e(0);
    return e;
  }
  // pinned staging, by role
  PinnedBuf in_a, in_b, in_c, in_d, out_a, out_b, out_c;

 private:
  dlb_ctx* ctx_ = nullptr;
};

// Per-key signing state.  On the GPU the transformed key lives in a device-side cache keyed
// by the packed key (built on first use, kept across calls); the host object keeps the
// validated packed key.
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

// scheduler.hpp:14-19.  `slot` is the device's global attempt slot (CTA * 128 + slot).
struct Assignment {
  uint32_t slot, task, attempt, kappa;
};

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
  std::function<void(const RoundTrace&)> trace;            // called once per logged round after the batch
  std::function<void(const Assignment&)> assignment_hook;  // per executed attempt, after the batch
  size_t trace_capacity = 1 << 20;                         // records kept per call when `trace` is set
  size_t assignment_capacity = 0;                          // 0 = 64 records per task
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

// coefficient vectors of an attempt, shaped like the reference's PolyVec (`v.p[i].c[m]`)
struct CoeffPoly {
  std::array<int32_t, kN> c{};
  friend bool operator==(const CoeffPoly&, const CoeffPoly&) = default;
};
template <size_t Dim>
struct CoeffVec {
  std::array<CoeffPoly, Dim> p{};
  friend bool operator==(const CoeffVec&, const CoeffVec&) = default;
};

enum class RejectStage { ZNorm, R0Norm, VtNorm, HintWeight };  // scheme.hpp:34

template <Params P>
struct AttemptResult {  // scheme.hpp:36-43
  bool accepted = false;
  RejectStage stage = RejectStage::ZNorm;  // meaningful only when rejected
  std::array<uint8_t, P.ctilde_bytes> c_tilde{};
  CoeffVec<P.l> z{};      // centered
  CoeffVec<P.k> hints{};  // 0/1 coefficients
};

namespace detail {

// Result vectors of a large batch are tens to hundreds of MB of fresh memory: with 4 KB pages the
// first touch (one page fault per 4 KB) costs more than the GPU work.  Ask for huge pages where
// the kernel offers them on request (transparent_hugepage = madvise); a no-op elsewhere.
inline void advise_huge(void* p, size_t bytes) {
#ifdef MADV_HUGEPAGE
  constexpr uintptr_t kHuge = 2u << 20;
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + kHuge - 1) & ~(kHuge - 1);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~(kHuge - 1);
  if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
#else
  (void)p;
  (void)bytes;
#endif
}

// fn(lo, hi) over [0, n) on up to `threads` host threads (the caller's included)
template <class Fn>
void parallel_ranges(size_t n, size_t threads, size_t min_per_thread, Fn&& fn) {
  size_t t = std::min(threads, std::max<size_t>(1, n / std::max<size_t>(1, min_per_thread)));
  if (t <= 1) {
    fn(size_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  for (size_t i = 1; i < t; ++i) pool.emplace_back([&fn, n, t, i] { fn(n * i / t, n * (i + 1) / t); });
  fn(size_t{0}, n / t);
  for (auto& th : pool) th.join();
}

// First touch of a fresh allocation on several threads (one write per 4 KB page): the page faults
// -- the dominant cost of a result vector of hundreds of MB -- then run in parallel instead of inside
// the single-threaded element construction that follows.
inline void prefault(void* p, size_t bytes, size_t threads) {
  auto* base = static_cast<volatile uint8_t*>(p);
  parallel_ranges((bytes + 4095) / 4096, threads, 2048, [&](size_t lo, size_t hi) {
    for (size_t pg = lo; pg < hi; ++pg) base[pg * 4096] = 0;
  });
}

inline size_t copy_threads() {
  const size_t hw = std::thread::hardware_concurrency();
  return std::clamp<size_t>(hw / 2, 1, 8);
}

// messages of jobs[lo, hi) back to back in `flat` (pinned), offsets relative to the part
template <class Jobs>
void flatten_messages(const Jobs& jobs, size_t lo, size_t hi, uint8_t* flat, uint64_t* off) {
  off[0] = 0;
  for (size_t i = lo; i < hi; ++i) {
    const auto& m = jobs[i].message;
    if (!m.empty()) std::memcpy(flat + off[i - lo], m.data(), m.size());
    off[i - lo + 1] = off[i - lo] + m.size();
  }
}

template <class Jobs>
size_t message_bytes(const Jobs& jobs, size_t lo, size_t hi) {
  size_t s = 0;
  for (size_t i = lo; i < hi; ++i) s += jobs[i].message.size();
  return s;
}

// scheme.hpp:133-219 through the device's single-round entry; bounds == nullptr = the scheme's
template <Params P>
AttemptResult<P> sign_attempt_impl(const SignPrecomp<P>& pre, std::span<const uint8_t, kCrhBytes> mu,
                                   std::span<const uint8_t, kCrhBytes> rho_prime, uint32_t kappa,
                                   const int32_t* bounds, Engine& eng) {
  AttemptResult<P> res;
  std::vector<int32_t> z(P.l * kN), h(P.k * kN);
  uint8_t accepted = 0, stage = 255;
  const int32_t b[3] = {bounds ? bounds[0] : P.gamma1 - P.beta, bounds ? bounds[1] : P.gamma2 - P.beta,
                        bounds ? bounds[2] : P.gamma2};
  check(dlb_dbg_sign_attempt_bounded(eng.ctx(), P.level, 1, pre.sk.data(), 0, mu.data(), rho_prime.data(),
                                     &kappa, b[0], b[1], b[2], &accepted, &stage, res.c_tilde.data(), z.data(),
                                     h.data()),
        "dlb_dbg_sign_attempt_bounded");
  res.accepted = accepted != 0;
  if (!res.accepted) res.stage = static_cast<RejectStage>(stage < 4 ? stage : 0);
  if (res.accepted) {
    for (size_t j = 0; j < P.l; ++j) std::memcpy(res.z.p[j].c.data(), z.data() + j * kN, kN * 4);
    for (size_t i = 0; i < P.k; ++i) std::memcpy(res.hints.p[i].c.data(), h.data() + i * kN, kN * 4);
  }
  return res;
}

// One rejection-loop iteration with injectable norm bounds (scheme.hpp:133-138; tests force
// individual reject stages through them)
template <Params P>
AttemptResult<P> sign_attempt_bounded(const SignPrecomp<P>& pre, std::span<const uint8_t, kCrhBytes> mu,
                                      std::span<const uint8_t, kCrhBytes> rho_prime, uint32_t kappa,
                                      int32_t z_bound, int32_t r0_bound, int32_t vt_bound,
                                      Engine& eng = Engine::instance()) {
  const int32_t b[3] = {z_bound, r0_bound, vt_bound};
  return sign_attempt_impl<P>(pre, mu, rho_prime, kappa, b, eng);
}

}  // namespace detail

// scheme.hpp:225-230
template <Params P>
AttemptResult<P> sign_attempt(const SignPrecomp<P>& pre, std::span<const uint8_t, kCrhBytes> mu,
                              std::span<const uint8_t, kCrhBytes> rho_prime, uint32_t kappa,
                              Engine& eng = Engine::instance()) {
  return detail::sign_attempt_impl<P>(pre, mu, rho_prime, kappa, nullptr, eng);
}

// scheme.hpp:240-248: mu = H(tr || M), rho' = H(K || mu), 64 bytes each, hashed on the device
template <Params P>
CrhArray message_digest(const SignPrecomp<P>& pre, std::span<const uint8_t> msg, Engine& eng = Engine::instance()) {
  static_assert(P.tr_bytes == 32, "round-3 sets only: FIPS 204 hashes a context prefix as well");
  std::vector<uint8_t> buf(pre.tr.size() + msg.size() + 8);
  std::memcpy(buf.data(), pre.tr.data(), pre.tr.size());
  if (!msg.empty()) std::memcpy(buf.data() + pre.tr.size(), msg.data(), msg.size());
  const uint64_t off[2] = {0, pre.tr.size() + msg.size()};
  CrhArray mu;
  check(dlb_dbg_shake256(eng.ctx(), 1, buf.data(), off, mu.data()), "dlb_dbg_shake256");
  return mu;
}

template <Params P>
CrhArray deterministic_rho_prime(const SignPrecomp<P>& pre, const CrhArray& mu, Engine& eng = Engine::instance()) {
  static_assert(P.tr_bytes == 32, "round-3 sets only");
  uint8_t buf[kSeedBytes + kCrhBytes + 8];
  std::memcpy(buf, pre.key.data(), kSeedBytes);
  std::memcpy(buf + kSeedBytes, mu.data(), kCrhBytes);
  const uint64_t off[2] = {0, kSeedBytes + kCrhBytes};
  CrhArray rp;
  check(dlb_dbg_shake256(eng.ctx(), 1, buf, off, rp.data()), "dlb_dbg_shake256");
  return rp;
}

// batch.hpp:159-166.  The batch is cut into parts; while the device generates part i + 1
// helper threads move part i from the pinned staging into the result vector.
template <Params P>
std::vector<std::pair<PkBytes<P>, SkBytes<P>>> batch_keygen(std::span<const SeedArray> zetas,
                                                            size_t /*workers*/ = 1,
                                                            Engine& eng = Engine::instance()) {
  using KeyPair = std::pair<PkBytes<P>, SkBytes<P>>;
  const size_t n = zetas.size();
  std::vector<KeyPair> out;
  if (n == 0) return out;
  ShimProf prof;
  out.reserve(n);
  detail::advise_huge(out.data(), n * sizeof(KeyPair));
  detail::prefault(out.data(), n * sizeof(KeyPair), detail::copy_threads());
  out.resize(n);
  prof.mark("keygen: result");
  constexpr size_t kPart = 16384;
  const size_t part = std::min(n, kPart);
  uint8_t* pk_stage[2] = {eng.out_a.get(2 * part * P.pk_bytes()), nullptr};
  uint8_t* sk_stage[2] = {eng.out_b.get(2 * part * P.sk_bytes()), nullptr};
  pk_stage[1] = pk_stage[0] + part * P.pk_bytes();
  sk_stage[1] = sk_stage[0] + part * P.sk_bytes();
  uint8_t* zin = eng.in_a.get(n * kSeedBytes);
  std::memcpy(zin, zetas.data()->data(), n * kSeedBytes);
  const size_t threads = detail::copy_threads();
  std::thread mover;
  auto move_part = [&out, threads](const uint8_t* pks, const uint8_t* sks, size_t lo, size_t cnt) {
    detail::parallel_ranges(cnt, threads, 512, [&](size_t a, size_t b) {
      for (size_t i = a; i < b; ++i) {
        std::memcpy(out[lo + i].first.data(), pks + i * P.pk_bytes(), P.pk_bytes());
        std::memcpy(out[lo + i].second.data(), sks + i * P.sk_bytes(), P.sk_bytes());
      }
    });
  };
  size_t pi = 0;
  for (size_t lo = 0; lo < n; lo += part, ++pi) {
    const size_t cnt = std::min(part, n - lo);
    const int b = static_cast<int>(pi & 1);
    const int rc = dlb_keygen_batch(eng.ctx(), P.level, cnt, zin + lo * kSeedBytes, pk_stage[b], sk_stage[b]);
    if (mover.joinable()) mover.join();  // part pi - 1 is in place; its buffer (b ^ 1) is free again
    check(rc, "dlb_keygen_batch");
    mover = std::thread(move_part, pk_stage[b], sk_stage[b], lo, cnt);
  }
  if (mover.joinable()) mover.join();
  prof.mark("keygen: device+move");
  return out;
}

// batch.hpp:53-137.  rho_prime_override: nullptr (deterministic signing), or ONE rho' used
// for every task (the reference's sign_with_precomp argument), or -- rho_prime_per_task --
// one rho' per task.
//
// batch_sign_into (an extension) writes into storage the caller provides instead of returning a
// fresh vector: with `into` in pinned memory (dlb_host_alloc) the device stores the signatures
// there directly and no host copy is left on the path.
namespace detail {
template <Params P>
std::vector<SigBytes<P>> batch_sign_impl(std::span<const SignJob<P>> jobs, const BatchConfig& cfg,
                                         BatchStats* stats, Engine& eng, const CrhArray* rho_prime_override,
                                         std::vector<uint32_t>* attempts_out,
                                         std::span<const CrhArray> rho_prime_per_task, SigBytes<P>* into) {
  const size_t n = jobs.size();
  std::vector<SigBytes<P>> out;
  if (n == 0) return out;
  ShimProf prof;
  if (!rho_prime_per_task.empty() && rho_prime_per_task.size() != n)
    throw std::invalid_argument("batch_sign: one rho' per task expected");
  static_assert(sizeof(SigBytes<P>) == P.sig_bytes());
  // SignJob.key is a non-owning pointer and jobs may share keys (batch.hpp:41-44): collect the
  // distinct keys once so the device precomputes each of them once, not once per task
  std::unordered_map<const SignPrecomp<P>*, uint32_t> key_of;
  std::vector<const SignPrecomp<P>*> keys;
  std::vector<uint32_t> key_idx(n);
  for (size_t i = 0; i < n; ++i) {
    if (!jobs[i].key) throw std::invalid_argument("batch_sign: job without a key");
    auto [it, fresh] = key_of.try_emplace(jobs[i].key, static_cast<uint32_t>(keys.size()));
    if (fresh) keys.push_back(jobs[i].key);
    key_idx[i] = it->second;
  }
  const bool shared = keys.size() == 1;
  prof.mark("sign: key table");
  uint8_t* skp = eng.in_a.get(keys.size() * P.sk_bytes());
  for (size_t k = 0; k < keys.size(); ++k) std::memcpy(skp + k * P.sk_bytes(), keys[k]->sk.data(), P.sk_bytes());

  // parts in flight: logs and an explicit psi describe ONE scheduler run, so they force one part
  const bool logged = static_cast<bool>(cfg.trace) || static_cast<bool>(cfg.assignment_hook);
  size_t parts = (logged || cfg.psi != 0) ? 1 : std::min<size_t>(8, (n + 4095) / 4096);
  if (parts < 1) parts = 1;
  const size_t total_msg = message_bytes(jobs, 0, n);
  uint8_t* flat = eng.in_b.get(total_msg + 8 * parts + 8);
  uint64_t* off = reinterpret_cast<uint64_t*>(eng.in_c.get((n + parts + 1) * 8));
  uint8_t* rp = nullptr;
  if (rho_prime_override || !rho_prime_per_task.empty()) {
    rp = eng.in_d.get(n * kCrhBytes);
    for (size_t i = 0; i < n; ++i)
      std::memcpy(rp + i * kCrhBytes,
                  rho_prime_override ? rho_prime_override->data() : rho_prime_per_task[i].data(), kCrhBytes);
  }
  uint8_t* sig_stage = into ? reinterpret_cast<uint8_t*>(into) : eng.out_a.get(n * P.sig_bytes() + 8);
  uint32_t* att = reinterpret_cast<uint32_t*>(eng.out_b.get(n * 4));
  uint8_t* failed = eng.out_c.get(n);

  const size_t acap = cfg.assignment_capacity ? cfg.assignment_capacity : 64 * n;
  if (cfg.trace) check(dlb_set_trace(eng.ctx(), cfg.trace_capacity), "dlb_set_trace");
  if (cfg.assignment_hook) check(dlb_set_assignment_log(eng.ctx(), acap), "dlb_set_assignment_log");

  prof.mark("sign: staging");
  struct Part {
    size_t lo, hi;
    uint64_t ticket = 0;
  };
  std::vector<Part> ps(parts);
  int rc = 0;
  size_t flat_pos = 0, off_pos = 0, submitted = 0;
  for (size_t p = 0; p < parts && rc == 0; ++p) {
    ps[p].lo = n * p / parts;
    ps[p].hi = n * (p + 1) / parts;
    const size_t cnt = ps[p].hi - ps[p].lo;
    flatten_messages(jobs, ps[p].lo, ps[p].hi, flat + flat_pos, off + off_pos);
    rc = dlb_sign_submit(eng.ctx(), P.level, shared ? 0 : keys.size(), skp, shared ? 0 : P.sk_bytes(), cnt,
                         shared ? nullptr : key_idx.data() + ps[p].lo, flat + flat_pos, off + off_pos,
                         rp ? rp + ps[p].lo * kCrhBytes : nullptr, cfg.psi, cfg.speculate ? 1 : 0,
                         sig_stage + ps[p].lo * P.sig_bytes(), att + ps[p].lo, failed + ps[p].lo, &ps[p].ticket);
    flat_pos += (off[off_pos + cnt] + 7) / 8 * 8;
    off_pos += cnt + 1;
    if (rc == 0) ++submitted;
  }
  prof.mark("sign: submit");
  if (!into) {  // while the device signs: allocate the result, fault its pages in (in parallel), size it
    out.reserve(n);
    advise_huge(out.data(), n * sizeof(SigBytes<P>));
    prefault(out.data(), n * sizeof(SigBytes<P>), copy_threads());
    // up to 64 MB the vector is sized now (its zero fill hides behind the device) and finished
    // parts are copied in by several threads; beyond, one appending pass per part is cheaper than
    // a zero fill plus a copy
    if (n * sizeof(SigBytes<P>) <= (size_t{64} << 20)) out.resize(n);
    prof.mark("sign: result pages");
  }
  dlb_sign_stats total{};
  for (size_t p = 0; p < submitted; ++p) {
    dlb_sign_stats st{};
    const int wrc = dlb_sign_wait(eng.ctx(), ps[p].ticket, &st);
    if (wrc != 0 && rc == 0) rc = wrc;
    if (rc != 0) continue;  // keep draining the tickets in flight
    total.rounds += st.rounds;
    total.attempts += st.attempts;
    total.speculative += st.speculative;
    total.idle_slot_rounds += st.idle_slot_rounds;
    total.accepted_attempt_sum += st.accepted_attempt_sum;
    if (into) continue;
    // finished part: pinned staging -> result vector on several threads, while later parts still sign
    const size_t lo = ps[p].lo, cnt = ps[p].hi - ps[p].lo;
    if (out.size() == n) {
      parallel_ranges(cnt, copy_threads(), 512, [&](size_t a, size_t b) {
        std::memcpy(out[lo + a].data(), sig_stage + (lo + a) * P.sig_bytes(), (b - a) * P.sig_bytes());
      });
    } else {
      const auto* first = reinterpret_cast<const SigBytes<P>*>(sig_stage + lo * P.sig_bytes());
      out.insert(out.end(), first, first + cnt);
    }
  }
  prof.mark("sign: wait+copy");
  if (cfg.trace) {
    std::vector<dlb_round_trace> recs(cfg.trace_capacity);
    const long long tot = rc == 0 ? dlb_get_trace(eng.ctx(), recs.data(), recs.size()) : 0;
    dlb_set_trace(eng.ctx(), 0);
    const size_t have = tot < 0 ? 0 : std::min<size_t>(static_cast<size_t>(tot), recs.size());
    std::sort(recs.begin(), recs.begin() + have, [](const dlb_round_trace& a, const dlb_round_trace& b) {
      return a.stream != b.stream ? a.stream < b.stream : a.round < b.round;
    });
    for (size_t i = 0; i < have; ++i)
      cfg.trace(RoundTrace{recs[i].round, recs[i].unfinished, recs[i].assigned, recs[i].speculative,
                           recs[i].idle_slots, recs[i].newly_done, recs[i].stream});
  }
  if (cfg.assignment_hook) {
    std::vector<dlb_assignment> recs(acap);
    const long long tot = rc == 0 ? dlb_get_assignment_log(eng.ctx(), recs.data(), recs.size()) : 0;
    dlb_set_assignment_log(eng.ctx(), 0);
    const size_t have = tot < 0 ? 0 : std::min<size_t>(static_cast<size_t>(tot), recs.size());
    for (size_t i = 0; i < have; ++i)
      cfg.assignment_hook(Assignment{recs[i].slot, recs[i].task, recs[i].attempt, recs[i].kappa});
  }
  if (rc == DLB_E_KEY) throw std::invalid_argument("batch_sign: malformed secret key");
  check(rc, "dlb_sign_submit / dlb_sign_wait");
  if (stats) {
    stats->rounds = total.rounds;
    stats->attempts = total.attempts;
    stats->speculative = total.speculative;
    stats->idle_slot_rounds = total.idle_slot_rounds;
    stats->accepted_attempt_sum = total.accepted_attempt_sum;
    stats->failed_tasks.clear();
    for (size_t i = 0; i < n; ++i)
      if (failed[i]) stats->failed_tasks.push_back(i);
  }
  if (attempts_out) attempts_out->assign(att, att + n);
  return out;
}
}  // namespace detail

template <Params P>
std::vector<SigBytes<P>> batch_sign(std::span<const SignJob<P>> jobs, const BatchConfig& cfg = {},
                                    BatchStats* stats = nullptr, Engine& eng = Engine::instance(),
                                    const CrhArray* rho_prime_override = nullptr,
                                    std::vector<uint32_t>* attempts_out = nullptr,
                                    std::span<const CrhArray> rho_prime_per_task = {}) {
  return detail::batch_sign_impl<P>(jobs, cfg, stats, eng, rho_prime_override, attempts_out, rho_prime_per_task,
                                    nullptr);
}

template <Params P>
void batch_sign_into(std::span<const SignJob<P>> jobs, std::span<SigBytes<P>> into, const BatchConfig& cfg = {},
                     BatchStats* stats = nullptr, Engine& eng = Engine::instance()) {
  if (into.size() != jobs.size()) throw std::invalid_argument("batch_sign_into: one output slot per job");
  detail::batch_sign_impl<P>(jobs, cfg, stats, eng, nullptr, nullptr, {}, into.data());
}

// batch.hpp:148-156; wrong-length pk/sig reject host-side (scheme.hpp:280-283)
template <Params P>
std::vector<uint8_t> batch_verify(std::span<const VerifyJob<P>> jobs, size_t /*workers*/ = 1,
                                  Engine& eng = Engine::instance()) {
  const size_t n = jobs.size();
  std::vector<uint8_t> flags(n, 0);
  std::vector<size_t> live;
  live.reserve(n);
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
  uint8_t* pks = eng.in_a.get(keys.size() * P.pk_bytes());
  for (size_t k = 0; k < keys.size(); ++k) std::memcpy(pks + k * P.pk_bytes(), keys[k], P.pk_bytes());
  size_t total_msg = 0;
  for (size_t a = 0; a < m; ++a) total_msg += jobs[live[a]].message.size();
  uint8_t* flat = eng.in_b.get(total_msg + 8);
  uint64_t* off = reinterpret_cast<uint64_t*>(eng.in_c.get((m + 1) * 8));
  uint8_t* sigs = eng.in_d.get(m * P.sig_bytes() + 8);
  uint8_t* f = eng.out_c.get(m);
  off[0] = 0;
  for (size_t a = 0; a < m; ++a) off[a + 1] = off[a] + jobs[live[a]].message.size();
  // gather the scattered job spans into the pinned staging on several host threads
  detail::parallel_ranges(m, detail::copy_threads(), 1024, [&](size_t lo, size_t hi) {
    for (size_t a = lo; a < hi; ++a) {
      const auto& j = jobs[live[a]];
      std::memcpy(sigs + a * P.sig_bytes(), j.sig.data(), P.sig_bytes());
      if (!j.message.empty()) std::memcpy(flat + off[a], j.message.data(), j.message.size());
    }
  });
  if (keys.size() == 1)
    check(dlb_verify_batch(eng.ctx(), P.level, m, pks, 0, flat, off, sigs, f), "dlb_verify_batch");
  else
    check(dlb_verify_batch_keyed(eng.ctx(), P.level, keys.size(), pks, m, key_idx.data(), flat, off, sigs, f),
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
// Shard g of G over an n-task batch is [n*g/G, n*(g+1)/G) -- the reference tool's partition
// (tools/dilithium_cli.cpp:323).  Uneven n leaves shards that differ by one task; G > n leaves
// empty shards.
inline std::vector<size_t> shard_bounds(size_t n, size_t shards) {
  if (shards == 0) throw std::invalid_argument("shard_bounds: no shards");
  std::vector<size_t> b(shards + 1);
  for (size_t g = 0; g <= shards; ++g) b[g] = n * g / shards;
  return b;
}

// BatchStats of the shards -> BatchStats of the batch: counters add up, a shard's failed task
// indices are rebased by the shard's first task so they index the caller's job list.
inline BatchStats merge_shard_stats(std::span<const BatchStats> parts, std::span<const size_t> bounds) {
  if (bounds.size() != parts.size() + 1) throw std::invalid_argument("merge_shard_stats: bounds / parts mismatch");
  BatchStats out;
  for (size_t g = 0; g < parts.size(); ++g) {
    const BatchStats& s = parts[g];
    out.rounds += s.rounds;
    out.attempts += s.attempts;
    out.speculative += s.speculative;
    out.idle_slot_rounds += s.idle_slot_rounds;
    out.accepted_attempt_sum += s.accepted_attempt_sum;
    for (size_t t : s.failed_tasks) {
      if (t >= bounds[g + 1] - bounds[g]) throw std::out_of_range("merge_shard_stats: failed index outside its shard");
      out.failed_tasks.push_back(bounds[g] + t);
    }
  }
  return out;
}

// The path has no exchange step: a batch is cut into contiguous ranges lo = n*g/G,
// hi = n*(g+1)/G exactly like the reference tool's multi-engine mode
// (tools/dilithium_cli.cpp:319-339), one Engine and one host thread per device, results
// land in order.  No collective, no NCCL.  (Listing a device twice gives two contexts on
// that GPU -- used by the tests, which see a single GPU.)  Each shard thread is pinned to the
// CPUs of its GPU's NUMA node (dlb_bind_thread_to_device) before it allocates or touches its
// engine's pinned staging, so staging pages and the copies through them stay node-local.
class ShardedEngine {
 public:
  explicit ShardedEngine(const std::vector<int>& devices) : devices_(devices) {
    if (devices.empty()) throw std::invalid_argument("ShardedEngine: no devices");
    engines_.resize(devices.size());
    // engines are created by their own (bound) threads: first-touch places the pinned staging
    run(devices.size(), [&](size_t g, size_t, size_t) { engines_[g] = std::make_unique<Engine>(devices_[g]); },
        /*per_engine=*/true);
  }
  size_t size() const { return engines_.size(); }
  // shard boundaries of an n-task batch (the partition run() uses)
  std::vector<size_t> partition(size_t n) const { return shard_bounds(n, engines_.size()); }

  template <Params P>
  std::vector<std::pair<PkBytes<P>, SkBytes<P>>> batch_keygen(std::span<const SeedArray> zetas) {
    std::vector<std::vector<std::pair<PkBytes<P>, SkBytes<P>>>> parts(engines_.size());
    run(zetas.size(), [&](size_t g, size_t lo, size_t hi) {
      parts[g] = b200::batch_keygen<P>(zetas.subspan(lo, hi - lo), 1, *engines_[g]);
    });
    std::vector<std::pair<PkBytes<P>, SkBytes<P>>> out;
    out.reserve(zetas.size());
    for (auto& p : parts) out.insert(out.end(), p.begin(), p.end());
    return out;
  }

  template <Params P>
  std::vector<SigBytes<P>> batch_sign(std::span<const SignJob<P>> jobs, const BatchConfig& cfg = {},
                                      BatchStats* stats = nullptr) {
    const size_t G = engines_.size();
    std::vector<std::vector<SigBytes<P>>> parts(G);
    std::vector<BatchStats> part_stats(G);
    run(jobs.size(), [&](size_t g, size_t lo, size_t hi) {
      parts[g] = b200::batch_sign<P>(jobs.subspan(lo, hi - lo), cfg, &part_stats[g], *engines_[g]);
    });
    std::vector<SigBytes<P>> out;
    out.reserve(jobs.size());
    for (auto& p : parts) out.insert(out.end(), p.begin(), p.end());
    if (stats) *stats = merge_shard_stats(part_stats, partition(jobs.size()));
    return out;
  }

  template <Params P>
  std::vector<uint8_t> batch_verify(std::span<const VerifyJob<P>> jobs) {
    std::vector<uint8_t> flags(jobs.size(), 0);
    run(jobs.size(), [&](size_t g, size_t lo, size_t hi) {
      auto part = b200::batch_verify<P>(jobs.subspan(lo, hi - lo), 1, *engines_[g]);
      std::copy(part.begin(), part.end(), flags.begin() + lo);
    });
    return flags;
  }

 private:
  // fork-join over the shards; the first exception is rethrown like WorkerPool::parallel_for
  template <class Fn>
  void run(size_t n, Fn&& fn, bool per_engine = false) {
    const size_t G = engines_.size();
    std::vector<std::thread> threads;
    std::vector<std::exception_ptr> errs(G);
    for (size_t g = 0; g < G; ++g) {
      const size_t lo = per_engine ? g : shard_bounds(n, G)[g], hi = per_engine ? g + 1 : shard_bounds(n, G)[g + 1];
      if (hi == lo) continue;
      threads.emplace_back([&, g, lo, hi] {
        try {
          dlb_bind_thread_to_device(devices_[g]);  // best effort: NUMA-local CPUs of that GPU
          fn(g, lo, hi);
        } catch (...) {
          errs[g] = std::current_exception();
        }
      });
    }
    for (auto& t : threads) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }
  std::vector<int> devices_;
  std::vector<std::unique_ptr<Engine>> engines_;
};

}  // namespace dilithium::b200
