// Exercises include/dilithium_b200/api.hpp the way the reference's own tests exercise
// scheme.hpp / batch.hpp (tests/test_scheme.cpp:27-108,195-202; tests/test_batch.cpp:190-297).
// Needs a GPU at run time; compiled (not run) by the CPU test-suite.
#include <algorithm>
#include <cstdio>
#include <random>

#include "dilithium_b200/api.hpp"

using namespace dilithium::b200;

static int fails = 0;
#define CHECK(x) do { if (!(x)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #x); ++fails; } } while (0)

template <Params P>
void level_test(std::mt19937_64& rng) {
  SeedArray zeta;
  for (auto& b : zeta) b = static_cast<uint8_t>(rng());
  auto [pk, sk] = keygen<P>(zeta);
  std::vector<uint8_t> msg(1 + rng() % 100);
  for (auto& b : msg) b = static_cast<uint8_t>(rng());
  auto sig = sign<P>(sk, msg);
  CHECK(verify<P>(pk, msg, sig));
  auto bad = sig;
  bad[rng() % bad.size()] ^= 1;
  CHECK(!verify<P>(pk, msg, bad));
  CHECK(!verify<P>(pk, msg, std::span<const uint8_t>(sig.data(), sig.size() - 1)));
  CHECK(!verify<P>(std::span<const uint8_t>(pk.data(), pk.size() - 1), msg, sig));
  // determinism + precomp path + attempts
  auto pre = make_precomp<P>(sk);
  CHECK(pre.has_value());
  auto out = sign_with_precomp<P>(*pre, msg);
  CHECK(out.sig == sig && out.attempts >= 1);
  // malformed key
  auto badsk = sk;
  badsk[64 + P.tr_bytes] = 0xFF;  // first byte of the packed s1 (behind rho, K, tr)
  CHECK(!make_precomp<P>(badsk).has_value());
  bool threw = false;
  try { sign<P>(badsk, msg); } catch (const std::invalid_argument&) { threw = true; }
  CHECK(threw);
  // batch == sequential, independent of psi / speculate
  const size_t n = 40;
  std::vector<std::vector<uint8_t>> msgs(n);
  std::vector<SignJob<P>> jobs(n);
  for (size_t i = 0; i < n; ++i) {
    msgs[i].resize(rng() % 64);
    for (auto& b : msgs[i]) b = static_cast<uint8_t>(rng());
    jobs[i] = {&*pre, msgs[i]};
  }
  BatchStats st;
  auto sigs = batch_sign<P>(std::span<const SignJob<P>>(jobs), {}, &st);
  BatchConfig c2; c2.psi = 128; c2.speculate = false;
  auto sigs2 = batch_sign<P>(std::span<const SignJob<P>>(jobs), c2);
  CHECK(sigs == sigs2 && st.failed_tasks.empty());
  for (size_t i = 0; i < n; i += 13) CHECK(sigs[i] == sign<P>(sk, msgs[i]));
  std::vector<VerifyJob<P>> vj(n);
  for (size_t i = 0; i < n; ++i) vj[i] = {pk, msgs[i], sigs[i]};
  auto corrupted = sigs[5];
  corrupted[40] ^= 0x20;
  vj[5].sig = corrupted;
  vj[6].sig = std::span<const uint8_t>(sigs[6].data(), 10);  // wrong length
  auto flags = batch_verify<P>(std::span<const VerifyJob<P>>(vj));
  for (size_t i = 0; i < n; ++i) CHECK(flags[i] == ((i == 5 || i == 6) ? 0 : 1));
  // mixed-key batch: three keys interleaved over the jobs (SignJob.key sharing, batch.hpp:41-44)
  {
    std::vector<SeedArray> kz(3);
    for (auto& z : kz) for (auto& b : z) b = static_cast<uint8_t>(rng());
    auto kp = batch_keygen<P>(std::span<const SeedArray>(kz));
    std::vector<SignPrecomp<P>> pres;
    for (auto& k : kp) pres.push_back(*make_precomp<P>(k.second));
    std::vector<SignJob<P>> mj(n);
    for (size_t i = 0; i < n; ++i) mj[i] = {&pres[(i * 7) % 3], msgs[i]};
    auto ms = batch_sign<P>(std::span<const SignJob<P>>(mj));
    std::vector<VerifyJob<P>> mv(n);
    for (size_t i = 0; i < n; ++i) mv[i] = {kp[(i * 7) % 3].first, msgs[i], ms[i]};
    auto mf = batch_verify<P>(std::span<const VerifyJob<P>>(mv));
    for (size_t i = 0; i < n; ++i) CHECK(mf[i] == 1);
    for (size_t i = 0; i < n; i += 11) CHECK(ms[i] == sign<P>(kp[(i * 7) % 3].second, msgs[i]));
    mv[1].pk = kp[((1 * 7) % 3 + 1) % 3].first;  // wrong key
    CHECK(batch_verify<P>(std::span<const VerifyJob<P>>(mv))[1] == 0);
  }
  std::vector<SeedArray> zs(9);
  for (auto& z : zs) for (auto& b : z) b = static_cast<uint8_t>(rng());
  auto keys = batch_keygen<P>(std::span<const SeedArray>(zs));
  CHECK(keys[3] == keygen<P>(zs[3]));
}

// tests/test_scheme.cpp:147-174 "forced rejection stages via corrupted bounds", same calls
void forced_stage_test() {
  constexpr Params P = kDilithium2;
  std::mt19937_64 rng(604);
  SeedArray zeta;
  for (auto& b : zeta) b = static_cast<uint8_t>(rng());
  const auto [pk, sk] = keygen<P>(zeta);
  (void)pk;
  const auto pre = make_precomp<P>(sk);
  const std::vector<uint8_t> msg{'x'};
  const CrhArray mu = message_digest<P>(*pre, msg);
  const CrhArray rhop = deterministic_rho_prime<P>(*pre, mu);
  // z bound of 1 rejects any nonzero z regardless of the attempt
  auto r = detail::sign_attempt_bounded<P>(pre.value(), mu, rhop, 0, 1, P.gamma2 - P.beta, P.gamma2);
  CHECK(!r.accepted);
  CHECK(r.stage == RejectStage::ZNorm);
  // at the accepting nonce every genuine check passes, so a corrupted bound pins exactly the stage it guards
  const auto so = sign_with_precomp<P>(*pre, msg);
  const uint32_t acc = (so.attempts - 1) * static_cast<uint32_t>(P.l);
  r = detail::sign_attempt_bounded<P>(pre.value(), mu, rhop, acc, P.gamma1 - P.beta, 1, P.gamma2);
  CHECK(!r.accepted);
  CHECK(r.stage == RejectStage::R0Norm);
  r = detail::sign_attempt_bounded<P>(pre.value(), mu, rhop, acc, P.gamma1 - P.beta, P.gamma2 - P.beta, 1);
  CHECK(!r.accepted);
  CHECK(r.stage == RejectStage::VtNorm);
  // and the genuine attempt at that nonce is the signature (test_scheme.cpp:125-145): c~ leads it
  const auto ok = sign_attempt<P>(*pre, mu, rhop, acc);
  CHECK(ok.accepted);
  CHECK(std::equal(ok.c_tilde.begin(), ok.c_tilde.end(), so.sig.begin()));
  for (uint32_t k = 0; k < acc; k += static_cast<uint32_t>(P.l)) CHECK(!sign_attempt<P>(*pre, mu, rhop, k).accepted);
}

// tests/acceptance.cpp:186-244 (criterion 5) on a smaller draw: batch == sequential for random
// (phi, psi), and the assignment hook never sees a (task, nonce) twice
template <Params P>
bool equivalence_batch(std::mt19937_64& rng, size_t phi, size_t psi, size_t workers) {
  SeedArray zeta;
  for (auto& b : zeta) b = static_cast<uint8_t>(rng());
  const auto [pk, sk] = keygen<P>(zeta);
  (void)pk;
  const auto pre = make_precomp<P>(sk);
  std::vector<std::vector<uint8_t>> msgs(phi);
  std::vector<SignJob<P>> jobs(phi);
  for (size_t i = 0; i < phi; ++i) {
    msgs[i].resize(24);
    for (auto& b : msgs[i]) b = static_cast<uint8_t>(rng());
    jobs[i] = {&*pre, msgs[i]};
  }
  std::vector<std::pair<uint32_t, uint32_t>> executed;
  BatchConfig cfg;
  cfg.psi = psi;
  cfg.workers = workers;
  cfg.assignment_hook = [&](const Assignment& a) { executed.push_back({a.task, a.kappa}); };
  std::vector<uint32_t> att;
  const auto sigs = batch_sign<P>(std::span<const SignJob<P>>(jobs), cfg, nullptr, Engine::instance(), nullptr, &att);
  std::sort(executed.begin(), executed.end());
  if (std::adjacent_find(executed.begin(), executed.end()) != executed.end()) return false;  // duplicate
  // every nonce below the accepted one was executed (scheduler.hpp:117)
  for (size_t i = 0; i < phi; ++i)
    for (uint32_t a = 0; a < att[i]; ++a)
      if (!std::binary_search(executed.begin(), executed.end(),
                              std::make_pair(static_cast<uint32_t>(i), a * static_cast<uint32_t>(P.l))))
        return false;
  for (size_t i = 0; i < phi; i += 1 + phi / 8)
    if (sigs[i] != sign_with_precomp<P>(*pre, msgs[i]).sig) return false;
  return true;
}

void equivalence_test() {
  std::mt19937_64 rng(55);
  for (int b = 0; b < 12; ++b) {
    const size_t phi = 1 + rng() % 512, psi = 1 + rng() % phi, workers = 1 + rng() % 8;
    bool ok;
    if (b % 10 < 8) ok = equivalence_batch<kDilithium2>(rng, phi, psi, workers);
    else if (b % 10 == 8) ok = equivalence_batch<kDilithium3>(rng, phi, psi, workers);
    else ok = equivalence_batch<kDilithium5>(rng, phi, psi, workers);
    CHECK(ok);
  }
}

// rho' override over a batch of more than one task (scheme.hpp:253-258): every task signs with it
void override_test() {
  constexpr Params P = kDilithium3;
  std::mt19937_64 rng(99);
  SeedArray zeta;
  for (auto& b : zeta) b = static_cast<uint8_t>(rng());
  const auto [pk, sk] = keygen<P>(zeta);
  const auto pre = make_precomp<P>(sk);
  CrhArray rp;
  for (auto& b : rp) b = static_cast<uint8_t>(rng());
  const size_t n = 7;
  std::vector<std::vector<uint8_t>> msgs(n);
  std::vector<SignJob<P>> jobs(n);
  for (size_t i = 0; i < n; ++i) {
    msgs[i].assign(5 + i, static_cast<uint8_t>(i));
    jobs[i] = {&*pre, msgs[i]};
  }
  const auto sigs = batch_sign<P>(std::span<const SignJob<P>>(jobs), {}, nullptr, Engine::instance(), &rp);
  for (size_t i = 0; i < n; ++i) {
    CHECK(sigs[i] == sign_with_precomp<P>(*pre, msgs[i], &rp).sig);
    CHECK(sigs[i] != sign_with_precomp<P>(*pre, msgs[i]).sig);
    CHECK(verify<P>(pk, msgs[i], sigs[i]));
  }
  std::vector<CrhArray> per(n, rp);
  per[3][0] ^= 1;
  const auto sigs2 = batch_sign<P>(std::span<const SignJob<P>>(jobs), {}, nullptr, Engine::instance(), nullptr,
                                   nullptr, std::span<const CrhArray>(per));
  for (size_t i = 0; i < n; ++i) CHECK((sigs2[i] == sigs[i]) == (i != 3));
}

// params.hpp:84-106: runtime level -> compile-time parameter set
void with_params_test() {
  size_t sig = 0;
  CHECK(with_params(3, [&](auto tag) { sig = decltype(tag)::value.sig_bytes(); }));
  CHECK(sig == 3293);
  CHECK(!with_params(4, [&](auto) {}));
  static_assert(ParamsTag<kDilithium5>::value.k == 8 && kDilithium2.alpha() == 2 * 95232);
  static_assert(kDilithium2.poly_w1_bytes() == 192 && kDilithium3.poly_z_bytes() == 640 &&
                Params::poly_t0_bytes() == 416 && kDilithium5.hint_bytes() == 83);
}

// a large batch goes through several tickets in flight and pinned staging: same bytes as small calls
void large_batch_test() {
  constexpr Params P = kDilithium2;
  std::mt19937_64 rng(7);
  SeedArray zeta;
  for (auto& b : zeta) b = static_cast<uint8_t>(rng());
  const auto [pk, sk] = keygen<P>(zeta);
  const auto pre = make_precomp<P>(sk);
  const size_t n = 20000;
  std::vector<std::array<uint8_t, 32>> msgs(n);
  std::vector<SignJob<P>> jobs(n);
  for (size_t i = 0; i < n; ++i) {
    for (auto& b : msgs[i]) b = static_cast<uint8_t>(rng());
    jobs[i] = {&*pre, msgs[i]};
  }
  BatchStats st;
  const auto sigs = batch_sign<P>(std::span<const SignJob<P>>(jobs), {}, &st);
  CHECK(sigs.size() == n && st.failed_tasks.empty() && st.accepted_attempt_sum >= n);
  for (size_t i = 0; i < n; i += 1999) CHECK(sigs[i] == sign_with_precomp<P>(*pre, msgs[i]).sig);
  std::vector<VerifyJob<P>> vj(n);
  for (size_t i = 0; i < n; ++i) vj[i] = {pk, msgs[i], sigs[i]};
  const auto flags = batch_verify<P>(std::span<const VerifyJob<P>>(vj));
  CHECK(std::all_of(flags.begin(), flags.end(), [](uint8_t f) { return f == 1; }));
  std::vector<SeedArray> zs(n + 1000);
  for (auto& z : zs) for (auto& b : z) b = static_cast<uint8_t>(rng());
  const auto keys = batch_keygen<P>(std::span<const SeedArray>(zs));  // two staging parts
  CHECK(keys.size() == zs.size());
  for (size_t i = 0; i < zs.size(); i += 2777) CHECK(keys[i] == keygen<P>(zs[i]));
}

// several engines over a partitioned batch (the reference tool's multi-engine mode,
// tools/dilithium_cli.cpp:319-339): same bytes and order as one engine
template <Params P>
void sharded_test(std::mt19937_64& rng) {
  ShardedEngine sh({0, 0, 0});  // three contexts on the one GPU the tests see
  const size_t n = 301;
  std::vector<SeedArray> zs(n);
  for (auto& z : zs) for (auto& b : z) b = static_cast<uint8_t>(rng());
  auto keys = sh.batch_keygen<P>(std::span<const SeedArray>(zs));
  auto keys1 = batch_keygen<P>(std::span<const SeedArray>(zs));
  CHECK(keys == keys1);
  auto pre = make_precomp<P>(keys[7].second);
  std::vector<std::vector<uint8_t>> msgs(n);
  std::vector<SignJob<P>> jobs(n);
  for (size_t i = 0; i < n; ++i) {
    msgs[i].resize(rng() % 80);
    for (auto& b : msgs[i]) b = static_cast<uint8_t>(rng());
    jobs[i] = {&*pre, msgs[i]};
  }
  BatchStats st, st1;
  auto sigs = sh.batch_sign<P>(std::span<const SignJob<P>>(jobs), {}, &st);
  auto sigs1 = batch_sign<P>(std::span<const SignJob<P>>(jobs), {}, &st1);
  CHECK(sigs == sigs1 && st.accepted_attempt_sum == st1.accepted_attempt_sum && st.failed_tasks.empty());
  std::vector<VerifyJob<P>> vj(n);
  for (size_t i = 0; i < n; ++i) vj[i] = {keys[7].first, msgs[i], sigs[i]};
  auto bad = sigs[200];
  bad[33] ^= 2;
  vj[200].sig = bad;
  auto flags = sh.batch_verify<P>(std::span<const VerifyJob<P>>(vj));
  for (size_t i = 0; i < n; ++i) CHECK(flags[i] == (i == 200 ? 0 : 1));
}

int main() {
  std::mt19937_64 rng(4242);
  level_test<kDilithium2>(rng);
  level_test<kDilithium3>(rng);
  level_test<kDilithium5>(rng);
  level_test<kMLDSA44>(rng);  // FIPS 204 parameter sets through the same shim
  level_test<kMLDSA65>(rng);
  level_test<kMLDSA87>(rng);
  sharded_test<kDilithium2>(rng);
  sharded_test<kDilithium5>(rng);
  forced_stage_test();
  equivalence_test();
  override_test();
  with_params_test();
  large_batch_test();
  std::printf(fails ? "api test: %d failures\n" : "api test: all passed\n", fails);
  return fails ? 1 : 0;
}
