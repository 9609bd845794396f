// Exercises include/dilithium_b200/api.hpp the way the reference's own tests exercise
// scheme.hpp / batch.hpp (tests/test_scheme.cpp:27-108,195-202; tests/test_batch.cpp:190-297).
// Needs a GPU at run time; compiled (not run) by the CPU test-suite.
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
  std::printf(fails ? "api test: %d failures\n" : "api test: all passed\n", fails);
  return fails ? 1 : 0;
}
