// bench_shim.cpp -- end-to-end numbers of the drop-in C++ API (include/dilithium_b200/api.hpp):
// the calls a user of the reference's batch.hpp makes, std::vector / std::span in and out,
// everything (marshalling, staging, transfers, kernels, result vectors) inside the timed region.
// Prints one JSON object.  Usage: bench_shim [level] [reps]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "dilithium_b200/api.hpp"

using namespace dilithium::b200;
using Clock = std::chrono::steady_clock;

static double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

template <class Fn>
static double median_ms(int reps, Fn&& fn) {
  for (int i = 0; i < 2; ++i) fn();
  std::vector<double> xs;
  for (int i = 0; i < reps; ++i) {
    const auto t0 = Clock::now();
    fn();
    xs.push_back(ms_since(t0));
  }
  std::sort(xs.begin(), xs.end());
  return xs[xs.size() / 2];
}

template <Params P>
static void run(int reps) {
  std::mt19937_64 rng(20221112);
  SeedArray zeta;
  for (auto& b : zeta) b = static_cast<uint8_t>(rng());
  const auto [pk, sk] = keygen<P>(zeta);
  const auto pre = make_precomp<P>(sk);
  std::printf("{\"level\": %d", P.level);
  for (const size_t n : {size_t{10000}, size_t{100000}}) {
    std::vector<std::array<uint8_t, 32>> msgs(n);
    for (auto& m : msgs)
      for (auto& b : m) b = static_cast<uint8_t>(rng());
    std::vector<SignJob<P>> jobs(n);
    for (size_t i = 0; i < n; ++i) jobs[i] = {&*pre, msgs[i]};
    std::vector<SigBytes<P>> sigs;
    const double t_sign = median_ms(reps, [&] { sigs = batch_sign<P>(std::span<const SignJob<P>>(jobs)); });
    // extension: signatures written into caller-provided pinned storage (no result vector)
    auto* pinned = static_cast<SigBytes<P>*>(dlb_host_alloc(n * sizeof(SigBytes<P>)));
    const double t_into = median_ms(reps, [&] {
      batch_sign_into<P>(std::span<const SignJob<P>>(jobs), std::span<SigBytes<P>>(pinned, n));
    });
    if (std::memcmp(pinned, sigs.data(), n * sizeof(SigBytes<P>)) != 0) {
      std::fprintf(stderr, "batch_sign_into differs from batch_sign\n");
      std::exit(1);
    }
    dlb_host_free(pinned);
    std::vector<VerifyJob<P>> vj(n);
    for (size_t i = 0; i < n; ++i) vj[i] = {pk, msgs[i], sigs[i]};
    std::vector<uint8_t> flags;
    const double t_ver = median_ms(reps, [&] { flags = batch_verify<P>(std::span<const VerifyJob<P>>(vj)); });
    if (!std::all_of(flags.begin(), flags.end(), [](uint8_t f) { return f == 1; })) {
      std::fprintf(stderr, "verify rejected a signature\n");
      std::exit(1);
    }
    std::vector<SeedArray> zs(n);
    for (auto& z : zs)
      for (auto& b : z) b = static_cast<uint8_t>(rng());
    size_t got = 0;
    const double t_kg = median_ms(reps, [&] { got = batch_keygen<P>(std::span<const SeedArray>(zs)).size(); });
    if (got != n) std::exit(1);
    std::printf(", \"n%zu\": {\"batch_sign_ms\": %.3f, \"batch_verify_ms\": %.3f, \"batch_keygen_ms\": %.3f, "
                "\"batch_sign_into_ms\": %.3f, \"sign_ops_per_s\": %.0f, \"sign_into_ops_per_s\": %.0f, "
                "\"verify_ops_per_s\": %.0f, \"keygen_ops_per_s\": %.0f}",
                n, t_sign, t_ver, t_kg, t_into, n / t_sign * 1e3, n / t_into * 1e3, n / t_ver * 1e3,
                n / t_kg * 1e3);
  }
  std::printf("}\n");
}

int main(int argc, char** argv) {
  const int level = argc > 1 ? std::atoi(argv[1]) : 2;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 7;
  const bool ok = with_params(level, [&](auto tag) { run<decltype(tag)::value>(reps); });
  return ok ? 0 : 2;
}
