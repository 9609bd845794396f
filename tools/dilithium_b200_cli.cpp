// dilithium_b200 -- command-line front end of the B200 engine.
//
// Same subcommands, options, file formats and exit codes as the reference tool
// (proj/tools/dilithium_cli.cpp:136-297 commands, :360-446 bench, :518-607 option table;
// behaviour pinned by proj/tests/test_cli.cpp:61-175):
//
//   keygen       --level L --pk F --sk F [--seed HEX64] [--out-format binary|hex]
//   sign         --level L --sk F --in MSG --out SIG [--out-format ...]
//   verify       --level L --pk F --in MSG --sig SIG        exit 0 accept / 1 reject / 2 bad input
//   batch-sign   --level L --sk F --out-dir D [--psi N] [--workers N] [--trace CSV] MSG...
//   batch-verify --level L --pk F --sig-dir D [--workers N] MSG...     exit 0 iff all accept
//   sweep        --level L [--phi N] [--reps N] [--psi-min N] [--psi-max N] [--psi-steps N] [--streams-max N]
//                CSV rows of the modes sweep-psi / sweep-batch / sweep-streams (same schema)
//   bench        --level L [--phi N] [--psi N] [--workers N] [--streams N] [--reps N]
//                CSV on stdout: schema,mode,op,level,phi,psi,workers,streams,reps,
//                               throughput_ops_s,mean_latency_us,attempts_mean
//
// Key and signature files are raw bytes or the hex text written with --out-format hex; the
// expected object length tells them apart.  --workers is accepted and ignored (the GPU grid
// replaces the worker pool).  --trace writes one row per scheduler round with the reference
// tool's columns; `stream` is the CTA whose round it was (the device scheduler runs one
// independent round loop per CTA).
//
// The option parser is this file's own (the reference uses CLI11, which this tree does not
// vendor): a table of named options per subcommand, positionals collected in order.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <random>
#include <set>
#include <string>

#include "dilithium_b200/api.hpp"

namespace fs = std::filesystem;
using namespace dilithium::b200;
using Bytes = std::vector<uint8_t>;

namespace {

constexpr int kOk = 0, kReject = 1, kBadInput = 2;

// ---- files ---------------------------------------------------------------------------

bool slurp(const std::string& path, Bytes& out) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return false;
  out.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
  return true;
}

bool unhex(const Bytes& text, Bytes& out) {
  size_t len = text.size();
  while (len && (text[len - 1] == '\n' || text[len - 1] == '\r' || text[len - 1] == ' ')) --len;
  if (len % 2) return false;
  auto val = [](uint8_t c) -> int {
    if (c >= '0' && c <= '9') return c - '0';
    c |= 0x20;
    return (c >= 'a' && c <= 'f') ? c - 'a' + 10 : -1;
  };
  out.resize(len / 2);
  for (size_t i = 0; i < out.size(); ++i) {
    const int hi = val(text[2 * i]), lo = val(text[2 * i + 1]);
    if (hi < 0 || lo < 0) return false;
    out[i] = static_cast<uint8_t>(hi * 16 + lo);
  }
  return true;
}

// raw bytes of the expected length, else hex text of that length
bool load_object(const std::string& path, size_t want, Bytes& out) {
  Bytes raw;
  if (!slurp(path, raw)) return false;
  if (raw.size() == want) {
    out.swap(raw);
    return true;
  }
  return unhex(raw, out) && out.size() == want;
}

bool store(const std::string& path, std::span<const uint8_t> data, bool hex) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) return false;
  if (!hex) {
    out.write(reinterpret_cast<const char*>(data.data()), static_cast<std::streamsize>(data.size()));
  } else {
    std::string text(2 * data.size() + 1, '\n');
    for (size_t i = 0; i < data.size(); ++i) {
      text[2 * i] = "0123456789abcdef"[data[i] >> 4];
      text[2 * i + 1] = "0123456789abcdef"[data[i] & 15];
    }
    out << text;
  }
  return static_cast<bool>(out);
}

// ---- options -------------------------------------------------------------------------

struct Args {
  std::map<std::string, std::string> opt;
  std::vector<std::string> positional;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string get(const std::string& k, const std::string& dflt = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? dflt : it->second;
  }
  bool number(const std::string& k, size_t dflt, size_t& out) const {
    out = dflt;
    if (!has(k)) return true;
    const std::string& v = opt.at(k);
    if (v.empty() || v.find_first_not_of("0123456789") != std::string::npos) return false;
    out = std::stoull(v);
    return true;
  }
};

struct Command {
  std::set<std::string> options, required;
  bool positionals;
};

const std::map<std::string, Command>& commands() {
  static const std::set<std::string> common = {"--level", "--out-format", "--seed"};
  auto with = [&](std::set<std::string> extra) {
    extra.insert(common.begin(), common.end());
    return extra;
  };
  static const std::map<std::string, Command> table = {
      {"keygen", {with({"--pk", "--sk"}), {"--level", "--pk", "--sk"}, false}},
      {"sign", {with({"--sk", "--in", "--out"}), {"--level", "--sk", "--in", "--out"}, false}},
      {"verify", {with({"--pk", "--in", "--sig"}), {"--level", "--pk", "--in", "--sig"}, false}},
      {"batch-sign", {with({"--sk", "--out-dir", "--psi", "--workers", "--trace"}), {"--level", "--sk", "--out-dir"}, true}},
      {"batch-verify", {with({"--pk", "--sig-dir", "--workers"}), {"--level", "--pk", "--sig-dir"}, true}},
      {"bench", {with({"--phi", "--psi", "--workers", "--streams", "--reps", "--trace"}), {"--level"}, false}},
      {"sweep", {with({"--phi", "--workers", "--reps", "--psi-min", "--psi-max", "--psi-steps", "--streams-max"}),
                 {"--level"}, false}},
  };
  return table;
}

int usage(const std::string& why) {
  std::cerr << "error: " << why << "\n"
            << "usage: dilithium_b200 <keygen|sign|verify|batch-sign|batch-verify|bench|sweep> --level {2,3,5,44,65,87} ...\n";
  return kBadInput;
}

bool parse(int argc, char** argv, const Command& cmd, Args& a, std::string& why) {
  for (int i = 2; i < argc; ++i) {
    std::string tok = argv[i];
    if (tok.rfind("--", 0) == 0) {
      std::string val;
      const size_t eq = tok.find('=');
      if (eq != std::string::npos) {
        val = tok.substr(eq + 1);
        tok = tok.substr(0, eq);
      } else if (i + 1 < argc) {
        val = argv[++i];
      } else {
        why = tok + " needs a value";
        return false;
      }
      if (!cmd.options.count(tok)) {
        why = "unknown option " + tok;
        return false;
      }
      a.opt[tok] = val;
    } else if (cmd.positionals) {
      a.positional.push_back(tok);
    } else {
      why = "unexpected argument " + tok;
      return false;
    }
  }
  for (const auto& r : cmd.required)
    if (!a.has(r)) {
      why = r + " is required";
      return false;
    }
  if (cmd.positionals && a.positional.empty()) {
    why = "at least one message file is required";
    return false;
  }
  const std::string lv = a.get("--level");
  if (lv != "2" && lv != "3" && lv != "5" && lv != "44" && lv != "65" && lv != "87") {
    why = "--level must be 2, 3 or 5 (Dilithium round 3) or 44, 65 or 87 (ML-DSA, FIPS 204)";
    return false;
  }
  const std::string fmt = a.get("--out-format", "binary");
  if (fmt != "binary" && fmt != "hex") {
    why = "--out-format must be binary or hex";
    return false;
  }
  return true;
}

template <class Fn>
int with_level(const Args& a, Fn&& fn) {
  switch (std::stoi(a.get("--level"))) {
    case 2: return fn(std::integral_constant<int, 2>{});
    case 3: return fn(std::integral_constant<int, 3>{});
    case 5: return fn(std::integral_constant<int, 5>{});
    case 44: return fn(std::integral_constant<int, 44>{});
    case 65: return fn(std::integral_constant<int, 65>{});
    default: return fn(std::integral_constant<int, 87>{});
  }
}
template <int L>
constexpr Params params_of() {
  switch (L) {
    case 2: return kDilithium2;
    case 3: return kDilithium3;
    case 5: return kDilithium5;
    case 44: return kMLDSA44;
    case 65: return kMLDSA65;
    default: return kMLDSA87;
  }
}

// strict hint-section check of a signature (packing.hpp:122-140): what the reference's
// unpack_sig refuses and its CLI reports as exit 2 rather than "reject"
template <Params P>
bool sig_encoding_ok(std::span<const uint8_t> sig) {
  const uint8_t* h = sig.data() + P.ctilde_bytes + P.l * 32 * P.z_bits;
  size_t prev = 0;
  for (size_t i = 0; i < P.k; ++i) {
    const size_t cnt = h[P.omega + i];
    if (cnt < prev || cnt > P.omega) return false;
    for (size_t j = prev + 1; j < cnt; ++j)
      if (h[j] <= h[j - 1]) return false;
    prev = cnt;
  }
  for (size_t j = prev; j < P.omega; ++j)
    if (h[j] != 0) return false;
  return true;
}

// ---- commands ------------------------------------------------------------------------

int cmd_keygen(const Args& a) {
  SeedArray zeta;
  if (a.has("--seed")) {
    Bytes seed;
    const std::string hex = a.get("--seed");
    if (!unhex(Bytes(hex.begin(), hex.end()), seed) || seed.size() != kSeedBytes) {
      std::cerr << "error: --seed must be " << 2 * kSeedBytes << " hex characters\n";
      return kBadInput;
    }
    std::copy(seed.begin(), seed.end(), zeta.begin());
    std::cerr << "warning: deterministic seed supplied; keys derived from it are for testing only\n";
  } else {
    std::random_device rd;
    for (auto& b : zeta) b = static_cast<uint8_t>(rd());
  }
  const bool hex = a.get("--out-format") == "hex";
  return with_level(a, [&](auto lv) {
    constexpr Params P = params_of<decltype(lv)::value>();
    const auto [pk, sk] = keygen<P>(zeta);
    if (store(a.get("--pk"), pk, hex) && store(a.get("--sk"), sk, hex)) return kOk;
    std::cerr << "error: cannot write key files\n";
    return kBadInput;
  });
}

int cmd_sign(const Args& a) {
  const bool hex = a.get("--out-format") == "hex";
  return with_level(a, [&](auto lv) {
    constexpr Params P = params_of<decltype(lv)::value>();
    Bytes sk, msg;
    if (!load_object(a.get("--sk"), P.sk_bytes(), sk) || !slurp(a.get("--in"), msg)) {
      std::cerr << "error: cannot read secret key or message\n";
      return kBadInput;
    }
    const auto pre = make_precomp<P>(sk);
    if (!pre) {
      std::cerr << "error: malformed secret key\n";
      return kBadInput;
    }
    const auto sig = sign_with_precomp<P>(*pre, msg).sig;
    if (store(a.get("--out"), sig, hex)) return kOk;
    std::cerr << "error: cannot write signature\n";
    return kBadInput;
  });
}

int cmd_verify(const Args& a) {
  return with_level(a, [&](auto lv) {
    constexpr Params P = params_of<decltype(lv)::value>();
    Bytes pk, sig, msg;
    if (!load_object(a.get("--pk"), P.pk_bytes(), pk) || !load_object(a.get("--sig"), P.sig_bytes(), sig) ||
        !slurp(a.get("--in"), msg)) {
      std::cerr << "error: malformed or missing input file\n";
      return kBadInput;
    }
    if (!sig_encoding_ok<P>(sig)) {
      std::cerr << "error: malformed key or signature encoding\n";
      return kBadInput;
    }
    const bool ok = verify<P>(pk, msg, sig);
    std::cout << (ok ? "accept\n" : "reject\n");
    return ok ? kOk : kReject;
  });
}

// --trace: one CSV row per scheduler round, the reference tool's columns
// (dilithium_cli.cpp:128-134); `stream` is the CTA that ran the round
struct TraceFile {
  std::ofstream out;
  explicit TraceFile(const std::string& path) {
    if (path.empty()) return;
    out.open(path, std::ios::trunc);
    out << "stream,round,unfinished,assigned,speculative,idle_slots,newly_done\n";
  }
  void attach(BatchConfig& cfg) {
    if (!out.is_open()) return;
    cfg.trace = [this](const RoundTrace& t) {
      out << t.stream << ',' << t.round << ',' << t.unfinished << ',' << t.assigned << ',' << t.speculative
          << ',' << t.idle_slots << ',' << t.newly_done << '\n';
    };
  }
};

int cmd_batch_sign(const Args& a) {
  const bool hex = a.get("--out-format") == "hex";
  size_t psi = 0;
  if (!a.number("--psi", 0, psi)) return usage("--psi must be a number");
  return with_level(a, [&](auto lv) {
    constexpr Params P = params_of<decltype(lv)::value>();
    Bytes sk;
    if (!load_object(a.get("--sk"), P.sk_bytes(), sk)) {
      std::cerr << "error: cannot read secret key\n";
      return kBadInput;
    }
    const auto pre = make_precomp<P>(sk);
    if (!pre) {
      std::cerr << "error: malformed secret key\n";
      return kBadInput;
    }
    std::vector<Bytes> msgs(a.positional.size());
    for (size_t i = 0; i < msgs.size(); ++i)
      if (!slurp(a.positional[i], msgs[i])) {
        std::cerr << "error: cannot read " << a.positional[i] << "\n";
        return kBadInput;
      }
    if (psi > msgs.size()) {  // the reference tool's rule (dilithium_cli.cpp:233)
      std::cerr << "error: --psi must not exceed the number of messages\n";
      return kBadInput;
    }
    std::vector<SignJob<P>> jobs;
    for (const auto& m : msgs) jobs.push_back({&*pre, m});
    BatchConfig cfg;
    cfg.psi = psi;
    TraceFile trace(a.get("--trace"));
    trace.attach(cfg);
    BatchStats st;
    const auto sigs = batch_sign<P>(std::span<const SignJob<P>>(jobs), cfg, &st);
    if (!st.failed_tasks.empty()) {
      std::cerr << "error: " << st.failed_tasks.size() << " task(s) exhausted the nonce space\n";
      return kBadInput;
    }
    std::error_code ec;
    fs::create_directories(a.get("--out-dir"), ec);
    for (size_t i = 0; i < sigs.size(); ++i) {
      const auto name = fs::path(a.positional[i]).filename().string() + ".sig";
      if (!store((fs::path(a.get("--out-dir")) / name).string(), sigs[i], hex)) {
        std::cerr << "error: cannot write " << name << "\n";
        return kBadInput;
      }
    }
    return kOk;
  });
}

int cmd_batch_verify(const Args& a) {
  return with_level(a, [&](auto lv) {
    constexpr Params P = params_of<decltype(lv)::value>();
    Bytes pk;
    if (!load_object(a.get("--pk"), P.pk_bytes(), pk)) {
      std::cerr << "error: cannot read public key\n";
      return kBadInput;
    }
    const size_t n = a.positional.size();
    std::vector<Bytes> msgs(n), sigs(n);
    for (size_t i = 0; i < n; ++i) {
      if (!slurp(a.positional[i], msgs[i])) {
        std::cerr << "error: cannot read " << a.positional[i] << "\n";
        return kBadInput;
      }
      const auto name = fs::path(a.positional[i]).filename().string() + ".sig";
      if (!load_object((fs::path(a.get("--sig-dir")) / name).string(), P.sig_bytes(), sigs[i]))
        sigs[i].clear();  // missing or wrong-size signature: rejected below
    }
    std::vector<VerifyJob<P>> jobs(n);
    for (size_t i = 0; i < n; ++i) jobs[i] = {pk, msgs[i], sigs[i]};
    const auto flags = batch_verify<P>(std::span<const VerifyJob<P>>(jobs));
    bool all = true;
    for (size_t i = 0; i < n; ++i) {
      std::cout << a.positional[i] << ": " << (flags[i] ? "accept" : "reject") << "\n";
      all = all && flags[i];
    }
    return all ? kOk : kReject;
  });
}

template <class Fn>
double median_seconds(size_t reps, Fn&& fn) {
  fn();  // warm-up: arenas, first-launch costs
  std::vector<double> t(reps);
  for (auto& x : t) {
    const auto t0 = std::chrono::steady_clock::now();
    fn();
    x = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int cmd_bench(const Args& a) {
  size_t phi, psi, workers, streams, reps;
  if (!a.number("--phi", 1000, phi) || !a.number("--psi", 0, psi) || !a.number("--workers", 1, workers) ||
      !a.number("--streams", 1, streams) || !a.number("--reps", 5, reps) || phi == 0 || reps == 0)
    return usage("bench options must be positive numbers");
  if (psi > phi) return usage("--psi must not exceed --phi");
  if (streams > 64) return usage("--streams must be at most 64");
  return with_level(a, [&](auto lv) {
    constexpr Params P = params_of<decltype(lv)::value>();
    std::mt19937_64 rng(20221112);
    std::vector<SeedArray> zetas(phi);
    for (auto& z : zetas)
      for (auto& b : z) b = static_cast<uint8_t>(rng());
    const auto [pk, sk] = keygen<P>(zetas[0]);
    const auto pre = make_precomp<P>(sk);
    // the reference bench signs 59-byte messages (dilithium_cli.cpp:366-370)
    std::vector<Bytes> msgs(phi, Bytes(59));
    for (auto& m : msgs)
      for (auto& b : m) b = static_cast<uint8_t>(rng());
    std::vector<SignJob<P>> jobs;
    for (const auto& m : msgs) jobs.push_back({&*pre, m});
    BatchConfig cfg;
    cfg.psi = psi;
    TraceFile trace(a.get("--trace"));  // rounds of every timed repetition are appended
    trace.attach(cfg);
    BatchStats st;
    std::vector<SigBytes<P>> sigs;
    std::cout << "schema,mode,op,level,phi,psi,workers,streams,reps,throughput_ops_s,mean_latency_us,attempts_mean\n";
    auto row = [&](const char* op, double sec, const std::string& attempts) {
      std::printf("1,batch-gpu,%s,%d,%zu,%zu,%zu,%zu,%zu,%.1f,%.3f,%s\n", op, P.level, phi, psi, workers,
                  streams, reps, phi / sec, sec / phi * 1e6, attempts.c_str());
    };
    // --streams S: S independent engines over a contiguous task partition (the reference
    // tool's multi-engine mode, dilithium_cli.cpp:319-339); here S contexts on GPU 0
    std::unique_ptr<ShardedEngine> sharded;
    if (streams > 1) sharded = std::make_unique<ShardedEngine>(std::vector<int>(streams, 0));
    row("keygen", median_seconds(reps, [&] {
          if (sharded) sharded->batch_keygen<P>(std::span<const SeedArray>(zetas));
          else batch_keygen<P>(std::span<const SeedArray>(zetas));
        }), "");
    const double ts = median_seconds(reps, [&] {
      sigs = sharded ? sharded->batch_sign<P>(std::span<const SignJob<P>>(jobs), cfg, &st)
                     : batch_sign<P>(std::span<const SignJob<P>>(jobs), cfg, &st);
    });
    char att[32];
    std::snprintf(att, sizeof att, "%.3f", double(st.accepted_attempt_sum) / phi);
    row("sign", ts, att);
    std::vector<VerifyJob<P>> vj(phi);
    for (size_t i = 0; i < phi; ++i) vj[i] = {pk, msgs[i], sigs[i]};
    std::vector<uint8_t> flags;
    row("verify", median_seconds(reps, [&] {
          flags = sharded ? sharded->batch_verify<P>(std::span<const VerifyJob<P>>(vj))
                          : batch_verify<P>(std::span<const VerifyJob<P>>(vj));
        }), "");
    for (auto f : flags)
      if (!f) {
        std::cerr << "error: bench produced a signature that does not verify\n";
        return kBadInput;
      }
    return kOk;
  });
}

// sweep: the reference tool's sensitivity study (tools/dilithium_cli.cpp:448-514)
// with its CSV schema and its three modes.  On the GPU engine `psi` is the number of resident
// attempt slots of the batch and `streams` the number of in-flight batches the task list is cut
// into (dlb_sign_submit x S, dlb_sign_wait x S -- the paper's streams).  Times cover the call with
// pinned host buffers in and out (messages up, signatures down); medians over --reps.
int cmd_sweep(const Args& a) {
  size_t phi, workers, reps, psi_min, psi_max, psi_steps, streams_max;
  if (!a.number("--phi", 10000, phi) || !a.number("--workers", 1, workers) || !a.number("--reps", 5, reps) ||
      !a.number("--psi-min", 1, psi_min) || !a.number("--psi-max", 0, psi_max) ||
      !a.number("--psi-steps", 6, psi_steps) || !a.number("--streams-max", 8, streams_max) || phi == 0 ||
      reps == 0)
    return usage("sweep options must be positive numbers");
  if (streams_max > 16) return usage("--streams-max must be at most 16 (batches in flight per engine)");
  return with_level(a, [&](auto lv) {
    constexpr Params P = params_of<decltype(lv)::value>();
    Engine& eng = Engine::instance();
    std::mt19937_64 rng(20221112);
    SeedArray zeta;
    for (auto& b : zeta) b = static_cast<uint8_t>(rng());
    const auto [pk, sk] = keygen<P>(zeta);
    (void)pk;
    // 59-byte messages like the reference sweep (dilithium_cli.cpp:458-462), flat in pinned memory
    constexpr size_t kMsg = 59;
    auto* msgs = static_cast<uint8_t*>(dlb_host_alloc(phi * kMsg + 8));
    auto* off = static_cast<uint64_t*>(dlb_host_alloc((phi + 1) * 8));
    auto* sigs = static_cast<uint8_t*>(dlb_host_alloc(phi * P.sig_bytes() + 8));
    auto* att = static_cast<uint32_t*>(dlb_host_alloc(phi * 4));
    auto* skp = static_cast<uint8_t*>(dlb_host_alloc(P.sk_bytes()));
    if (!msgs || !off || !sigs || !att || !skp) throw std::runtime_error("pinned allocation failed");
    for (size_t i = 0; i < phi * kMsg; ++i) msgs[i] = static_cast<uint8_t>(rng());
    for (size_t i = 0; i <= phi; ++i) off[i] = i * kMsg;
    std::memcpy(skp, sk.data(), P.sk_bytes());
    std::cout << "schema,mode,op,level,phi,psi,workers,streams,reps,throughput_ops_s,mean_latency_us,attempts_mean\n";
    double attempts_mean = 0;
    auto timed = [&](size_t n, size_t psi, size_t streams) {
      std::vector<uint64_t> tickets(streams);
      for (size_t s = 0; s < streams; ++s) {
        const size_t lo = n * s / streams, hi = n * (s + 1) / streams;
        const size_t part_psi = psi == 0 ? 0 : std::max<size_t>(1, std::min(psi, hi - lo));
        check(dlb_sign_submit(eng.ctx(), P.level, 0, skp, 0, hi - lo, nullptr, msgs + lo * kMsg, off /* equal lengths: relative offsets */, nullptr, part_psi,
                              1, sigs + lo * P.sig_bytes(), att + lo, nullptr, &tickets[s]),
              "dlb_sign_submit");
      }
      for (size_t s = 0; s < streams; ++s) check(dlb_sign_wait(eng.ctx(), tickets[s], nullptr), "dlb_sign_wait");
      uint64_t sum = 0;
      for (size_t i = 0; i < n; ++i) sum += att[i];
      attempts_mean = double(sum) / double(n);
    };
    auto point = [&](const char* mode, size_t n, size_t psi, size_t streams) {
      const double sec = median_seconds(reps, [&] { timed(n, psi, streams); });
      std::printf("1,%s,sign,%d,%zu,%zu,%zu,%zu,%zu,%.1f,%.3f,%.3f\n", mode, P.level, n, psi, workers, streams,
                  reps, n / sec, sec / n * 1e6, attempts_mean);
    };
    // throughput vs psi at fixed phi
    psi_max = std::min(psi_max == 0 ? phi : psi_max, phi);
    psi_min = std::max<size_t>(1, std::min(psi_min, psi_max));
    const size_t steps = std::max<size_t>(2, psi_steps);
    for (size_t st = 0; st < steps; ++st) point("sweep-psi", phi, psi_min + (psi_max - psi_min) * st / (steps - 1), 1);
    // throughput vs batch size at the engine's default psi
    for (size_t batch = std::max<size_t>(1, phi / 16);; batch *= 2) {
      if (batch >= phi) {
        point("sweep-batch", phi, 0, 1);
        break;
      }
      point("sweep-batch", batch, 0, 1);
    }
    // throughput vs batches in flight at full phi
    for (size_t st = 1; st <= streams_max; st *= 2) point("sweep-streams", phi, 0, st);
    dlb_host_free(msgs);
    dlb_host_free(off);
    dlb_host_free(sigs);
    dlb_host_free(att);
    dlb_host_free(skp);
    return kOk;
  });
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage("missing subcommand");
  const std::string name = argv[1];
  const auto it = commands().find(name);
  if (it == commands().end()) return usage("unknown subcommand " + name);
  Args a;
  std::string why;
  if (!parse(argc, argv, it->second, a, why)) return usage(why);
  try {
    if (name == "keygen") return cmd_keygen(a);
    if (name == "sign") return cmd_sign(a);
    if (name == "verify") return cmd_verify(a);
    if (name == "batch-sign") return cmd_batch_sign(a);
    if (name == "batch-verify") return cmd_batch_verify(a);
    if (name == "sweep") return cmd_sweep(a);
    return cmd_bench(a);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kBadInput;
  }
}
