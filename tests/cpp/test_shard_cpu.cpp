// CPU-only: the partition and the stats / failed-index rebasing that ShardedEngine applies
// (include/dilithium_b200/api.hpp; reference partition tools/dilithium_cli.cpp:319-339).
#include <cstdio>
#include <numeric>

#include "dilithium_b200/api.hpp"

using namespace dilithium::b200;

static int fails = 0;
#define CHECK(x) do { if (!(x)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #x); ++fails; } } while (0)

int main() {
  for (size_t n : {size_t{0}, size_t{1}, size_t{7}, size_t{1001}, size_t{100000}})
    for (size_t G : {size_t{1}, size_t{2}, size_t{3}, size_t{5}, size_t{8}}) {
      const auto b = shard_bounds(n, G);
      CHECK(b.size() == G + 1 && b.front() == 0 && b.back() == n);
      size_t lo = ~size_t{0}, hi = 0;
      for (size_t g = 0; g < G; ++g) {
        CHECK(b[g] <= b[g + 1] && b[g] == n * g / G);
        lo = std::min(lo, b[g + 1] - b[g]);
        hi = std::max(hi, b[g + 1] - b[g]);
      }
      CHECK(hi - lo <= 1);  // shards differ by at most one task
    }
  // three uneven shards of 1001 tasks: 333 / 334 / 334
  const auto b = shard_bounds(1001, 3);
  CHECK(b[1] == 333 && b[2] == 667);
  std::vector<BatchStats> parts(3);
  for (size_t g = 0; g < 3; ++g) {
    parts[g].rounds = 10 + g;
    parts[g].attempts = 1000 * (g + 1);
    parts[g].speculative = 7 * g;
    parts[g].idle_slot_rounds = g;
    parts[g].accepted_attempt_sum = 900 * (g + 1);
  }
  parts[0].failed_tasks = {0, 332};
  parts[2].failed_tasks = {5, 333};
  const BatchStats m = merge_shard_stats(parts, b);
  CHECK(m.rounds == 33 && m.attempts == 6000 && m.speculative == 21 && m.idle_slot_rounds == 3 &&
        m.accepted_attempt_sum == 5400);
  CHECK((m.failed_tasks == std::vector<size_t>{0, 332, 672, 1000}));
  parts[1].failed_tasks = {334};  // outside a 334-task shard
  bool threw = false;
  try { merge_shard_stats(parts, b); } catch (const std::out_of_range&) { threw = true; }
  CHECK(threw);
  threw = false;
  try { shard_bounds(5, 0); } catch (const std::invalid_argument&) { threw = true; }
  CHECK(threw);
  std::printf(fails ? "shard test: %d failures\n" : "shard test: all passed\n", fails);
  return fails ? 1 : 0;
}
