"""world_size-2 gloo worker for tests/test_dist_cpu.py: the multi-GPU plumbing of
bench.py (barrier, max-over-ranks timing, per-rank shards) on CPU."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2211_12265_b200.sharding import merge_shard_stats, shard_ranges  # noqa: E402

d = bench.Dist()
d.init(use_cuda=False)
d.barrier()
n = 1001
lo, hi = shard_ranges(n, d.world)[d.rank]
t_max = d.max(10.0 + d.rank, use_cuda=False)       # slowest rank defines the step time
total = d.sum(float(hi - lo), use_cuda=False)      # shards cover the batch exactly once
msgs, off = bench.make_inputs(4, 20221112 + d.rank)
# every rank reports what an engine would: counters of its shard and the LOCAL indices of failed
# tasks (first and last task of the shard); rank 0 merges them like ShardedEngine / MultiEngine do
mine = {"rounds": 10 + d.rank, "attempts": 1000 * (d.rank + 1), "speculative": 7 * d.rank,
        "idle_slot_rounds": d.rank, "accepted_attempt_sum": 900 * (d.rank + 1), "failed_tasks": 2,
        "failed_local": [0, hi - lo - 1], "range": [lo, hi]}
merged = None
if d.pg:
    gathered = [None] * d.world
    d.pg.all_gather_object(gathered, mine)
    if d.rank == 0:
        merged = merge_shard_stats(gathered, [g["failed_local"] for g in gathered],
                                   [tuple(g["range"]) for g in gathered])
d.barrier()
if d.rank == 0:
    print(json.dumps({"t_max": t_max, "total": total, "world": d.world}))
    if merged is not None:
        with open(os.path.join(sys.argv[1], "merged.json"), "w") as f:
            json.dump({"stats": merged[0], "failed": merged[1]}, f)
with open(os.path.join(sys.argv[1], "rank%d.json" % d.rank), "w") as f:
    json.dump({"lo": lo, "hi": hi, "first": msgs[0].tolist()}, f)
d.done()
