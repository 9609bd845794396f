"""Steps in flight, many runs, levels interleaved in one engine context: prints each run's
throughput and, for a run well below the level's best, the per-ticket claim / commit timeline
next to the host's submit / wait times.  Usage: python scripts/pipe_stress.py [ROUNDS] [DEPTH] [STEPS]"""
import ctypes as C
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2211_12265_b200 import Engine, LEVELS
from paper_2211_12265_b200.engine import SignStats

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 6
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 32
levels = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [2, 3, 65, 5, 87, 44]
n = 100000
dev = torch.device("cuda", 0)
eng = Engine(0)
lib, ctx = eng.lib, eng.ctx
p = lambda t: C.c_void_p(t.data_ptr())
rng = np.random.default_rng(5)
d_msgs = torch.from_numpy(rng.integers(0, 256, (n, 32), dtype=np.uint8)).to(dev)
d_off = torch.from_numpy((np.arange(n + 1, dtype=np.int64) * 32)).to(dev)
state = {}
for level in levels:
    sgb = LEVELS[level][4]
    pks, sks = eng.batch_keygen(level, np.arange(32, dtype=np.uint8))
    state[level] = (torch.from_numpy(sks[0].copy()).to(dev),
                    [(torch.zeros((n, sgb), dtype=torch.uint8, device=dev), torch.zeros(n, dtype=torch.int32, device=dev),
                      torch.zeros(n, dtype=torch.uint8, device=dev)) for _ in range(depth)])


def run(level, steps_now):
    d_sk, ring = state[level]
    inflight, stats, host = [], [], []
    t00 = time.perf_counter()

    def wait(t):
        st = SignStats()
        a = time.perf_counter()
        rc = lib.dlb_sign_wait(ctx, t, C.byref(st))
        b = time.perf_counter()
        assert rc == 0, "dlb_sign_wait: %d" % rc
        stats.append(st)
        host.append(("wait", t, (a - t00) * 1e3, (b - t00) * 1e3))
    for i in range(steps_now):
        if len(inflight) >= depth:
            wait(inflight.pop(0))
        sig, att, fail = ring[i % depth]
        t = C.c_uint64(0)
        a = time.perf_counter()
        assert lib.dlb_sign_submit_dev(ctx, level, 0, p(d_sk), 0, n, None, p(d_msgs), p(d_off), None, 0, 1,
                                       p(sig), p(att), p(fail), C.byref(t)) == 0
        b = time.perf_counter()
        host.append(("submit", t.value, (a - t00) * 1e3, (b - t00) * 1e3))
        inflight.append(t.value)
    for t in inflight:
        wait(t)
    return stats, host


import os
mimic = os.environ.get("MIMIC", "")
if "s" in mimic:  # bench.py's levels leg runs on a torch side stream
    side = torch.cuda.Stream(dev)
    eng.set_stream(side.cuda_stream)
d_flags = torch.zeros(n, dtype=torch.uint8, device=dev)


def sync_legs(level):  # the synchronous sign / verify / keygen legs bench.py times before the pipe
    k, l, pkb, skb, sgb = LEVELS[level]
    d_sk, ring = state[level]
    st = SignStats()
    d_pk = torch.zeros((n, pkb), dtype=torch.uint8, device=dev)
    d_sks = torch.zeros((n, skb), dtype=torch.uint8, device=dev)
    for _ in range(3):
        assert lib.dlb_sign_batch_dev(ctx, level, n, p(d_sk), 0, p(d_msgs), p(d_off), None, 0, 1,
                                      p(ring[0][0]), p(ring[0][1]), p(ring[0][2]), C.byref(st)) == 0
    torch.cuda.synchronize()
    for _ in range(6):
        assert lib.dlb_keygen_batch_dev(ctx, level, n, p(d_msgs), p(d_pk), p(d_sks)) == 0
    torch.cuda.synchronize()
    for _ in range(6):
        assert lib.dlb_verify_batch_dev(ctx, level, n, p(d_pk), pkb, p(d_msgs), p(d_off), p(ring[0][0]), p(d_flags)) == 0
    torch.cuda.synchronize()


best = {}
for r in range(rounds):
    for level in levels:
        if "l" in mimic:
            sync_legs(level)
        run(level, depth)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        stats, host = run(level, steps)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / steps
        rate = n / ms / 1e3
        best[level] = max(best.get(level, 0.0), rate)
        slow = rate < 0.9 * best[level] or (r == 0 and os.environ.get("TRACE"))
        print("round %d level %2d: %.3f ms/step = %.2f M/s%s" % (r, level, ms, rate, "  <-- slow" if slow else ""), flush=True)
        if slow:
            base = min(s.t_first_start_ns for s in stats)
            for i, s in enumerate(stats):
                print("  %2d claim %.2f..%.2f commit %.2f..%.2f ms  attempts/sig %.2f" % (
                    i, (s.t_first_start_ns - base) / 1e6, (s.t_last_start_ns - base) / 1e6,
                    (s.t_first_exit_ns - base) / 1e6, (s.t_last_exit_ns - base) / 1e6, s.attempts / n))
            for h in host:
                if h[3] - h[2] > 1.0:
                    print("  host %-6s ticket %d: %.2f -> %.2f ms" % h)
eng.close()
