"""Sign throughput by key mode (device-resident inputs): one shared key, a table of T keys indexed
per task, one key per task.  Usage: python scripts/keymode_probe.py [LEVEL] [N]"""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2211_12265_b200 import Engine, LEVELS
from paper_2211_12265_b200.engine import SignStats

level = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
dev = torch.device("cuda", 0)
eng = Engine(0)
lib, ctx = eng.lib, eng.ctx
k, l, pkb, skb, sgb = LEVELS[level]
rng = np.random.default_rng(3)
p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
zetas = torch.from_numpy(rng.integers(0, 256, (n, 32), dtype=np.uint8)).to(dev)
d_pks = torch.empty((n, pkb), dtype=torch.uint8, device=dev)
d_sks = torch.empty((n, skb), dtype=torch.uint8, device=dev)
assert lib.dlb_keygen_batch_dev(ctx, level, n, p(zetas), p(d_pks), p(d_sks)) == 0
d_msgs = torch.from_numpy(rng.integers(0, 256, (n, 32), dtype=np.uint8)).to(dev)
d_off = (torch.arange(n + 1, dtype=torch.int64) * 32).to(dev)
depth = 8
ring = [(torch.empty((n, sgb), dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
         torch.empty(n, dtype=torch.uint8, device=dev)) for _ in range(depth)]
d_flags = torch.empty(n, dtype=torch.uint8, device=dev)


import os
def run(n_keys, stride, kidx, steps, show=False):
    inflight, stats = [], []
    for i in range(steps):
        if len(inflight) >= depth:
            st = SignStats()
            assert lib.dlb_sign_wait(ctx, inflight.pop(0), C.byref(st)) == 0
            stats.append(st)
        sig, att, fail = ring[i % depth]
        t = C.c_uint64(0)
        rc = lib.dlb_sign_submit_dev(ctx, level, n_keys, p(d_sks), stride, n, p(kidx), p(d_msgs), p(d_off), None, 0, 1,
                                     p(sig), p(att), p(fail), C.byref(t))
        assert rc == 0, rc
        inflight.append(t.value)
    for t in inflight:
        st = SignStats()
        assert lib.dlb_sign_wait(ctx, t, C.byref(st)) == 0
        stats.append(st)
    if show and os.environ.get("TRACE"):
        base = min(s.t_first_start_ns for s in stats)
        for i, s in enumerate(stats):
            print("  %2d claim %.2f..%.2f commit %.2f..%.2f ms  attempts/sig %.2f spec %.3f" % (
                i, (s.t_first_start_ns - base) / 1e6, (s.t_last_start_ns - base) / 1e6,
                (s.t_first_exit_ns - base) / 1e6, (s.t_last_exit_ns - base) / 1e6,
                s.attempts / n, s.speculative / max(1, s.attempts)))


modes = [("one shared key", 0, 0, None)]
for T in (16, 1024):
    modes.append(("table of %d keys" % T, T, skb, torch.from_numpy(rng.integers(0, T, n).astype(np.uint32)).to(dev)))
modes.append(("one key per task", 0, skb, None))
if os.environ.get("ONLY"):  # e.g. ONLY="one key per task" ONCE=1 under ncu: one synchronous batch of that mode
    modes = [m for m in modes if m[0] == os.environ["ONLY"]]
if os.environ.get("ONCE"):
    for name, nk, stride, kidx in modes:
        depth = 1
        run(nk, stride, kidx, 2)
    eng.close()
    sys.exit(0)
for name, nk, stride, kidx in modes:
    for d_, steps in ((1, 6), (depth, 32)):
        depth_saved = depth
        depth = d_
        run(nk, stride, kidx, 2 * d_)  # every arena set the timed run will use exists afterwards
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(nk, stride, kidx, steps, show=(d_ > 1))
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        depth = depth_saved
        print("level %d n=%d %-18s in flight %d: %.3f ms/batch = %.2f M sign/s" % (level, n, name, d_, ms, n / ms / 1e3))
    # the signatures of the last batch verify under the keys they were made with
    sig = ring[(32 - 1) % depth][0]
    if kidx is None and stride:
        assert lib.dlb_verify_batch_dev(ctx, level, n, p(d_pks), pkb, p(d_msgs), p(d_off), p(sig), p(d_flags)) == 0
        assert bool(d_flags.all().item())
eng.close()
