"""End-to-end sign pipeline from pinned host buffers (the bench's e2e shape): per-step host times.
Usage: [DLB_ZERO_COPY_MAX=0] python scripts/e2e_probe.py [DEPTH] [STEPS]"""
import ctypes as C
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2211_12265_b200 import Engine, LEVELS
from paper_2211_12265_b200.engine import SignStats

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 16
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 48
level, n = 2, 100000
eng = Engine(0)
lib, ctx = eng.lib, eng.ctx
sgb = LEVELS[level][4]
pks, sks = eng.batch_keygen(level, np.arange(32, dtype=np.uint8))
rng = np.random.default_rng(5)
h_msgs = torch.from_numpy(rng.integers(0, 256, (n, 32), dtype=np.uint8)).pin_memory()
h_off = torch.from_numpy((np.arange(n + 1, dtype=np.int64) * 32)).pin_memory()
h_sk = torch.from_numpy(sks[0].copy()).pin_memory()
ring = [torch.zeros((n, sgb), dtype=torch.uint8).pin_memory() for _ in range(depth)]
vp = lambda t: C.c_void_p(t.data_ptr())


def run(k, show=False):
    inflight, waits, subs = [], [], []
    t00 = time.perf_counter()
    for i in range(k):
        if len(inflight) >= depth:
            a = time.perf_counter()
            assert lib.dlb_sign_wait(ctx, inflight.pop(0), None) == 0
            waits.append((time.perf_counter() - a) * 1e3)
        t = C.c_uint64(0)
        a = time.perf_counter()
        assert lib.dlb_sign_submit(ctx, level, 0, vp(h_sk), 0, n, None, vp(h_msgs), vp(h_off), None, 0, 1,
                                   vp(ring[i % depth]), None, None, C.byref(t)) == 0
        subs.append((time.perf_counter() - a) * 1e3)
        inflight.append(t.value)
    for t in inflight:
        a = time.perf_counter()
        assert lib.dlb_sign_wait(ctx, t, None) == 0
        waits.append((time.perf_counter() - a) * 1e3)
    tot = (time.perf_counter() - t00) * 1e3
    if show:
        print("total %.1f ms = %.2f M sign/s; submit mean %.3f max %.3f ms; waits: %s" % (
            tot, n * k / tot / 1e3, np.mean(subs), np.max(subs), " ".join("%.1f" % w for w in waits)))
    return tot


run(depth + 4)
torch.cuda.synchronize()
for _ in range(3):
    run(steps, show=True)
    torch.cuda.synchronize()
eng.close()
