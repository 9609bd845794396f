"""Device-resident sign: one synchronous call per step vs steps in flight, with the per-ticket
claim / commit timeline.  Usage: python scripts/pipe_probe.py LEVEL [N] [DEPTH] [STEPS]"""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2211_12265_b200 import Engine, LEVELS
from paper_2211_12265_b200.engine import SignStats

level = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
depth = int(sys.argv[3]) if len(sys.argv) > 3 else 3
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 12
dev = torch.device("cuda", 0)
eng = Engine(0)
lib, ctx = eng.lib, eng.ctx
sgb = LEVELS[level][4]
pks, sks = eng.batch_keygen(level, np.arange(32, dtype=np.uint8))
rng = np.random.default_rng(5)
d_msgs = torch.from_numpy(rng.integers(0, 256, (n, 32), dtype=np.uint8)).to(dev)
d_off = torch.from_numpy((np.arange(n + 1, dtype=np.int64) * 32)).to(dev)
d_sk = torch.from_numpy(sks[0].copy()).to(dev)
ring = [(torch.zeros((n, sgb), dtype=torch.uint8, device=dev), torch.zeros(n, dtype=torch.int32, device=dev),
         torch.zeros(n, dtype=torch.uint8, device=dev)) for _ in range(depth)]
p = lambda t: C.c_void_p(t.data_ptr())


def run(depth_now, steps_now, show=False):
    inflight, stats = [], []

    def wait(t):
        st = SignStats()
        rc = lib.dlb_sign_wait(ctx, t, C.byref(st))
        assert rc == 0, "dlb_sign_wait: %d" % rc
        stats.append(st)
    for i in range(steps_now):
        if len(inflight) >= depth_now:
            wait(inflight.pop(0))
        sig, att, fail = ring[i % depth]
        t = C.c_uint64(0)
        assert lib.dlb_sign_submit_dev(ctx, level, 0, p(d_sk), 0, n, None, p(d_msgs), p(d_off), None, 0, 1,
                                       p(sig), p(att), p(fail), C.byref(t)) == 0
        inflight.append(t.value)
    for t in inflight:
        wait(t)
    if show:
        base = min(s.t_first_start_ns for s in stats)
        for i, s in enumerate(stats):
            print("  %2d claim %.2f..%.2f commit %.2f..%.2f ms  attempts/sig %.2f spec %.3f" % (
                i, (s.t_first_start_ns - base) / 1e6, (s.t_last_start_ns - base) / 1e6,
                (s.t_first_exit_ns - base) / 1e6, (s.t_last_exit_ns - base) / 1e6,
                s.attempts / n, s.speculative / max(1, s.attempts)))


for d in (1, depth):
    run(d, depth)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(d, steps, show=(d == depth))
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print("level %d n=%d depth=%d: %.3f ms/step = %.2f M/s" % (level, n, d, ms, n / ms / 1e3))
eng.close()
