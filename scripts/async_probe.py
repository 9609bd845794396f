"""Batches in flight: sequential dlb_sign_batch calls vs dlb_sign_submit / dlb_sign_wait pipelines
(host pinned buffers in and out).  Usage: python scripts/async_probe.py [level] [depth]"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2211_12265_b200 import Engine
from paper_2211_12265_b200.engine import LEVELS


def pinned(eng, shape, dtype=np.uint8):
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    p = eng.lib.dlb_host_alloc(nbytes)
    buf = (C.c_uint8 * nbytes).from_address(p)
    return np.frombuffer(buf, dtype=dtype).reshape(shape)


def run(level, n, batches, depth, eng, sk, reps=3):
    sgb = LEVELS[level][4]
    rng = np.random.default_rng(n)
    msgs = [(rng.integers(0, 256, n * 32, dtype=np.uint8), np.arange(n + 1, dtype=np.uint64) * 32)
            for _ in range(batches)]
    outs = [pinned(eng, (n, sgb)) for _ in range(batches)]
    ref = []
    best_seq = best_pipe = 1e9
    for r in range(reps):
        t0 = time.perf_counter()
        for b in range(batches):
            h = eng.sign_submit(level, sk, msgs[b], out=outs[b])
            eng.sign_wait(h)
        best_seq = min(best_seq, time.perf_counter() - t0)
        if r == 0:
            ref = [o.copy() for o in outs]
            for o in outs:
                o[:] = 0
    for r in range(reps):
        t0 = time.perf_counter()
        hs = []
        spec = 0
        att = 0
        for b in range(batches):
            if len(hs) >= depth:
                st = eng.sign_wait(hs.pop(0))[3]
                spec += st["speculative"]; att += st["attempts"]
            hs.append(eng.sign_submit(level, sk, msgs[b], out=outs[b]))
        for h in hs:
            st = eng.sign_wait(h)[3]
            spec += st["speculative"]; att += st["attempts"]
        best_pipe = min(best_pipe, time.perf_counter() - t0)
    same = all(np.array_equal(a, b) for a, b in zip(ref, outs))
    tot = n * batches
    print(f"level {level} n={n} x{batches} depth={depth}: sequential {tot / best_seq / 1e6:.2f} M/s "
          f"({best_seq * 1e3 / batches:.2f} ms/batch), in flight {tot / best_pipe / 1e6:.2f} M/s "
          f"({best_pipe * 1e3 / batches:.2f} ms/batch), bytes equal: {same}, "
          f"speculative share {spec / max(att, 1):.3f}, attempts/sig {att / tot:.2f}", flush=True)


if __name__ == "__main__":
    level = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    depth = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    eng = Engine(0)
    pks, sks = eng.batch_keygen(level, np.arange(32, dtype=np.uint8))
    sk = sks[0]
    nb = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    run(level, 100000, nb, depth, eng, sk)
    if len(sys.argv) <= 3:
        run(level, 10000, 10, 10, eng, sk)
        run(level, 10000, 40, 8, eng, sk)
        run(level, 1000, 32, 8, eng, sk)
    eng.close()
