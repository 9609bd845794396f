"""Psi (resident attempt slots) sweep for small batches: host API latency, median of 21."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2211_12265_b200 import Engine
eng = Engine(0)
rng = np.random.default_rng(11)
level = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pk, sk = eng.batch_keygen(level, rng.integers(0, 256, 32, dtype=np.uint8))
for n in (1, 10, 100, 1000, 4000, 10000):
    msgs = rng.integers(0, 256, 32 * n, dtype=np.uint8)
    off = np.arange(n + 1, dtype=np.uint64) * 32
    row = []
    for mult in (0, 3, 5, 9, 16):
        psi = mult * n
        def fn(): return eng.batch_sign(level, sk[0], (msgs, off), psi=psi, return_info=True)
        fn(); fn()
        ts, ex = [], 0
        for _ in range(21):
            t0 = time.perf_counter(); r = fn(); ts.append(time.perf_counter() - t0); ex = r[3]["attempts"] / n
        row.append("psi=%2dn %.3f ms (%.1f att)" % (mult, np.median(ts) * 1e3, ex))
    print("L%d n=%5d  " % (level, n) + "  ".join(row), flush=True)
