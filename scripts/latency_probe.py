"""Small-batch latency through the host API (n = 1 .. 10k), median of 21 calls."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2211_12265_b200 import Engine
eng = Engine(0)
rng = np.random.default_rng(11)
for level in (2, 3, 5):
    pk, sk = eng.batch_keygen(level, rng.integers(0, 256, 32, dtype=np.uint8))
    for n in (1, 10, 100, 1000, 10000):
        msgs = rng.integers(0, 256, 32 * n, dtype=np.uint8)
        off = np.arange(n + 1, dtype=np.uint64) * 32
        z = rng.integers(0, 256, (n, 32), dtype=np.uint8)
        sigs = eng.batch_sign(level, sk[0], (msgs, off))
        def med(fn):
            fn(); fn()
            ts = []
            for _ in range(21):
                t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
            return np.median(ts) * 1e3
        ts = med(lambda: eng.batch_sign(level, sk[0], (msgs, off)))
        tv = med(lambda: eng.batch_verify(level, pk[0], (msgs, off), sigs))
        tk = med(lambda: eng.batch_keygen(level, z))
        print("L%d n=%5d  sign %.3f ms  verify %.3f ms  keygen %.3f ms" % (level, n, ts, tv, tk), flush=True)
