"""Device-side rate of one large batch and of a 100k batch (A/B of library builds via DLB_LIB)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2211_12265_b200 import Engine
from scripts.async_probe import pinned
from paper_2211_12265_b200.engine import LEVELS
level = int(sys.argv[1]) if len(sys.argv) > 1 else 2
eng = Engine(0)
pks, sks = eng.batch_keygen(level, np.arange(32, dtype=np.uint8))
sk = sks[0]
rng = np.random.default_rng(1)
for n in (1000000, 100000):
    msgs = (rng.integers(0, 256, n * 32, dtype=np.uint8), np.arange(n + 1, dtype=np.uint64) * 32)
    out = pinned(eng, (n, LEVELS[level][4]))
    best = 1e9
    for rep in range(3):
        st = eng.sign_wait(eng.sign_submit(level, sk, msgs, out=out))[3]
        best = min(best, (st["t_last_exit_ns"] - st["t_first_start_ns"]) / 1e9)
    print(f"level {level} n={n}: {n / best / 1e6:.2f} M/s device (first claim -> last commit), attempts/sig {st['attempts']/n:.2f}")
eng.close()
