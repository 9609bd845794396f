"""Claim / commit timeline of batches in flight (device %globaltimer from dlb_sign_stats)."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
from paper_2211_12265_b200 import Engine
from scripts.async_probe import pinned
from paper_2211_12265_b200.engine import LEVELS

level = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
batches = int(sys.argv[3]) if len(sys.argv) > 3 else 4
eng = Engine(0)
pks, sks = eng.batch_keygen(level, np.arange(32, dtype=np.uint8))
sk = sks[0]
rng = np.random.default_rng(1)
msgs = [(rng.integers(0, 256, n * 32, dtype=np.uint8), np.arange(n + 1, dtype=np.uint64) * 32) for _ in range(batches)]
outs = [pinned(eng, (n, LEVELS[level][4])) for _ in range(batches)]
for rep in range(6):
    t0 = time.perf_counter()
    hs = [eng.sign_submit(level, sk, msgs[b], out=outs[b]) for b in range(batches)]
    t1 = time.perf_counter()
    sts = [eng.sign_wait(h)[3] for h in hs]
    t2 = time.perf_counter()
base = min(s["t_first_start_ns"] for s in sts)
print(f"submit all {1e3*(t1-t0):.2f} ms, total {1e3*(t2-t0):.2f} ms -> {n*batches/(t2-t0)/1e6:.2f} M/s")
for b, s in enumerate(sts):
    print(b, "first claim %.3f last claim %.3f first commit %.3f last commit %.3f ms | attempts/sig %.2f spec %.3f rounds %d idle %d" % (
        (s["t_first_start_ns"] - base) / 1e6, (s["t_last_start_ns"] - base) / 1e6,
        (s["t_first_exit_ns"] - base) / 1e6, (s["t_last_exit_ns"] - base) / 1e6,
        s["attempts"] / n, s["speculative"] / max(1, s["attempts"]), s["rounds"], s["idle_slot_rounds"]))
eng.close()
