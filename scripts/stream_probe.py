"""Development probe for bench.streamed_sign (two engine contexts on one GPU)."""
import sys, faulthandler, time
faulthandler.enable()
faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, ".")
import numpy as np, torch
import bench
from paper_2211_12265_b200 import Engine
n_total = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
lanes = int(sys.argv[3]) if len(sys.argv) > 3 else 2
d = bench.Dist()
eng = Engine(0)
pk, sk = eng.batch_keygen(2, np.arange(32, dtype=np.uint8))
print("keygen ok", flush=True)
msgs = np.random.default_rng(5150).integers(0, 256, (n_total, 32), dtype=np.uint8)
off = np.arange(n_total + 1, dtype=np.uint64) * 32
print("inputs ok", flush=True)
for L in ([1, lanes] if lanes > 1 else [1]):
    v, sample = bench.streamed_sign(torch, d, 0, 2, sk[0], msgs, off, chunk, L, 1)
    print("lanes", L, "ops/s", v, flush=True)
