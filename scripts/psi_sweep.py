"""Psi (resident attempt slots) sweep for batch_sign -- the paper's sensitivity study
 on B200; development aid."""
import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2211_12265_b200 import Engine, LEVELS
from paper_2211_12265_b200.engine import SignStats
eng = Engine(0); lib, ctx = eng.lib, eng.ctx
level = int(sys.argv[1]) if len(sys.argv) > 1 else 2
k, l, pkb, skb, sgb = LEVELS[level]
rng = np.random.default_rng(1)
pk1, sk1 = eng.batch_keygen(level, rng.integers(0, 256, 32, dtype=np.uint8))
dev = torch.device("cuda:0")
P = lambda t: C.c_void_p(t.data_ptr())
for n in [int(x) for x in sys.argv[2].split(",")]:
    msgs = torch.from_numpy(rng.integers(0, 256, (n, 32), dtype=np.uint8)).to(dev)
    off = (torch.arange(n + 1, dtype=torch.int64) * 32).to(dev)
    sigs = torch.empty((n, sgb), dtype=torch.uint8, device=dev)
    att = torch.empty(n, dtype=torch.int32, device=dev); fl = torch.empty(n, dtype=torch.uint8, device=dev)
    sk_d = torch.from_numpy(sk1[0].copy()).to(dev)
    for psi in [int(x) for x in sys.argv[3].split(",")]:
        st = SignStats(); ms = []
        for _ in range(6):
            assert lib.dlb_sign_batch_dev(ctx, level, n, P(sk_d), 0, P(msgs), P(off), None, psi, 1, P(sigs), P(att), P(fl), C.byref(st)) == 0
            ms.append(eng.last_kernel_ms)
        m = sorted(ms[1:])[2]
        print("L%d n=%d psi=%6d: %.3f ms  %.2fM/s executed/op=%.2f" % (level, n, psi, m, n / m / 1e3, st.attempts / n))
