"""Quick throughput probe (device-resident + host API) -- development aid, not the bench."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2211_12265_b200 import Engine, LEVELS
import ctypes as C

eng = Engine(0)
import os
if not os.environ.get("DLB_NO_PEAK"):
    print("int32 peaks (Tlane-op/s):", eng.measure_int32_peak())
lib, ctx = eng.lib, eng.ctx
levels = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2"])]
sizes = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["10000", "100000"])]
only = sys.argv[3].split(",") if len(sys.argv) > 3 else ["keygen", "sign", "verify"]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
for level in levels:
    k, l, pkb, skb, sgb = LEVELS[level]
    rng = np.random.default_rng(1)
    pk1, sk1 = eng.batch_keygen(level, rng.integers(0, 256, 32, dtype=np.uint8))
    for n in sizes:
        dev = torch.device("cuda:0")
        zetas = torch.from_numpy(rng.integers(0, 256, (n, 32), dtype=np.uint8)).to(dev)
        msgs = torch.from_numpy(rng.integers(0, 256, (n, 32), dtype=np.uint8)).to(dev)
        off = (torch.arange(n + 1, dtype=torch.int64) * 32).to(dev)
        pks = torch.empty((n, pkb), dtype=torch.uint8, device=dev)
        sks = torch.empty((n, skb), dtype=torch.uint8, device=dev)
        sigs = torch.empty((n, sgb), dtype=torch.uint8, device=dev)
        att = torch.empty(n, dtype=torch.int32, device=dev)
        fl = torch.empty(n, dtype=torch.uint8, device=dev)
        sk_d = torch.from_numpy(sk1[0].copy()).to(dev)
        pk_d = torch.from_numpy(pk1[0].copy()).to(dev)
        torch.cuda.synchronize()
        P = lambda t: C.c_void_p(t.data_ptr())
        from paper_2211_12265_b200.engine import SignStats
        st = SignStats()
        def kg(): return lib.dlb_keygen_batch_dev(ctx, level, n, P(zetas), P(pks), P(sks))
        def sg(): return lib.dlb_sign_batch_dev(ctx, level, n, P(sk_d), 0, P(msgs), P(off), None, 0, 1, P(sigs), P(att), P(fl), C.byref(st))
        def vf(): return lib.dlb_verify_batch_dev(ctx, level, n, P(pk_d), 0, P(msgs), P(off), P(sigs), P(fl))
        if "sign" not in only and "verify" in only:
            assert sg() == 0
        for name, fn in (("keygen", kg), ("sign", sg), ("verify", vf)):
            if name not in only: continue
            if reps == 0:
                assert fn() == 0
                print("L%d n=%d %s single call %.3f ms" % (level, n, name, eng.last_kernel_ms))
                continue
            for _ in range(min(2, reps)): assert fn() == 0
            ms = []
            for _ in range(reps):
                assert fn() == 0
                ms.append(eng.last_kernel_ms)
            best, med = min(ms), sorted(ms)[len(ms) // 2]
            extra = ""
            if name == "sign":
                extra = " attempts/op=%.2f executed/op=%.2f rounds=%d" % (st.accepted_attempt_sum / n, st.attempts / n, st.rounds)
            if name == "verify":
                extra = " all_ok=%s" % bool(fl.all().item())
            print("L%d n=%d %-6s med %.3f ms  -> %.0f ops/s (best %.0f)%s" % (level, n, name, med, n / med * 1e3, n / best * 1e3, extra))
