"""Timeline of the scheduler kernel under two engine contexts (development probe)."""
import sys, faulthandler, threading, ctypes as C
faulthandler.enable(); faulthandler.dump_traceback_later(90, exit=True)
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2211_12265_b200 import Engine
from paper_2211_12265_b200.engine import SignStats
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = 3
engs = [Engine(0) for _ in range(lanes)]
pk, sk = engs[0].batch_keygen(2, np.arange(32, dtype=np.uint8))
dev = torch.device("cuda:0")
msgs = torch.from_numpy(np.random.default_rng(1).integers(0, 256, (n, 32), dtype=np.uint8)).to(dev)
off = (torch.arange(n + 1, dtype=torch.int64) * 32).to(dev)
sk_d = torch.from_numpy(sk[0].copy()).to(dev)
sigs = [torch.empty((n, 2420), dtype=torch.uint8, device=dev) for _ in range(lanes)]
P = lambda t: C.c_void_p(t.data_ptr())
log = []
def worker(l):
    e = engs[l]
    for r in range(reps):
        st = SignStats()
        rc = e.lib.dlb_sign_batch_dev(e.ctx, 2, n, P(sk_d), 0, P(msgs), P(off), None, 0, 1, P(sigs[l]), None, None, C.byref(st))
        assert rc == 0
        log.append((l, r, st.t_first_start_ns, st.t_last_start_ns, st.t_first_exit_ns, st.t_last_exit_ns, 0))
for w in range(2):
    log.clear()
    ts = [threading.Thread(target=worker, args=(l,)) for l in range(lanes)]
    [t.start() for t in ts]; [t.join() for t in ts]
t0 = min(x[2] for x in log)
for l, r, a, b, c, d, rq in sorted(log, key=lambda x: x[2]):
    print("lane %d rep %d: first start %8.3f ms  last start %8.3f  first exit %8.3f  last exit %8.3f  requeued %d" % (
        l, r, (a - t0) / 1e6, (b - t0) / 1e6, (c - t0) / 1e6, (d - t0) / 1e6, rq))
