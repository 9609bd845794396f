"""Where the end-to-end sign call spends its time: wall clock vs kernel-only events, pinned
(zero-copy commit) vs device-resident output."""
import sys, time, ctypes as C
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2211_12265_b200 import Engine, LEVELS
level, n = 2, int(sys.argv[1]) if len(sys.argv) > 1 else 100000
eng = Engine(0); lib, ctx = eng.lib, eng.ctx
k, l, pkb, skb, sgb = LEVELS[level]
rng = np.random.default_rng(3)
pk1, sk1 = eng.batch_keygen(level, rng.integers(0, 256, 32, dtype=np.uint8))
msgs = rng.integers(0, 256, (n, 32), dtype=np.uint8)
off = np.arange(n + 1, dtype=np.uint64) * 32
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
h_m, h_off, h_sk = pin(msgs), pin(off.astype(np.int64)), pin(sk1[0])
h_sig = torch.zeros((n, sgb), dtype=torch.uint8).pin_memory()
dev = torch.device("cuda:0")
d_m, d_off, d_sk = h_m.to(dev), h_off.to(dev), h_sk.to(dev)
d_sig = torch.zeros((n, sgb), dtype=torch.uint8, device=dev)
u8 = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_uint8))
u64 = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_uint64))
P = lambda t: C.c_void_p(t.data_ptr())
def host(): return lib.dlb_sign_batch(ctx, level, n, u8(h_sk), 0, u8(h_m), u64(h_off), None, 0, 1, u8(h_sig), None, None, None)
def devc(): return lib.dlb_sign_batch_dev(ctx, level, n, P(d_sk), 0, P(d_m), P(d_off), None, 0, 1, P(d_sig), None, None, None)
def devhost(): return lib.dlb_sign_batch_dev(ctx, level, n, P(d_sk), 0, P(d_m), P(d_off), None, 0, 1, P(h_sig), None, None, None)
for name, fn in (("device-resident", devc), ("device inputs, pinned-host output", devhost), ("host API (pinned)", host)):
    for _ in range(3): assert fn() == 0
    wall, kern, main = [], [], []
    for _ in range(9):
        torch.cuda.synchronize(); t0 = time.perf_counter(); assert fn() == 0; wall.append((time.perf_counter() - t0) * 1e3)
        kern.append(eng.last_kernel_ms); main.append(eng.last_main_kernel_ms)
    print("%-36s wall %.3f ms  call events %.3f ms  scheduler kernel %.3f ms" % (name, np.median(wall), np.median(kern), np.median(main)))
