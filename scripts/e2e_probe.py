"""Host-buffer (e2e) keygen / verify throughput probe: pinned buffers, copies timed."""
import sys, time, ctypes as C
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2211_12265_b200 import Engine, LEVELS
level = 2
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
eng = Engine(0); lib, ctx = eng.lib, eng.ctx
k, l, pkb, skb, sgb = LEVELS[level]
rng = np.random.default_rng(3)
pk1, sk1 = eng.batch_keygen(level, rng.integers(0, 256, 32, dtype=np.uint8))
msgs = rng.integers(0, 256, (n, 32), dtype=np.uint8)
off = np.arange(n + 1, dtype=np.uint64) * 32
sigs = eng.batch_sign(level, sk1[0], (msgs.reshape(-1), off))
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
h_m, h_off, h_sig = pin(msgs), pin(off.astype(np.int64)), pin(sigs)
h_pk = pin(np.repeat(pk1, n, axis=0)); h_fl = pin(np.zeros(n, np.uint8))
h_z = pin(msgs); h_pks = pin(np.zeros((n, pkb), np.uint8)); h_sks = pin(np.zeros((n, skb), np.uint8))
u8 = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_uint8))
u64 = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_uint64))
def run(fn, reps=7):
    fn(); fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); assert fn() == 0; ts.append(time.perf_counter() - t0)
    return float(np.median(ts))
tv = run(lambda: lib.dlb_verify_batch(ctx, level, n, u8(h_pk), pkb, u8(h_m), u64(h_off), u8(h_sig), u8(h_fl)))
assert bool(h_fl.all())
tk = run(lambda: lib.dlb_keygen_batch(ctx, level, n, u8(h_z), u8(h_pks), u8(h_sks)))
print("n=%d e2e verify (pk per task) %.2f M/s  keygen %.2f M/s" % (n, n / tv / 1e6, n / tk / 1e6))
