"""Small end-to-end pass used under compute-sanitizer (memcheck / racecheck / initcheck)."""
import os
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2211_12265_b200 import Engine
eng = Engine(0)
rng = np.random.default_rng(5)
for level, n in ((2, 300), (3, 150), (5, 130), (65, 120)):  # 65 = ML-DSA-65 (FIPS 204 mode)
    zetas = rng.integers(0, 256, (n, 32), dtype=np.uint8)
    msgs = [bytes(rng.integers(0, 256, int(rng.integers(0, 300)), dtype=np.uint8)) for _ in range(n)]
    pks, sks = eng.batch_keygen(level, zetas)
    sigs, att, failed, st = eng.batch_sign(level, sks, msgs, return_info=True)
    sigs2 = eng.batch_sign(level, sks[0], msgs, psi=256)
    assert eng.batch_verify(level, pks, msgs, sigs).all()
    assert eng.batch_verify(level, pks[0], msgs, sigs2).all()
    if os.environ.get("DLB_NO_KEYED"):
        continue
    kidx = rng.integers(0, 5, n).astype(np.uint32)  # mixed-key batch over a 5-key table
    sigs3 = eng.batch_sign(level, sks[:5], msgs, key_idx=kidx)
    assert eng.batch_verify(level, pks[:5], msgs, sigs3, key_idx=kidx).all()
    if level == 65:  # a context string exercises the prefix gather of the mu hash
        eng.set_mldsa_context(b"sanitizer context")
        s4 = eng.batch_sign(level, sks[0], msgs[:40])
        assert eng.batch_verify(level, pks[0], msgs[:40], s4).all()
        eng.set_mldsa_context(b"")
    # batches in flight (several tickets, waited out of order), the assignment log, injected bounds.
    # (memcheck validates a kernel's accesses against the allocations that existed when it was
    # launched; the arena sets of tickets 2..4 are therefore first sized by a pass whose kernels
    # have finished before the next submission allocates)
    import time
    warm = []
    for i in range(4):
        warm.append(eng.sign_submit(level, sks[0], msgs[i::4]))
        time.sleep(1.0 if os.environ.get("DLB_SLOW_WARM") else 0.05)
    for h in warm:
        eng.sign_wait(h)
    hs = [eng.sign_submit(level, sks[0], msgs[i::4]) for i in range(4)]
    for i in (2, 0, 3, 1):
        got = eng.sign_wait(hs[i])[0]
        assert np.array_equal(got, sigs2[i::4])
    eng.set_assignment_log(64 * n)
    eng.batch_sign(level, sks[0], msgs[:50], psi=64)
    recs, total = eng.get_assignment_log()
    eng.set_assignment_log(0)
    assert total == len(recs) and total >= 50
    mus = rng.integers(0, 256, (8, 64), dtype=np.uint8)
    acc, stage, _, _, _ = eng.dbg_sign_attempt_bounded(level, sks[0], mus, mus[::-1].copy(),
                                                        np.zeros(8, np.uint32), 1, 1000, 1000)
    assert not acc.any() and (stage == 0).all()
    print("level", level, "ok, mean attempts %.2f" % att.mean())
