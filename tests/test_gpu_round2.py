"""Round-2 boundary and scheduler tests on the device (-m gpu): the assignment hook and the
scheduler-equivalence criterion (tests/acceptance.cpp:186-244), injected norm bounds and reject
stages (tests/test_scheme.cpp:147-174), nonce-space exhaustion (scheduler.hpp:52,122-128),
batches in flight (tools/dilithium_cli.cpp:309-345), the cross-call key cache."""
import os

import numpy as np
import pytest

from tests.cpu_checkers import PARAMS, mt19937_64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    from paper_2211_12265_b200 import Engine
    e = Engine(0)
    yield e
    e.close()


def _cpu_sign_all(checker, ref, level, sk, flat, off):
    """Sequential signatures of every message: the compiled reference when it is there (all
    host threads; batch == sequential is its own criterion 5), else the oracle one by one."""
    n = len(off) - 1
    try:
        from tests.cpu_checkers import load_ref, ref_available
        if ref_available():
            r = load_ref()
            return r.batch_sign(level, sk, flat, off, workers=max(1, r.hw_threads()))[0]
    except Exception:
        pass
    return np.stack([np.frombuffer(checker.sign(level, sk.tobytes(), flat[int(off[i]):int(off[i + 1])].tobytes())[0],
                                   np.uint8) for i in range(n)])


def test_acceptance5_scheduler_equivalence_with_hook(eng, oracle):
    """acceptance.cpp:221-244: 100 random batches (phi <= 512, psi <= phi, 8 of 10 at level 2, one
    each at 3 and 5): bytes identical to sequential signing, and the assignment hook's records
    (here: the device's executed-attempt log) hold no (task, nonce) twice and every nonce below
    each task's accepted one."""
    rng = mt19937_64(55)
    for b in range(100):
        phi = 1 + int(rng()) % 512
        psi = 1 + int(rng()) % phi
        level = 2 if b % 10 < 8 else (3 if b % 10 == 8 else 5)
        L = PARAMS[level]["l"]
        pk, sk = oracle.keygen(level, rng.bytes(32))
        sk_a = np.frombuffer(sk, np.uint8)
        flat = np.frombuffer(rng.bytes(24 * phi), np.uint8)
        off = np.arange(phi + 1, dtype=np.uint64) * 24
        eng.set_assignment_log(64 * phi + 4096)
        sigs, att, failed, st = eng.batch_sign(level, sk_a, (flat, off), psi=psi, return_info=True)
        recs, total = eng.get_assignment_log()
        eng.set_assignment_log(0)
        assert not failed.any()
        assert total == len(recs) == st["attempts"], (total, len(recs), st["attempts"])
        pairs = recs[:, 1].astype(np.int64) * 65536 + recs[:, 3]
        assert len(np.unique(pairs)) == len(pairs), "a (task, nonce) was executed twice"
        assert np.array_equal(recs[:, 3], recs[:, 2] * L)  # kappa = attempt * l
        have = set(pairs.tolist())
        for t in range(phi):
            for a in range(int(att[t])):
                assert t * 65536 + a * L in have, "an attempt below the accepted one never ran"
        assert np.array_equal(sigs, _cpu_sign_all(oracle, None, level, sk_a, flat, off)), "batch != sequential"


@pytest.mark.parametrize("level", [2, 3, 5, 65])
def test_forced_reject_stages(eng, oracle, ref, level):
    """test_scheme.cpp:147-174 at scale: sign_attempt_bounded with the production bounds, with each
    bound corrupted to 1, and with bounds tightened just enough that all four stages occur --
    accepted flag, reject stage, c~, z and hints equal the CPU checker's."""
    P = PARAMS[level]
    n = 160
    rng = mt19937_64(6040 + level)
    pk, sk = oracle.keygen(level, rng.bytes(32))
    sk_a = np.frombuffer(sk, np.uint8)
    mus = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64)
    rps = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64)
    kappas = np.array([(int(rng()) % 50) * P["l"] for _ in range(n)], np.uint32)
    g1b, g2b, g2 = P["gamma1"] - P["beta"], P["gamma2"] - P["beta"], P["gamma2"]
    checker = oracle if level > 5 else ref  # the reference has no FIPS 204 sets
    seen = set()
    for zb, rb, vb in ((g1b, g2b, g2), (1, g2b, g2), (g1b, 1, g2), (g1b, g2b, 1),
                       (g1b, g2b, g2 // 3), (g1b - g1b // 40, g2b - g2b // 12, (g2 * 2) // 5)):
        acc, stage, ct, z, h = eng.dbg_sign_attempt_bounded(level, sk_a, mus, rps, kappas, zb, rb, vb)
        for i in range(n):
            rc, st, ect, ez, eh = checker.sign_attempt_bounded(level, sk, mus[i].tobytes(), rps[i].tobytes(),
                                                               int(kappas[i]), zb, rb, vb)
            assert acc[i] == rc, (i, zb, rb, vb)
            assert ct[i].tobytes() == ect
            if rc:
                assert stage[i] == 255 and np.array_equal(z[i], ez) and np.array_equal(h[i], eh)
            else:
                assert stage[i] == st, (i, stage[i], st, zb, rb, vb)
                seen.add(int(st))
    assert seen == {0, 1, 2} or seen == {0, 1, 2, 3}, seen
    with pytest.raises(Exception):  # chknorm's domain (rounding.hpp:65)
        eng.dbg_sign_attempt_bounded(level, sk_a, mus[:1], rps[:1], kappas[:1], (8380417 - 1) // 8 + 1, rb, vb)


@pytest.mark.parametrize("level", [2, 5])
def test_nonce_space_exhaustion_reports_failed_tasks(eng, oracle, level):
    """scheduler.hpp:52,122-128 / batch.hpp:128-131: a task whose nonce space runs out is reported
    failed, gets an all-zero signature, and the others still complete.  The real limit is
    unreachable, so the stage-test knob shrinks it to three attempts."""
    n = 600
    rng = mt19937_64(1220 + level)
    pk, sk = oracle.keygen(level, rng.bytes(32))
    sk_a = np.frombuffer(sk, np.uint8)
    flat = np.frombuffer(rng.bytes(20 * n), np.uint8)
    off = np.arange(n + 1, dtype=np.uint64) * 20
    expect = [oracle.sign(level, sk, flat[20 * i:20 * i + 20].tobytes()) for i in range(n)]
    eng.dbg_set_max_attempt(2)
    try:
        for psi, spec in ((0, True), (64, False), (4096, True)):
            sigs, att, failed, st = eng.batch_sign(level, sk_a, (flat, off), psi=psi, speculate=spec,
                                                   return_info=True)
            want_failed = np.array([a > 3 for _, a in expect], np.uint8)
            assert np.array_equal(failed, want_failed) and 0 < want_failed.sum() < n
            assert st["failed_tasks"] == int(want_failed.sum())
            for i in range(n):
                if want_failed[i]:
                    assert not sigs[i].any() and att[i] == 0
                else:
                    assert sigs[i].tobytes() == expect[i][0] and att[i] == expect[i][1]
    finally:
        eng.dbg_set_max_attempt(0)
    sigs = eng.batch_sign(level, sk_a, (flat, off))
    assert all(sigs[i].tobytes() == expect[i][0] for i in range(n))


def test_batches_in_flight_mixed_levels_and_keys(eng, oracle):
    """dlb_sign_submit / dlb_sign_wait: sixteen batches of different sizes, levels, keys and key
    modes (plus sixteen single-task batches, filling the ring of 32) in flight at once, waited out of order -- every byte as if each had run alone."""
    rng = mt19937_64(31415)
    shapes = [(2, 3000, "shared"), (3, 700, "shared"), (2, 1, "shared"), (5, 900, "per_task"),
              (2, 5000, "table"), (2, 64, "shared"), (3, 2000, "table"), (44, 800, "shared"),
              (2, 12000, "shared"), (5, 300, "shared"), (2, 2500, "per_task"), (87, 100, "shared"),
              (2, 9000, "shared"), (3, 33, "per_task"), (2, 777, "shared"), (65, 400, "table")]
    jobs = []
    for level, n, mode in shapes:
        nk = {"shared": 1, "per_task": n, "table": 5}[mode]
        zetas = np.frombuffer(rng.bytes(32 * nk), np.uint8).reshape(nk, 32)
        pks, sks = eng.batch_keygen(level, zetas)
        lens = [int(rng()) % 70 for _ in range(n)]
        off = np.zeros(n + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        flat = np.frombuffer(rng.bytes(int(off[-1]) + 1), np.uint8)
        kidx = np.array([int(rng()) % nk for _ in range(n)], np.uint32) if mode == "table" else None
        jobs.append((level, n, mode, sks, flat, off, kidx))
    alone = []
    for level, n, mode, sks, flat, off, kidx in jobs:
        alone.append(eng.batch_sign(level, sks[0] if mode == "shared" else sks, (flat, off), key_idx=kidx,
                                    return_info=True))
    handles = [eng.sign_submit(level, sks[0] if mode == "shared" else sks, (flat, off), key_idx=kidx)
               for level, n, mode, sks, flat, off, kidx in jobs]
    extra = [eng.sign_submit(2, jobs[2][3][0], (jobs[2][4], jobs[2][5])) for _ in range(16)]
    with pytest.raises(Exception):  # the ring holds 32 consecutive tickets: the 33rd submission is refused
        eng.sign_submit(2, jobs[0][3][0], (jobs[0][4], jobs[0][5]))
    for h in extra[::-1]:
        assert np.array_equal(eng.sign_wait(h)[0], alone[2][0])
    order = [7, 0, 15, 3, 8, 1, 2, 12, 4, 5, 6, 9, 10, 11, 13, 14]
    for j in order:
        sigs, att, failed, st = eng.sign_wait(handles[j])
        assert not failed.any() and np.array_equal(sigs, alone[j][0]) and np.array_equal(att, alone[j][1])
        assert st["accepted_attempt_sum"] == int(att.sum())
    for j in (0, 3, 4, 7, 15):  # and those bytes are the CPU oracle's
        level, n, mode, sks, flat, off, kidx = jobs[j]
        for i in range(0, n, max(1, n // 9)):
            k = 0 if mode == "shared" else (int(kidx[i]) if mode == "table" else i)
            assert alone[j][0][i].tobytes() == oracle.sign(level, sks[k].tobytes(),
                                                           flat[int(off[i]):int(off[i + 1])].tobytes())[0]
    # the engine is usable afterwards, synchronously and with new tickets
    h = eng.sign_submit(2, jobs[0][3][0], (jobs[0][4], jobs[0][5]))
    assert np.array_equal(eng.sign_wait(h)[0], alone[0][0])


def test_key_cache_across_calls(oracle, monkeypatch):
    """SignPrecomp kept across calls (scheme.hpp:106-125): a two-entry cache is hit, missed and
    evicted; outputs never change; a malformed shared key is refused before any work."""
    from paper_2211_12265_b200 import Engine
    monkeypatch.setenv("DLB_KEY_CACHE", "2")
    e = Engine(0)
    try:
        rng = mt19937_64(2718)
        level = 3
        keys = [oracle.keygen(level, rng.bytes(32)) for _ in range(4)]
        msgs = [rng.bytes(40) for _ in range(50)]
        want = {k: [oracle.sign(level, keys[k][1], m)[0] for m in msgs[:6]] for k in range(4)}
        for k in (0, 1, 0, 2, 3, 1, 0, 0, 3):
            sigs = e.batch_sign(level, np.frombuffer(keys[k][1], np.uint8), msgs)
            assert [sigs[i].tobytes() for i in range(6)] == want[k]
        bad = bytearray(keys[0][1])
        bad[64 + 32] = 0xFF  # an eta field out of range (packing.hpp:79-86)
        with pytest.raises(ValueError):
            e.batch_sign(level, np.frombuffer(bytes(bad), np.uint8), msgs)
        with pytest.raises(ValueError):
            e.sign_submit(level, np.frombuffer(bytes(bad), np.uint8), msgs)
    finally:
        e.close()
    monkeypatch.setenv("DLB_KEY_CACHE", "0")  # cache off: the per-call path
    e = Engine(0)
    try:
        sigs = e.batch_sign(level, np.frombuffer(keys[2][1], np.uint8), msgs)
        assert [sigs[i].tobytes() for i in range(6)] == want[2]
    finally:
        e.close()


def test_in_flight_stress_random_pipeline(eng):
    """A long random pipeline: 240 batches of random size (1 .. 30,000), level and key -- 40 shared
    keys per level, more than the 32-entry key cache holds, plus per-task-key batches -- submitted
    with a randomly varying number of tickets in flight and waited in random order.  Every
    signature and attempt count must equal what the same batch gives when it runs alone."""
    rs = np.random.default_rng(977)
    levels = (2, 3, 5, 44)
    keys = {lv: eng.batch_keygen(lv, rs.integers(0, 256, (40, 32), dtype=np.uint8)) for lv in levels}
    pool = {}

    def make(lv):
        n = int(rs.choice([1, 7, 100, 900, 4000, 12000, 30000], p=[.1, .1, .2, .25, .2, .1, .05]))
        per_task = n <= 40 and rs.random() < 0.3
        k = None if per_task else int(rs.integers(0, 40))
        lens = rs.integers(0, 90, n)
        off = np.zeros(n + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        flat = rs.integers(0, 256, int(off[-1]) + 1, dtype=np.uint8)
        sk = keys[lv][1][:n] if per_task else keys[lv][1][k]
        return lv, sk, flat, off

    inflight, checked = [], 0
    iters = int(os.environ.get("DLB_STRESS_ITERS", "240"))  # a longer soak: DLB_STRESS_ITERS=3000
    for it in range(iters):
        lv = int(rs.choice(levels, p=[.55, .2, .15, .1]))
        job = make(lv)
        want = eng.batch_sign(job[0], job[1], (job[2], job[3]), return_info=True) if it % 3 == 0 else None
        depth = int(rs.integers(1, 25))
        newest = max([h["ticket"] for h, _, _ in inflight], default=0) + (2 if want is not None else 1)
        # (the ring holds 32 consecutive tickets: whatever was submitted 32 tickets ago must have
        # been waited for; the synchronous call above consumed a ticket as well)
        while len(inflight) >= depth or (inflight and newest - min(h["ticket"] for h, _, _ in inflight) >= 31):
            old = min(range(len(inflight)), key=lambda i: inflight[i][0]["ticket"])
            j = old if newest - inflight[old][0]["ticket"] >= 31 else int(rs.integers(0, len(inflight)))
            h, jb, w = inflight.pop(j)
            sigs, att, failed, st = eng.sign_wait(h)
            assert not failed.any() and st["accepted_attempt_sum"] == int(att.sum())
            if w is not None:
                assert np.array_equal(sigs, w[0]) and np.array_equal(att, w[1])
                checked += 1
            else:  # every signature at least verifies under its key
                pk = keys[jb[0]][0]
                kk = pk[:len(att)] if jb[1].ndim == 2 else pk[[i for i in range(40) if np.array_equal(keys[jb[0]][1][i], jb[1])][0]]
                assert eng.batch_verify(jb[0], kk, (jb[2], jb[3]), sigs).all()
        inflight.append((eng.sign_submit(job[0], job[1], (job[2], job[3])), job, want))
    for h, jb, w in inflight:
        sigs, att, failed, _ = eng.sign_wait(h)
        assert not failed.any()
        if w is not None:
            assert np.array_equal(sigs, w[0]) and np.array_equal(att, w[1])
            checked += 1
    assert checked >= 60


def test_steady_flow_reuses_ring_slots_under_resident_ctas(eng, oracle):
    """A steady flow of equal batches, 24 in flight, over four turns of the 32-slot ring: the
    scheduler CTAs stay resident across batches (their views of a ring slot are re-tagged when the
    slot gets its next ticket; claims are compare-and-swaps against the slot's ticket), so every
    batch must still give the bytes of a synchronous call, a stage test (an exclusive batch of
    another kernel) in the middle of the flow included."""
    rs = np.random.default_rng(4242)
    level, n, depth, batches = 2, 20000, 24, 130
    pks, sks = eng.batch_keygen(level, rs.integers(0, 256, (1, 32), dtype=np.uint8))
    flat = rs.integers(0, 256, n * 32, dtype=np.uint8)
    off = np.arange(n + 1, dtype=np.uint64) * 32
    want, want_att, _, _ = eng.batch_sign(level, sks[0], (flat, off), return_info=True)
    for i in range(0, n, n // 5):
        assert want[i].tobytes() == oracle.sign(level, sks[0].tobytes(), flat[32 * i:32 * i + 32].tobytes())[0]
    mus = rs.integers(0, 256, (8, 64), dtype=np.uint8)
    inflight = []
    for b in range(batches):
        if len(inflight) >= depth:
            sigs, att, failed, st = eng.sign_wait(inflight.pop(0))
            assert not failed.any() and np.array_equal(sigs, want) and np.array_equal(att, want_att)
            assert st["accepted_attempt_sum"] == int(want_att.sum()) and st["attempts"] >= st["accepted_attempt_sum"]
        if b == 70:  # one round of the bounds-injected kernel while 23 batches are in flight
            acc, stage, _, _, _ = eng.dbg_sign_attempt_bounded(level, sks[0], mus, mus[::-1].copy(),
                                                                np.zeros(8, np.uint32), 1, 1000, 1000)
            assert not acc.any() and (stage == 0).all()
        inflight.append(eng.sign_submit(level, sks[0], (flat, off)))
    for h in inflight:
        sigs, att, failed, st = eng.sign_wait(h)
        assert not failed.any() and np.array_equal(sigs, want) and np.array_equal(att, want_att)


def test_staged_result_copies_option(oracle, monkeypatch):
    """DLB_ZERO_COPY_MAX=0: signatures for a pinned caller buffer go through device memory and are
    copied at wait time (copies of batches that completed meanwhile are queued behind the waited
    one); bytes are those of the default in-place path and of the oracle.  Straight through the
    C ABI with every result buffer pinned."""
    import ctypes as C
    from paper_2211_12265_b200 import Engine
    from paper_2211_12265_b200.engine import LEVELS, SignStats
    level, n, batches = 3, 700, 6
    sgb = LEVELS[level][4]
    rs = np.random.default_rng(99)
    flats = [rs.integers(0, 256, n * 24, dtype=np.uint8) for _ in range(batches)]
    off = np.arange(n + 1, dtype=np.uint64) * 24
    vp = C.c_void_p
    got = {}
    for knob in ("0", None):
        if knob is None:
            monkeypatch.delenv("DLB_ZERO_COPY_MAX", raising=False)
        else:
            monkeypatch.setenv("DLB_ZERO_COPY_MAX", knob)
        e = Engine(0)
        try:
            pks, sks = e.batch_keygen(level, np.arange(32, dtype=np.uint8))
            sk = np.ascontiguousarray(sks[0])

            def pinned(nbytes, dtype):
                p = e.lib.dlb_host_alloc(nbytes)
                assert p
                return p, np.frombuffer((C.c_uint8 * nbytes).from_address(p), dtype)

            bufs = [(pinned(n * sgb, np.uint8), pinned(n * 4, np.uint32), pinned(n, np.uint8)) for _ in range(batches)]
            tickets = []
            for b in range(batches):
                (ps, _), (pa, _), (pf, _) = bufs[b]
                t = C.c_uint64(0)
                assert e.lib.dlb_sign_submit(e.ctx, level, 0, vp(sk.ctypes.data), 0, n, None, vp(flats[b].ctypes.data),
                                             vp(off.ctypes.data), None, 0, 1, vp(ps), vp(pa), vp(pf), C.byref(t)) == 0
                tickets.append(t.value)
            for b in (3, 0, 5, 1, 2, 4):
                st = SignStats()
                assert e.lib.dlb_sign_wait(e.ctx, tickets[b], C.byref(st)) == 0
                assert not bufs[b][2][1].any() and st.accepted_attempt_sum == int(bufs[b][1][1].sum())
            got[knob] = [bufs[b][0][1].reshape(n, sgb).copy() for b in range(batches)]
            for trio in bufs:
                for p, _ in trio:
                    e.lib.dlb_host_free(p)
        finally:
            e.close()
    for b in range(batches):
        assert np.array_equal(got["0"][b], got[None][b])
        assert got["0"][b][7].tobytes() == oracle.sign(level, sks[0].tobytes(), flats[b][7 * 24:8 * 24].tobytes())[0]
