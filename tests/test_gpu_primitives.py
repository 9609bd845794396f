"""Device parity of the building blocks, through the C ABI's stage-level entry points,
against the CPU oracle (and the compiled reference where it travelled).  -m gpu."""
import hashlib

import numpy as np
import pytest

from tests.cpu_checkers import PARAMS, Q, mt19937_64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    from paper_2211_12265_b200 import Engine
    e = Engine(0)
    yield e
    e.close()


def test_keccak_permutation(eng, oracle, kat):
    rng = np.random.default_rng(1)
    states = rng.integers(0, 2**63, (300, 25), dtype=np.uint64) * 2 + rng.integers(0, 2, (300, 25), dtype=np.uint64)
    states[0] = 0
    states[1] = np.array(kat["kKeccakRandIn"], dtype=np.uint64)
    out = eng.dbg_keccak_f1600(states)
    assert [int(v) for v in out[0]] == kat["kKeccakZeroState"]
    assert [int(v) for v in out[1]] == kat["kKeccakRandOut"]
    for i in range(2, 300):
        assert np.array_equal(out[i], oracle.keccak_f1600(states[i]))


def test_shake256_lengths(eng, kat):
    rng = mt19937_64(2)
    lens = [0, 1, 7, 8, 9, 31, 32, 33, 63, 64, 100, 135, 136, 137, 200, 271, 272, 273, 407, 408, 1312, 2592, 5000]
    msgs = [rng.bytes(n) for n in lens] + [b"\xa3" * 200]
    out = eng.dbg_shake256(msgs)
    for m, o in zip(msgs, out):
        assert o.tobytes() == hashlib.shake_256(m).digest(64), len(m)
    assert out[-1].tobytes().hex() == kat["kShake256Msg1600"]
    assert out[0].tobytes().hex() == kat["kShake256Empty"]


@pytest.mark.parametrize("level", [2, 3, 5])
def test_expand_a(eng, oracle, kat, level):
    P = PARAMS[level]
    rng = mt19937_64(30 + level)
    n = 11
    rhos = np.frombuffer(rng.bytes(32 * n), np.uint8).reshape(n, 32).copy()
    rhos[0] = 0
    out = eng.dbg_expand_a(level, rhos)
    assert out[0, 0, 0].tolist() == kat["kExpandA_r0_00"]
    assert out[0, 1, 2].tolist() == kat["kExpandA_r0_12"]
    for t in range(n):
        for i in range(P["k"]):
            for j in range(P["l"]):
                assert np.array_equal(out[t, i, j], oracle.expand_a(rhos[t].tobytes(), i, j)), (t, i, j)


@pytest.mark.parametrize("level", [2, 3, 5])
def test_expand_s(eng, oracle, kat, level):
    P = PARAMS[level]
    rng = mt19937_64(40 + level)
    n = 13
    rps = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64).copy()
    rps[0] = np.arange(64, dtype=np.uint8)
    out = eng.dbg_expand_s(level, rps)
    if P["eta"] == 2:
        assert out[0, 0].tolist() == kat["kExpandS_eta2_n0"]
        assert out[0, 7].tolist() == kat["kExpandS_eta2_n7"]
    else:
        assert out[0, 0].tolist() == kat["kExpandS_eta4_n0"]
    for t in range(n):
        for r in range(P["k"] + P["l"]):
            assert np.array_equal(out[t, r], oracle.expand_s(rps[t].tobytes(), r, P["eta"])), (t, r)


@pytest.mark.parametrize("level", [2, 3, 5])
def test_expand_mask(eng, oracle, kat, level):
    P = PARAMS[level]
    rng = mt19937_64(50 + level)
    n = 37
    rps = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64).copy()
    rps[0] = np.arange(64, dtype=np.uint8)
    kappas = np.array([0, 65535, 65533] + [int(rng()) % 60000 for _ in range(n - 3)], np.uint32)
    out = eng.dbg_expand_mask(level, rps, kappas)
    if level == 2:
        assert out[0, 0].tolist() == kat["kExpandMask_g17_n0"]
        assert out[0, 3].tolist() == kat["kExpandMask_g17_n3"]
    else:
        assert out[0, 0].tolist() == kat["kExpandMask_g19_n0"]
    for t in range(n):
        for j in range(P["l"]):
            exp = oracle.expand_mask(rps[t].tobytes(), (int(kappas[t]) + j) & 0xFFFF, P["gamma1"], P["z_bits"])
            assert np.array_equal(out[t, j], exp), (t, j)


@pytest.mark.parametrize("level", [2, 3, 5])
def test_sample_in_ball(eng, oracle, kat, level):
    P = PARAMS[level]
    rng = mt19937_64(60 + level)
    n = 200
    cts = np.frombuffer(rng.bytes(32 * n), np.uint8).reshape(n, 32).copy()
    cts[0] = np.arange(32, dtype=np.uint8)
    out = eng.dbg_sample_in_ball(level, cts)
    assert out[0].tolist() == kat["kBall_tau%d" % P["tau"]]
    for t in range(n):
        assert np.array_equal(out[t], oracle.sample_in_ball(cts[t].tobytes(), P["tau"])), t


def test_ntt_values(eng, oracle):
    rng = np.random.default_rng(7)
    a = rng.integers(0, Q, (64, 256), dtype=np.int32)
    a[0] = 0
    a[1] = Q - 1
    a[2] = np.arange(256)
    f = eng.dbg_ntt(a)
    for i in range(len(a)):
        assert np.array_equal(f[i], oracle.ntt(a[i])), i
    g = eng.dbg_ntt(f, inverse=True)
    assert np.array_equal(g, a)
    b = eng.dbg_ntt(a, inverse=True)
    for i in range(len(a)):
        assert np.array_equal(b[i], oracle.intt(a[i])), i


def test_inverse_ntt_lazy_bound_worst_case(eng, oracle):
    """The inverse transform reduces nothing between levels: sums double eight times, so inputs
    in (-q, q) reach 2^8 * q < 2^31 on the all-sums path (ntt.hpp:92-110 relies on the same
    bound).  Feed the representatives that maximise every partial sum -- all +(q-1), all
    -(q-1), sign patterns of each butterfly stride, random signed -- and compare values."""
    rng = np.random.default_rng(11)
    rows = [np.full(256, Q - 1), np.full(256, -(Q - 1))]
    idx = np.arange(256)
    for stride in (1, 2, 4, 8, 16, 32, 64, 128):
        sign = np.where((idx // stride) % 2 == 0, 1, -1)
        rows += [sign * (Q - 1), -sign * (Q - 1)]
    rows += [rng.integers(-(Q - 1), Q, 256) for _ in range(40)]
    rows += [rng.choice([-(Q - 1), Q - 1], 256) for _ in range(40)]
    a = np.array(rows, dtype=np.int32)
    got = eng.dbg_ntt(a, inverse=2)
    for i in range(len(a)):
        assert np.array_equal(got[i], oracle.intt((a[i].astype(np.int64) % Q).astype(np.int32))), i
    # forward transform of the largest inputs the kernels feed it: t1 * 2^13 (up to 1023 << 13)
    big = np.array([np.full(256, 1023 << 13), rng.integers(0, 1024, 256) << 13], dtype=np.int32)
    f = eng.dbg_ntt(big)
    for i in range(len(big)):
        assert np.array_equal(f[i], oracle.ntt((big[i].astype(np.int64) % Q).astype(np.int32))), i


@pytest.mark.parametrize("divisor", [88, 32])
def test_rounding_exhaustive(eng, oracle, divisor):
    """Power2Round, Decompose and UseHint on the device for EVERY r in [0, q)
    (tests/test_rounding.cpp:17-49,93-105; acceptance.cpp:109-145), against the definitions
    written out in numpy, themselves spot-checked against the oracle's functions."""
    q = 8380417
    gamma2 = (q - 1) // divisor
    alpha = 2 * gamma2
    m = (q - 1) // alpha
    r = np.arange(q, dtype=np.int64)
    # definitions (SPEC / FIPS 204 Alg. 35-40): centred remainders
    lo13 = ((r + 4095) % 8192) - 4095                      # r mod+- 2^13 in (-2^12, 2^12]
    p2_hi, p2_lo = (r - lo13) >> 13, lo13
    r0 = ((r + gamma2 - 1) % alpha) - (gamma2 - 1)          # r mod+- alpha in (-gamma2, gamma2]
    wrap = (r - r0) == q - 1
    d_hi = np.where(wrap, 0, (r - r0) // alpha)
    d_lo = np.where(wrap, r0 - 1, r0)
    u1 = np.where(d_lo > 0, (d_hi + 1) % m, (d_hi - 1) % m)
    got = np.concatenate([eng.dbg_rounding(divisor, lo, min(1 << 22, q - lo)) for lo in range(0, q, 1 << 22)], axis=1)
    for name, exp, g in (("p2r_hi", p2_hi, got[0]), ("p2r_lo", p2_lo, got[1]), ("dec_hi", d_hi, got[2]),
                         ("dec_lo", d_lo, got[3]), ("use0", d_hi, got[4]), ("use1", u1, got[5])):
        bad = np.flatnonzero(exp != g)
        assert bad.size == 0, (name, bad[:5], exp[bad[:5]], g[bad[:5]])
    rs = np.random.default_rng(5)
    for v in np.concatenate([rs.integers(0, q, 3000), [0, 1, q - 1, q - 2, gamma2, gamma2 + 1, q - 1 - gamma2, q - gamma2]]):
        v = int(v)
        assert oracle.power2round(v) == (int(p2_hi[v]), int(p2_lo[v]))
        assert oracle.decompose(v, gamma2) == (int(d_hi[v]), int(d_lo[v]))
        assert oracle.use_hint(1, v, gamma2) == int(u1[v]) and oracle.use_hint(0, v, gamma2) == int(d_hi[v])
