"""Pins the CPU oracle (oracle/dilithium_oracle.c) -- CPU only, no GPU.

Three anchors, per the parity contract:
  * the reference's own known-answer vectors (tests/golden/ref_kat.json, extracted
    from proj/tests/vectors/ref_vectors.hpp; consumed by the reference at
    tests/test_keccak.cpp:31-76, tests/test_sampling.cpp:72-140, tests/test_scheme.cpp:27-69)
  * seeded outputs of the reference itself (tests/golden/ref_seeded.json)
  * the reference compiled in place (oracle/_ref) on fresh random inputs
"""
import hashlib
import os

import numpy as np
import pytest

from tests.cpu_checkers import PARAMS, Q, mt19937_64


def test_keccak_kats(oracle, kat):
    out = oracle.keccak_f1600([0] * 25)
    assert [int(v) for v in out] == kat["kKeccakZeroState"]
    out = oracle.keccak_f1600(kat["kKeccakRandIn"])
    assert [int(v) for v in out] == kat["kKeccakRandOut"]


def test_shake_kats(oracle, kat):
    assert oracle.shake(128, b"", 64).hex() == kat["kShake128Empty"]
    assert oracle.shake(256, b"", 64).hex() == kat["kShake256Empty"]
    assert oracle.shake(128, b"\xa3" * 200, 64).hex() == kat["kShake128Msg1600"]
    assert oracle.shake(256, b"\xa3" * 200, 64).hex() == kat["kShake256Msg1600"]


def test_shake_vs_hashlib(oracle):
    rng = mt19937_64(7)
    for n in [0, 1, 31, 135, 136, 137, 167, 168, 169, 271, 272, 273, 1312, 2592]:
        data = rng.bytes(n)
        assert oracle.shake(128, data, 400) == hashlib.shake_128(data).digest(400)
        assert oracle.shake(256, data, 400) == hashlib.shake_256(data).digest(400)


def test_sampler_kats(oracle, kat):
    rho0 = bytes(32)
    rp = bytes(range(64))
    assert oracle.expand_a(rho0, 0, 0).tolist() == kat["kExpandA_r0_00"]
    assert oracle.expand_a(rho0, 1, 2).tolist() == kat["kExpandA_r0_12"]
    assert oracle.expand_s(rp, 0, 2).tolist() == kat["kExpandS_eta2_n0"]
    assert oracle.expand_s(rp, 7, 2).tolist() == kat["kExpandS_eta2_n7"]
    assert oracle.expand_s(rp, 0, 4).tolist() == kat["kExpandS_eta4_n0"]
    assert oracle.expand_mask(rp, 0, 1 << 17, 18).tolist() == kat["kExpandMask_g17_n0"]
    assert oracle.expand_mask(rp, 3, 1 << 17, 18).tolist() == kat["kExpandMask_g17_n3"]
    assert oracle.expand_mask(rp, 0, 1 << 19, 20).tolist() == kat["kExpandMask_g19_n0"]
    ct = bytes(range(32))
    assert oracle.sample_in_ball(ct, 39).tolist() == kat["kBall_tau39"]
    assert oracle.sample_in_ball(ct, 49).tolist() == kat["kBall_tau49"]
    assert oracle.sample_in_ball(ct, 60).tolist() == kat["kBall_tau60"]


@pytest.mark.parametrize("level", [2, 3, 5])
def test_full_kat(oracle, kat, level):
    seed = bytes.fromhex(kat["kKatSeed"])
    msg = bytes.fromhex(kat["kKatMessage"])
    pk, sk = oracle.keygen(level, seed)
    assert pk.hex() == kat["kKatPk%d" % level]
    assert sk.hex() == kat["kKatSk%d" % level]
    sig, att = oracle.sign(level, sk, msg)
    assert sig.hex() == kat["kKatSig%d" % level]
    assert att == kat["kKatAttempts%d" % level]
    assert oracle.verify(level, pk, msg, sig) == 1
    assert oracle.verify(level, pk, msg + b"x", sig) == 0


@pytest.mark.parametrize("level", [2, 3, 5])
def test_seeded_fixture(oracle, seeded, level):
    fx = seeded[str(level)]
    rng = mt19937_64(fx["seed"])
    n = fx["n"]
    zetas = rng.bytes(32 * n)
    msgs = [rng.bytes(1 + (i * 37) % 97) for i in range(n)]
    h_pk, h_sk, h_sig = hashlib.sha3_256(), hashlib.sha3_256(), hashlib.sha3_256()
    atts = []
    for i in range(n):
        pk, sk = oracle.keygen(level, zetas[32 * i:32 * i + 32])
        sig, att = oracle.sign(level, sk, msgs[i])
        if i == 0:
            assert pk.hex() == fx["first"]["pk"] and sk.hex() == fx["first"]["sk"]
            assert sig.hex() == fx["first"]["sig"]
        h_pk.update(pk); h_sk.update(sk); h_sig.update(sig)
        atts.append(att)
    assert h_pk.hexdigest() == fx["pk_sha3"]
    assert h_sk.hexdigest() == fx["sk_sha3"]
    assert h_sig.hexdigest() == fx["sig_sha3"]
    assert atts == fx["attempts"]


def test_ntt_vs_ref(oracle, ref):
    rng = np.random.default_rng(3)
    for _ in range(50):
        a = rng.integers(0, Q, 256, dtype=np.int32)
        assert np.array_equal(oracle.ntt(a), np.mod(ref.ntt(a), Q))
        assert np.array_equal(oracle.intt(a), np.mod(ref.intt(a), Q))
        assert np.array_equal(oracle.intt(oracle.ntt(a)), a)


def test_rounding_vs_ref(oracle, ref):
    rng = np.random.default_rng(4)
    edge = [0, 1, 4095, 4096, 4097, 8191, 8192, Q - 1, Q - 2, (Q - 1) // 2, (Q - 1) // 2 + 1]
    vals = edge + rng.integers(0, Q, 4000).tolist()
    for g2 in (PARAMS[2]["gamma2"], PARAMS[3]["gamma2"]):
        vals2 = vals + [g2 * m + d for m in range(0, 2 * (Q - 1) // (2 * g2) + 1) for d in (-1, 0, 1)
                        if 0 <= g2 * m + d < Q]
        for r in vals2:
            assert oracle.decompose(r, g2) == ref.decompose(r, g2)
            for h in (0, 1):
                assert oracle.use_hint(h, r, g2) == ref.use_hint(h, r, g2)
        for r, z in zip(vals2[:3000], rng.integers(0, Q, 3000).tolist()):
            assert oracle.make_hint(z, r, g2) == ref.make_hint(z, r, g2)
    for a in vals:
        assert oracle.power2round(a) == ref.power2round(a)


def test_samplers_vs_ref(oracle, ref):
    rng = mt19937_64(5)
    for t in range(40):
        rho, rp, ct = rng.bytes(32), rng.bytes(64), rng.bytes(32)
        i, j, nonce = t % 8, (t * 3) % 7, (t * 1021) & 0xFFFF
        assert np.array_equal(oracle.expand_a(rho, i, j), ref.expand_a(rho, i, j))
        for eta in (2, 4):
            assert np.array_equal(oracle.expand_s(rp, nonce, eta), ref.expand_s(rp, nonce, eta))
        for g1, zb in ((1 << 17, 18), (1 << 19, 20)):
            assert np.array_equal(oracle.expand_mask(rp, nonce, g1, zb),
                                  ref.expand_mask(rp, nonce, g1, zb))
        for tau in (39, 49, 60):
            assert np.array_equal(oracle.sample_in_ball(ct, tau), ref.sample_in_ball(ct, tau))


@pytest.mark.parametrize("level", [2, 3, 5])
def test_scheme_vs_ref(oracle, ref, level):
    rng = mt19937_64(600 + level)
    P = PARAMS[level]
    for t in range(12):
        zeta = rng.bytes(32)
        msg = rng.bytes(rng() % 200)
        pk, sk = oracle.keygen(level, zeta)
        assert (pk, sk) == ref.keygen(level, zeta)
        sig, att = oracle.sign(level, sk, msg)
        assert (sig, att) == ref.sign(level, sk, msg)
        rp = rng.bytes(64)
        assert oracle.sign(level, sk, msg, rp) == ref.sign(level, sk, msg, rp)
        assert oracle.verify(level, pk, msg, sig) == 1 == ref.verify(level, pk, msg, sig)
        # bit flips, truncation (tests/test_scheme.cpp:73-108,195-202)
        bad = bytearray(sig)
        pos = rng() % len(bad)
        bad[pos] ^= 1 << (rng() % 8)
        assert oracle.verify(level, pk, msg, bytes(bad)) == ref.verify(level, pk, msg, bytes(bad))
        assert oracle.verify(level, pk, msg, sig[:-1]) == 0
        assert oracle.verify(level, pk[:-1], msg, sig) == 0
        # hint region corruptions exercise the strict decoder (packing.hpp:122-140)
        for off in range(1, P["omega"] + P["k"] + 1, 7):
            bad = bytearray(sig)
            bad[-off] ^= 0x01 << (off % 8)
            assert oracle.verify(level, pk, msg, bytes(bad)) == ref.verify(level, pk, msg, bytes(bad))
        # single attempts: accept flag, reject stage, c~, z
        mu, rho_p = rng.bytes(64), rng.bytes(64)
        for kappa in (0, P["l"], 65535 - 2):
            ro, so, co, zo, ho = oracle.sign_attempt(level, sk, mu, rho_p, kappa)
            rr, sr, cr, zr, hr = ref.sign_attempt(level, sk, mu, rho_p, kappa)
            assert ro == rr and co == cr
            if rr == 1:
                assert np.array_equal(zo, zr) and np.array_equal(ho, hr)
            else:
                assert so == sr


def test_malformed_sk(oracle, ref):
    pk, sk = oracle.keygen(2, bytes(32))
    bad = bytearray(sk)
    bad[96] = 0xFF  # eta field raw 7 > 2*eta (packing.hpp:79-86)
    with pytest.raises(ValueError):
        oracle.sign(2, bytes(bad), b"m")
    with pytest.raises(ValueError):
        ref.sign(2, bytes(bad), b"m")


# ---- FIPS 204 (ML-DSA-44 / 65 / 87) mode of the oracle -----------------------------------
# Not in the reference (proj/README.md:120-121 declares it a non-goal): pinned against
# OpenSSL through the fixtures written by tests/golden/make_mldsa_golden.py.

@pytest.fixture(scope="module")
def mldsa_golden():
    import json
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mldsa_openssl.json")))


@pytest.mark.parametrize("level", [44, 65, 87])
def test_mldsa_oracle_against_openssl_vectors(oracle, mldsa_golden, level):
    for case in mldsa_golden["levels"][str(level)]:
        seed, pk = bytes.fromhex(case["seed"]), bytes.fromhex(case["pk"])
        opk, osk = oracle.keygen(level, seed)
        assert opk == pk and len(osk) == case["sk_sha_len"]  # OpenSSL's public key for this seed
        for s in case["sigs"]:
            msg = bytes.fromhex(s["msg"])
            theirs = bytes.fromhex(s["openssl_sig"])
            assert oracle.verify(level, pk, msg, theirs) == 1          # OpenSSL's signature verifies
            assert oracle.verify(level, pk, msg + b"x", theirs) == 0
            flipped = bytearray(theirs)
            flipped[len(flipped) // 3] ^= 4
            assert oracle.verify(level, pk, msg, bytes(flipped)) == 0
            ours, att = oracle.sign(level, osk, msg)                    # OpenSSL accepted these bytes
            assert ours.hex() == s["oracle_sig"] and att == s["oracle_attempts"]
            assert oracle.verify(level, pk, msg, ours) == 1
        for s in case["ctx_sigs"]:  # FIPS 204 context strings
            ctx, msg, theirs = (bytes.fromhex(s[k]) for k in ("ctx", "msg", "openssl_sig"))
            assert oracle.verify(level, pk, msg, theirs) == 0      # empty context: reject
            oracle.set_mldsa_context(ctx)
            try:
                assert oracle.verify(level, pk, msg, theirs) == 1
                ours, att = oracle.sign(level, osk, msg)
                assert ours.hex() == s["oracle_sig"] and att == s["oracle_attempts"]
            finally:
                oracle.set_mldsa_context(b"")


def test_reference_scheduler_commit_rule(ref):
    """scheduler.hpp:58-136 replayed on random validity tables: whatever (phi, psi, speculate), the
    reference's NonceScheduler accepts each task's FIRST valid attempt and executes every attempt
    below it -- the rule the device scheduler's parity tests (assignment log, attempt counts) rely on."""
    import numpy as np
    rng = np.random.default_rng(58)
    for _ in range(40):
        phi = int(rng.integers(1, 200))
        psi = int(rng.integers(1, 2 * phi + 1))
        depth = 24
        valid = (rng.random((phi, depth)) < 0.25).astype(np.uint8)
        valid[:, -1] = 1  # every task terminates inside the table
        for speculate in (True, False):
            acc, executed = ref.scheduler_replay(phi, psi, 4, speculate, valid)
            first = valid.argmax(axis=1)
            assert np.array_equal(acc, first)
            assert executed >= int((first + 1).sum())  # every attempt up to the accepted one ran
            if not speculate:
                assert executed == int((first + 1).sum())  # and without speculation nothing else
