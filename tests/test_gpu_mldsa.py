"""ML-DSA-44 / 65 / 87 (FIPS 204) on the device: levels 44 / 65 / 87 of the same engine.
Not in the reference; the checker is the oracle's FIPS 204 mode, itself pinned against
OpenSSL (tests/test_oracle.py::test_mldsa_oracle_against_openssl_vectors), plus OpenSSL's
own vectors directly (tests/golden/mldsa_openssl.json).  -m gpu."""
import json
import os

import numpy as np
import pytest

from tests.cpu_checkers import PARAMS, mt19937_64

pytestmark = pytest.mark.gpu
LEVELS = [44, 65, 87]


@pytest.fixture(scope="module")
def eng():
    from paper_2211_12265_b200 import Engine
    e = Engine(0)
    yield e
    e.close()


@pytest.fixture(scope="module")
def golden():
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mldsa_openssl.json")))


@pytest.mark.parametrize("level", LEVELS)
def test_openssl_vectors(eng, golden, level):
    """OpenSSL's public key for a seed, OpenSSL's signatures verify, the signature bytes
    OpenSSL accepted at fixture time are reproduced bit for bit."""
    for case in golden["levels"][str(level)]:
        seed, pk = bytes.fromhex(case["seed"]), bytes.fromhex(case["pk"])
        gpk, gsk = eng.keygen(level, seed)
        assert gpk == pk and len(gsk) == PARAMS[level]["sk"]
        for s in case["sigs"]:
            msg = bytes.fromhex(s["msg"])
            assert eng.verify(level, pk, msg, bytes.fromhex(s["openssl_sig"])) == 1
            assert eng.verify(level, pk, msg + b"!", bytes.fromhex(s["openssl_sig"])) == 0
            sig, att = eng.sign(level, gsk, msg)
            assert sig.hex() == s["oracle_sig"] and att == s["oracle_attempts"]
        for s in case["ctx_sigs"]:  # context strings: 5 and 255 bytes
            ctx, msg, theirs = (bytes.fromhex(s[k]) for k in ("ctx", "msg", "openssl_sig"))
            assert eng.verify(level, pk, msg, theirs) == 0
            eng.set_mldsa_context(ctx)
            try:
                assert eng.verify(level, pk, msg, theirs) == 1
                sig, att = eng.sign(level, gsk, msg)
                assert sig.hex() == s["oracle_sig"] and att == s["oracle_attempts"]
            finally:
                eng.set_mldsa_context(b"")
            with pytest.raises(Exception):
                eng.set_mldsa_context(bytes(256))


@pytest.mark.parametrize("level", LEVELS)
def test_batches_match_oracle(eng, oracle, level):
    n, nk = 400, 5
    rng = mt19937_64(8800 + level)
    zetas = np.frombuffer(rng.bytes(32 * nk), np.uint8).reshape(nk, 32)
    pks, sks = eng.batch_keygen(level, zetas)
    for i in range(nk):
        assert (pks[i].tobytes(), sks[i].tobytes()) == oracle.keygen(level, zetas[i].tobytes())
    lens = [int(rng()) % 300 for _ in range(n)]  # crosses the 136-byte block boundary of mu
    lens[:6] = [0, 1, 5, 6, 7, 70]               # around the two-byte M' prefix and tr || M' = one block
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    flat = np.frombuffer(rng.bytes(int(off[-1]) + 1), np.uint8)
    kidx = np.array([int(rng()) % nk for _ in range(n)], np.uint32)
    sigs, att, failed, _ = eng.batch_sign(level, sks, (flat, off), key_idx=kidx, return_info=True)
    assert not failed.any()
    for i in range(n):
        m = flat[int(off[i]):int(off[i + 1])].tobytes()
        assert (sigs[i].tobytes(), int(att[i])) == oracle.sign(level, sks[kidx[i]].tobytes(), m), i
    assert np.array_equal(sigs[:64], eng.batch_sign(level, sks[kidx[:64]], (flat[:int(off[64])], off[:65])))
    shared = eng.batch_sign(level, sks[0], (flat, off))
    assert shared[3].tobytes() == oracle.sign(level, sks[0].tobytes(), flat[int(off[3]):int(off[4])].tobytes())[0]
    assert eng.batch_verify(level, pks, (flat, off), sigs, key_idx=kidx).all()
    assert eng.batch_verify(level, pks[0], (flat, off), shared).all()
    bad = sigs.copy()
    pos = [0, PARAMS[level]["ct"] - 1, PARAMS[level]["ct"], bad.shape[1] - 1, bad.shape[1] // 2]
    for t, p in enumerate(pos):
        bad[t, p] ^= 1
    flags = eng.batch_verify(level, pks, (flat, off), bad, key_idx=kidx)
    for t in range(n):
        m = flat[int(off[t]):int(off[t + 1])].tobytes()
        if t < 32:
            assert flags[t] == oracle.verify(level, pks[kidx[t]].tobytes(), m, bad[t].tobytes())
    assert not flags[:len(pos)].any() and flags[len(pos):].all()


@pytest.mark.parametrize("level", LEVELS)
def test_single_attempts_and_malformed_key(eng, oracle, level):
    rng = mt19937_64(8900 + level)
    pk, sk = oracle.keygen(level, rng.bytes(32))
    n = 48
    mus = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64)
    rps = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64)
    kappas = np.array([int(rng()) % 60000 for _ in range(n)], np.uint32)
    acc, ct, z, h = eng.dbg_sign_attempt(level, np.frombuffer(sk, np.uint8), mus, rps, kappas)
    for i in range(n):
        ok, stage, oct_, oz, oh = oracle.sign_attempt(level, sk, mus[i].tobytes(), rps[i].tobytes(), int(kappas[i]))
        assert int(acc[i]) == ok
        assert ct[i].tobytes() == oct_
        if ok:
            assert np.array_equal(z[i], oz) and np.array_equal(h[i], oh)
    bad = bytearray(sk)
    bad[64 + 64] = 0xFF  # first eta field byte (the secret vectors start behind the 64-byte tr)
    with pytest.raises(ValueError):
        eng.sign(level, bytes(bad), b"x")


@pytest.mark.parametrize("level", LEVELS)
def test_context_strings_match_oracle(eng, oracle, level):
    """Every prefix length 2 .. 257 shifts the message differently inside the first Keccak
    blocks of mu; a few lengths around word and block boundaries, ragged messages."""
    rng = mt19937_64(9100 + level)
    pk, sk = oracle.keygen(level, rng.bytes(32))
    sk_a, pk_a = np.frombuffer(sk, np.uint8), np.frombuffer(pk, np.uint8)
    msgs = [rng.bytes(int(rng()) % 200) for _ in range(24)]
    try:
        for clen in (0, 1, 5, 6, 7, 13, 70, 71, 134, 254, 255):
            ctx = rng.bytes(clen)
            eng.set_mldsa_context(ctx)
            oracle.set_mldsa_context(ctx)
            sigs = eng.batch_sign(level, sk_a, msgs)
            for m, sg in zip(msgs, sigs):
                assert sg.tobytes() == oracle.sign(level, sk, m)[0], clen
            assert eng.batch_verify(level, pk_a, msgs, sigs).all()
            eng.set_mldsa_context(ctx + b"\x00" if clen < 255 else ctx[:-1])
            assert not eng.batch_verify(level, pk_a, msgs, sigs).any()
    finally:
        eng.set_mldsa_context(b"")
        oracle.set_mldsa_context(b"")


def test_hash_mldsa_prehash_mode(oracle):
    """HashML-DSA (FIPS 204 Alg. 4 / 5): M' = 1 || |ctx| || ctx || OID || PH(M).  With the SHA-512 and
    SHAKE256 OIDs set, signatures over caller-computed digests equal the oracle's pre-hash mode byte
    for byte, verify, differ from pure ML-DSA over the same bytes, and are rejected by it."""
    import hashlib
    from paper_2211_12265_b200 import Engine
    oids = {"sha512": bytes.fromhex("0609608648016503040203"),     # 2.16.840.1.101.3.4.2.3
            "shake256": bytes.fromhex("060960864801650304020C")}   # 2.16.840.1.101.3.4.2.12
    eng = Engine(0)
    try:
        for level in (44, 65, 87):
            pks, sks = eng.batch_keygen(level, np.arange(32, dtype=np.uint8))
            msgs = [bytes([i]) * (3 * i + 1) for i in range(24)]
            for name, oid in oids.items():
                dig = [hashlib.sha512(m).digest() if name == "sha512" else hashlib.shake_256(m).digest(64) for m in msgs]
                ctx = b"prehash ctx" if name == "sha512" else b""
                eng.set_mldsa_prehash(oid, ctx)
                oracle.set_mldsa_prehash(oid, ctx)
                sigs = eng.batch_sign(level, sks[0], dig)
                for i in range(len(dig)):
                    assert sigs[i].tobytes() == oracle.sign(level, sks[0].tobytes(), dig[i])[0]
                assert eng.batch_verify(level, pks[0], dig, sigs).all()
                for i in (0, 7):
                    assert oracle.verify(level, pks[0].tobytes(), dig[i], sigs[i].tobytes()) == 1
                eng.set_mldsa_prehash(b"", ctx)     # pure ML-DSA over the same bytes: other signatures
                oracle.set_mldsa_prehash(b"", ctx)
                pure = eng.batch_sign(level, sks[0], dig)
                assert not np.array_equal(pure, sigs)
                assert not eng.batch_verify(level, pks[0], dig, sigs).any()
        with pytest.raises(Exception):
            eng.set_mldsa_prehash(bytes(17))
    finally:
        oracle.set_mldsa_prehash(b"", b"")
        eng.close()
