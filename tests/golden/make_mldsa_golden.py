#!/usr/bin/env python3
"""Generates tests/golden/mldsa_openssl.json: ML-DSA-44/65/87 (FIPS 204) vectors from an
independent implementation -- OpenSSL through the `cryptography` package -- used to pin the
FIPS 204 mode of the CPU oracle (levels 44 / 65 / 87), which the reference does not have.

Run in the build container (cryptography >= 48 with an OpenSSL that has ML-DSA):
    python tests/golden/make_mldsa_golden.py
Per level and seed it records
  * seed -> public key bytes (OpenSSL keygen, FIPS 204 Alg. 6);
  * OpenSSL signatures (hedged, so not reproducible) over fixed messages, empty context:
    the oracle must ACCEPT them;
  * the oracle's own deterministic signatures over the same messages, recorded only after
    OpenSSL ACCEPTED them here (and rejected a corrupted copy): a regression anchor.
Deterministic-mode signature BYTES have no independent known-answer vector in this image
(the binding exposes hedged signing only); that limit is stated in oracle/dilithium_oracle.h."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from cryptography.exceptions import InvalidSignature  # noqa: E402
from cryptography.hazmat.primitives.asymmetric import mldsa  # noqa: E402
from tests.cpu_checkers import load_oracle  # noqa: E402

KEYS = {44: mldsa.MLDSA44PrivateKey, 65: mldsa.MLDSA65PrivateKey, 87: mldsa.MLDSA87PrivateKey}
oracle = load_oracle()
out = {"generator": "tests/golden/make_mldsa_golden.py", "levels": {}}
for level, cls in KEYS.items():
    cases = []
    for s in range(2):
        seed = bytes((17 * s + 3 * i + level) & 0xFF for i in range(32))
        sk_obj = cls.from_seed_bytes(seed)
        pk = sk_obj.public_key().public_bytes_raw()
        opk, osk = oracle.keygen(level, seed)
        assert opk == pk, "oracle keygen differs from OpenSSL at level %d" % level
        msgs = [b"", bytes(range(200)), b"FIPS 204 interop message %d\n" % s * 9]
        sigs = []
        for m in msgs:
            theirs = sk_obj.sign(m)  # hedged
            assert oracle.verify(level, pk, m, theirs) == 1, "oracle rejects an OpenSSL signature"
            bad = bytearray(theirs)
            bad[len(bad) // 2] ^= 1
            assert oracle.verify(level, pk, m, bytes(bad)) == 0
            ours, attempts = oracle.sign(level, osk, m)
            sk_obj.public_key().verify(ours, m)  # raises if OpenSSL rejects the oracle's signature
            bad = bytearray(ours)
            bad[7] ^= 0x10
            try:
                sk_obj.public_key().verify(bytes(bad), m)
                raise AssertionError("OpenSSL accepted a corrupted signature")
            except InvalidSignature:
                pass
            sigs.append({"msg": m.hex(), "openssl_sig": theirs.hex(), "oracle_sig": ours.hex(),
                         "oracle_attempts": attempts})
        # non-empty context strings (FIPS 204 Alg. 2 / 3): one short, one of maximal length
        ctx_sigs = []
        for ctx in (b"ctx-%d" % s, bytes((i * 7 + level) & 0xFF for i in range(255))):
            m = b"message under a context string %d" % s
            oracle.set_mldsa_context(ctx)
            theirs = sk_obj.sign(m, ctx)
            assert oracle.verify(level, pk, m, theirs) == 1
            ours, attempts = oracle.sign(level, osk, m)
            sk_obj.public_key().verify(ours, m, ctx)
            oracle.set_mldsa_context(b"")
            assert oracle.verify(level, pk, m, theirs) == 0  # wrong context rejects
            ctx_sigs.append({"ctx": ctx.hex(), "msg": m.hex(), "openssl_sig": theirs.hex(),
                             "oracle_sig": ours.hex(), "oracle_attempts": attempts})
        cases.append({"seed": seed.hex(), "pk": pk.hex(), "sk_sha_len": len(osk), "sigs": sigs,
                      "ctx_sigs": ctx_sigs})
    out["levels"][str(level)] = cases
path = os.path.join(ROOT, "tests", "golden", "mldsa_openssl.json")
json.dump(out, open(path, "w"), indent=0)
print("wrote", path, os.path.getsize(path), "bytes")
