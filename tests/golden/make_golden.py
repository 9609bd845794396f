#!/usr/bin/env python3
"""Generates the committed golden fixtures (run in the BUILD container only).

Sources (neither is copied into the repo; only derived vectors are committed):
  1. the reference's own known-answer data file
     /root/reference/proj/tests/vectors/ref_vectors.hpp   -> ref_kat.json
  2. the unmodified reference headers compiled in place (oracle/_ref, built by
     oracle/Makefile), run on seeded inputs                -> ref_seeded.json
     (SHA3-256 digests of outputs + a few full vectors, to keep fixtures small)

Usage: python tests/golden/make_golden.py
"""
import ctypes
import hashlib
import json
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

REF_VEC = "/root/reference/proj/tests/vectors/ref_vectors.hpp"


def extract_kats():
    txt = open(REF_VEC).read()
    out = {}
    for m in re.finditer(r'inline constexpr char (\w+)\[\] = "([0-9a-f]*)";', txt):
        out[m.group(1)] = m.group(2)
    for m in re.finditer(r"inline constexpr (u?int\d+_t) (\w+)\[(\d+)\] = \{([^}]*)\};", txt):
        vals = [int(v.replace("ull", ""), 0) for v in m.group(4).split(",")]
        assert len(vals) == int(m.group(3))
        out[m.group(2)] = vals
    for m in re.finditer(r"inline constexpr int (\w+) = (\d+);", txt):
        out[m.group(1)] = int(m.group(2))
    return out


def seeded_vectors():
    from tests.cpu_checkers import load_ref, mt_bytes, PARAMS

    ref = load_ref()
    out = {}
    for level in (2, 3, 5):
        P = PARAMS[level]
        rng = mt_bytes(20221112 + level)
        n = 24
        zetas = rng(32 * n)
        msgs = [rng(1 + (i * 37) % 97) for i in range(n)]
        h_pk, h_sk, h_sig = hashlib.sha3_256(), hashlib.sha3_256(), hashlib.sha3_256()
        attempts = []
        first = {}
        for i in range(n):
            pk, sk = ref.keygen(level, zetas[32 * i:32 * i + 32])
            sig, att = ref.sign(level, sk, msgs[i])
            assert ref.verify(level, pk, msgs[i], sig) == 1
            h_pk.update(pk); h_sk.update(sk); h_sig.update(sig)
            attempts.append(att)
            if i == 0:
                first = {"pk": pk.hex(), "sk": sk.hex(), "sig": sig.hex(), "msg": msgs[0].hex()}
        out[str(level)] = {
            "seed": 20221112 + level, "n": n,
            "pk_sha3": h_pk.hexdigest(), "sk_sha3": h_sk.hexdigest(), "sig_sha3": h_sig.hexdigest(),
            "attempts": attempts, "first": first,
        }
    return out


if __name__ == "__main__":
    kat = extract_kats()
    json.dump(kat, open(os.path.join(HERE, "ref_kat.json"), "w"))
    print("ref_kat.json:", sorted(kat))
    sv = seeded_vectors()
    json.dump(sv, open(os.path.join(HERE, "ref_seeded.json"), "w"))
    print("ref_seeded.json written")
