"""The command-line front end (tools/dilithium_b200), exercised the way the reference tests
its own tool (proj/tests/test_cli.cpp:61-175): round trips at every level, hex files, batch
sign / verify with a corrupted signature, the reference's known-answer vectors, exit codes
0 / 1 / 2, the bench CSV schema.  -m gpu (argument errors are covered on CPU in
test_cabi_cpu.py)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "dilithium_b200")


def run(*args):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)
    return r.returncode, r.stdout, r.stderr


@pytest.fixture(scope="module", autouse=True)
def built():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools"), "all"], check=True)


@pytest.mark.parametrize("level", [2, 3, 5, 65])  # 65 = ML-DSA-65 (FIPS 204 mode)
def test_roundtrip(tmp_path, level, oracle):
    pk, sk, sig, msg, msg2 = (tmp_path / n for n in ("pk.bin", "sk.bin", "sig.bin", "msg.bin", "msg2.bin"))
    msg.write_bytes(b"hello dilithium\n")
    msg2.write_bytes(b"hello dilithiun\n")
    seed = "%064x" % (level * 0x1234567)
    assert run("keygen", "--level", level, "--pk", pk, "--sk", sk, "--seed", seed)[0] == 0
    assert (pk.read_bytes(), sk.read_bytes()) == oracle.keygen(level, bytes.fromhex(seed))
    assert run("sign", "--level", level, "--sk", sk, "--in", msg, "--out", sig)[0] == 0
    assert sig.read_bytes() == oracle.sign(level, sk.read_bytes(), msg.read_bytes())[0]
    rc, out, _ = run("verify", "--level", level, "--pk", pk, "--in", msg, "--sig", sig)
    assert rc == 0 and out.strip() == "accept"
    rc, out, _ = run("verify", "--level", level, "--pk", pk, "--in", msg2, "--sig", sig)
    assert rc == 1 and out.strip() == "reject"
    # truncated signature file: malformed input, not "reject"
    short = tmp_path / "short.sig"
    short.write_bytes(sig.read_bytes()[:-1])
    assert run("verify", "--level", level, "--pk", pk, "--in", msg, "--sig", short)[0] == 2
    # broken hint encoding (count byte above omega): exit 2 as the reference's unpack_sig check
    bad = bytearray(sig.read_bytes())
    bad[-1] = 0xFF
    (tmp_path / "bad.sig").write_bytes(bytes(bad))
    assert run("verify", "--level", level, "--pk", pk, "--in", msg, "--sig", tmp_path / "bad.sig")[0] == 2
    # keygen without a seed draws a fresh key that still round-trips
    assert run("keygen", "--level", level, "--pk", tmp_path / "p2", "--sk", tmp_path / "s2")[0] == 0
    assert (tmp_path / "p2").read_bytes() != pk.read_bytes()


def test_hex_files(tmp_path):
    msg = tmp_path / "msg.bin"
    msg.write_bytes(bytes(range(200)))
    args = ("--level", 2, "--out-format", "hex")
    assert run("keygen", *args, "--pk", tmp_path / "pk.hex", "--sk", tmp_path / "sk.hex")[0] == 0
    text = (tmp_path / "pk.hex").read_text()
    assert len(text) == 2 * 1312 + 1 and text.endswith("\n") and text.strip() == text.strip().lower()
    assert run("sign", *args, "--sk", tmp_path / "sk.hex", "--in", msg, "--out", tmp_path / "sig.hex")[0] == 0
    assert run("verify", "--level", 2, "--pk", tmp_path / "pk.hex", "--in", msg, "--sig", tmp_path / "sig.hex")[0] == 0
    assert run("sign", "--level", 3, "--sk", tmp_path / "sk.hex", "--in", msg, "--out", tmp_path / "x")[0] == 2


def test_batch_sign_verify(tmp_path, oracle):
    level = 3
    pk, sk = tmp_path / "pk3.bin", tmp_path / "sk3.bin"
    assert run("keygen", "--level", level, "--pk", pk, "--sk", sk, "--seed", "ab" * 32)[0] == 0
    msgs = []
    for i in range(12):
        m = tmp_path / ("m%02d.txt" % i)
        m.write_bytes(b"message %d " % i * (i + 1))
        msgs.append(m)
    sigs, trace = tmp_path / "sigs", tmp_path / "trace.csv"
    assert run("batch-sign", "--level", level, "--sk", sk, "--out-dir", sigs, "--workers", 3, "--trace", trace, *msgs)[0] == 0
    for m in msgs:
        s = (sigs / (m.name + ".sig")).read_bytes()
        assert s == oracle.sign(level, sk.read_bytes(), m.read_bytes())[0]
    rows = trace.read_text().strip().splitlines()
    assert rows[0] == "stream,round,unfinished,assigned,speculative,idle_slots,newly_done"
    recs = [list(map(int, r.split(","))) for r in rows[1:]]
    assert sum(r[6] for r in recs) == 12 and all(r[3] >= 1 and r[3] <= r[2] * 9 for r in recs)
    rc, out, _ = run("batch-verify", "--level", level, "--pk", pk, "--sig-dir", sigs, *msgs)
    assert rc == 0 and out.count("accept") == 12
    victim = sigs / (msgs[4].name + ".sig")
    b = bytearray(victim.read_bytes())
    b[100] ^= 0x10
    victim.write_bytes(bytes(b))
    (sigs / (msgs[7].name + ".sig")).unlink()  # missing signature rejects too
    rc, out, _ = run("batch-verify", "--level", level, "--pk", pk, "--sig-dir", sigs, *msgs)
    lines = out.strip().splitlines()
    assert rc == 1 and [l.endswith("reject") for l in lines] == [i in (4, 7) for i in range(12)]
    assert run("batch-sign", "--level", level, "--sk", sk, "--out-dir", sigs, "--psi", 13, *msgs)[0] == 2


def test_known_answer_vectors(tmp_path, kat):
    """The reference's KAT (tests/vectors/ref_vectors.hpp:26-39) through the tool."""
    msg = tmp_path / "kat_msg.bin"
    msg.write_bytes(bytes.fromhex(kat["kKatMessage"]))
    for level in (2, 3, 5):
        pk, sk, sig = (tmp_path / ("kat_%s%d.bin" % (n, level)) for n in ("pk", "sk", "sig"))
        assert run("keygen", "--level", level, "--pk", pk, "--sk", sk, "--seed", kat["kKatSeed"])[0] == 0
        assert pk.read_bytes().hex() == kat["kKatPk%d" % level] and sk.read_bytes().hex() == kat["kKatSk%d" % level]
        assert run("sign", "--level", level, "--sk", sk, "--in", msg, "--out", sig)[0] == 0
        assert sig.read_bytes().hex() == kat["kKatSig%d" % level]
        assert run("verify", "--level", level, "--pk", pk, "--in", msg, "--sig", sig)[0] == 0
        flipped = bytearray(sig.read_bytes())
        flipped[40] ^= 1
        (tmp_path / "f.sig").write_bytes(bytes(flipped))
        assert run("verify", "--level", level, "--pk", pk, "--in", msg, "--sig", tmp_path / "f.sig")[0] == 1


def test_bench_csv():
    rc, out, _ = run("bench", "--level", 2, "--phi", 64, "--workers", 2, "--reps", 1)
    lines = out.strip().splitlines()
    assert rc == 0
    assert lines[0] == ("schema,mode,op,level,phi,psi,workers,streams,reps,throughput_ops_s,"
                        "mean_latency_us,attempts_mean")
    assert [l.split(",")[2] for l in lines[1:]] == ["keygen", "sign", "verify"]
    assert all(l.split(",")[0] == "1" and float(l.split(",")[9]) > 0 for l in lines[1:])
    rc, out, _ = run("bench", "--level", 3, "--phi", 50, "--streams", 3, "--reps", 1)
    assert rc == 0 and [l.split(",")[7] for l in out.strip().splitlines()[1:]] == ["3", "3", "3"]


def test_sweep_modes():
    """tools/dilithium_cli.cpp:448-514: the three sensitivity modes in the bench CSV schema."""
    rc, out, err = run("sweep", "--level", 2, "--phi", 512, "--reps", 1, "--psi-min", 64, "--psi-max", 512,
                       "--psi-steps", 3, "--streams-max", 4)
    assert rc == 0, err
    lines = out.strip().splitlines()
    assert lines[0] == ("schema,mode,op,level,phi,psi,workers,streams,reps,throughput_ops_s,"
                        "mean_latency_us,attempts_mean")
    rows = [l.split(",") for l in lines[1:]]
    modes = [r[1] for r in rows]
    assert modes == ["sweep-psi"] * 3 + ["sweep-batch"] * 5 + ["sweep-streams"] * 3
    assert [r[5] for r in rows[:3]] == ["64", "288", "512"]          # psi grid
    assert [r[4] for r in rows[3:8]] == ["32", "64", "128", "256", "512"]  # phi/16 doubling to phi
    assert [r[7] for r in rows[8:]] == ["1", "2", "4"]               # batches in flight
    assert all(r[0] == "1" and r[2] == "sign" and float(r[9]) > 0 and 1.5 < float(r[11]) < 12.0 for r in rows)
    assert run("sweep", "--level", 2, "--streams-max", 64)[0] == 2
