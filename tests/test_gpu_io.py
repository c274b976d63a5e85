"""Key and ciphertext files (keyio.hpp HEGK / HEGC) against files written by the
unmodified reference (tests/golden/io_n1024, made by oracle/_ref/ref_harness io):
the GPU loads the reference's keys and ciphertext and decrypts the reference's
values bit for bit, and the files the GPU writes are byte-identical to the
reference's for the same keys / ciphertext."""
import json
import os
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
IO = os.path.join(ROOT, "tests", "golden", "io_n1024")


def _case():
    with open(os.path.join(IO, "case.json")) as f:
        return json.load(f)


def _read(name):
    with open(os.path.join(IO, name), "rb") as f:
        return f.read()


def test_load_reference_keys_and_ciphertext(cuda_ok):
    import torch

    import paper_1810_10121_b200 as P

    ctx, keys = P.Keys.load(os.path.join(IO, "keys.hegk"))
    case = _case()
    assert ctx.n == case["n"] and ctx.bits == case["bits"] and ctx.scale_bits == case["scale_bits"]
    size, level, scale = P.C.c_int(), P.C.c_int(), P.C.c_double()
    path = os.path.join(IO, "ct.hegc").encode()
    P.call("hg_ciphertext_load", ctx, path, None, 0, P.C.byref(size), P.C.byref(level), P.C.byref(scale))
    words = size.value * (level.value + 1) * ctx.n
    ct = torch.zeros(words, dtype=torch.int64, device="cuda")
    P.call("hg_ciphertext_load", ctx, path, ct, words, P.C.byref(size), P.C.byref(level), P.C.byref(scale))
    want = np.frombuffer(_read("decrypted.f64"), dtype=np.float64)
    got = np.zeros(want.size, dtype=np.float64)
    P.call("hg_decrypt", ctx, keys, ct, 1, size.value, level.value, scale.value, want.size,
           got.ctypes.data_as(P.f64p))
    assert np.array_equal(got, want), "decrypting the reference's ciphertext with its own keys on the GPU"


def test_saved_files_are_byte_identical(cuda_ok):
    import torch

    import paper_1810_10121_b200 as P

    case = _case()
    ctx = P.Context(case["n"], case["bits"], case["scale_bits"], security=0)
    keys = P.Keys(ctx, case["key_seed"])  # GPU keygen == reference generate_keys
    with tempfile.TemporaryDirectory() as d:
        kp = os.path.join(d, "k.hegk")
        keys.save(kp)
        with open(kp, "rb") as f:
            assert f.read() == _read("keys.hegk"), "HEGK differs from the reference's save_keys"
        # round trip of the reference ciphertext through the GPU
        lctx, _ = P.Keys.load(os.path.join(IO, "keys.hegk"))
        size, level, scale = P.C.c_int(), P.C.c_int(), P.C.c_double()
        src = os.path.join(IO, "ct.hegc").encode()
        P.call("hg_ciphertext_load", lctx, src, None, 0, P.C.byref(size), P.C.byref(level), P.C.byref(scale))
        words = size.value * (level.value + 1) * lctx.n
        ct = torch.zeros(words, dtype=torch.int64, device="cuda")
        P.call("hg_ciphertext_load", lctx, src, ct, words, P.C.byref(size), P.C.byref(level), P.C.byref(scale))
        cp = os.path.join(d, "c.hegc")
        P.call("hg_ciphertext_save", lctx, ct, size.value, level.value, scale.value, cp.encode())
        with open(cp, "rb") as f:
            assert f.read() == _read("ct.hegc"), "HEGC differs from the reference's save_ciphertext"


def test_bad_files_raise_reference_errors(cuda_ok):
    import paper_1810_10121_b200 as P

    with tempfile.TemporaryDirectory() as d:
        bad = os.path.join(d, "bad.hegk")
        with open(bad, "wb") as f:
            f.write(b"XXXX" + _read("keys.hegk")[4:])
        with pytest.raises(P.HEError) as ei:
            P.Keys.load(bad)
        assert ei.value.category == "io" and "bad magic" in str(ei.value)
        trunc = os.path.join(d, "trunc.hegk")
        with open(trunc, "wb") as f:
            f.write(_read("keys.hegk")[:5000])
        with pytest.raises(P.HEError) as ei:
            P.Keys.load(trunc)
        assert ei.value.category == "io" and "unexpected end of data" in str(ei.value)
