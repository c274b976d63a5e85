"""GPU slot encoder (hg_encode / hg_encode_batch, hg_encode.cu) against the
oracle's restatement of SlotEncoder::values_to_coeffs + CkksBackend::encode
(encoder.hpp:58-77, ckks_backend.hpp:182-197): bit-exact NTT-form plaintexts,
including the split-FFT path (N > 8192), partial slot counts, strided batch
columns and the overflow error."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _empty(words):
    import torch

    return torch.zeros(words, dtype=torch.int64, device="cuda")


def _host(t):
    return t.cpu().numpy().view(np.uint64).copy()


CASES = [(4096, [30, 30, 30]), (8192, [36, 26, 36]), (16384, [50, 30, 50]), (32768, [30, 30])]


@pytest.mark.parametrize("n,bits", CASES)
def test_encode_matches_oracle(n, bits, cuda_ok):
    import paper_1810_10121_b200 as P
    from oracle import oracle as O

    ctx = P.Context(n, bits, 30 if bits[1] == 30 else 26, security=0)
    octx = O.Context(n, bits, 30 if bits[1] == 30 else 26)
    rng = np.random.default_rng(n)
    L = ctx.L
    for count, lo, hi in [(n // 2, -1.0, 1.0), (n // 2 - 3, 0.0, 255.0), (1, -5.0, 5.0), (0, 0.0, 0.0), (77, -1e3, 1e3)]:
        v = rng.uniform(lo, hi, count)
        pt = _empty(ctx.words(L))
        P.call("hg_encode", ctx, v.ctypes.data_as(P.f64p), v.size, L, ctx.default_scale, pt)
        want = octx.encode(v, L, octx.scale)
        assert np.array_equal(_host(pt), want), f"n={n} count={count}"


def test_encode_batch_strided_columns(cuda_ok):
    """[batch][elements] row-major input, columns read with elem_stride = elements (pack_cipher)."""
    import torch

    import paper_1810_10121_b200 as P
    from oracle import oracle as O

    n, bits = 8192, [36, 26, 26, 36]
    ctx = P.Context(n, bits, 26, security=0)
    octx = O.Context(n, bits, 26)
    batch, elems = 4000, 7
    x = np.random.default_rng(3).integers(0, 256, (batch, elems)).astype(np.float64) / 255.0
    for lvl in (ctx.L, 1):
        out = _empty(elems * ctx.words(lvl))
        # host source
        P.call("hg_encode_batch", ctx, x.ctypes.data, elems, batch, 1, elems, lvl, ctx.default_scale, out)
        got = _host(out).reshape(elems, -1)
        # device source gives the same words
        xd = torch.from_numpy(x).cuda()
        out2 = _empty(elems * ctx.words(lvl))
        P.call("hg_encode_batch", ctx, xd, elems, batch, 1, elems, lvl, ctx.default_scale, out2)
        assert np.array_equal(_host(out2).reshape(elems, -1), got)
        for e in range(elems):
            assert np.array_equal(got[e], octx.encode(x[:, e].copy(), lvl, octx.scale)), f"column {e} level {lvl}"


def test_encode_overflow_is_validation_error(cuda_ok):
    import paper_1810_10121_b200 as P

    ctx = P.Context(4096, [30, 30, 30], 30, security=0)
    v = np.array([1e15, 0.5])  # coefficients ~ v * 2/N * scale = 5e20 > 9e18
    pt = _empty(ctx.words(ctx.L))
    with pytest.raises(P.HEError) as ei:
        P.call("hg_encode", ctx, v.ctypes.data_as(P.f64p), v.size, ctx.L, 2.0 ** 30, pt)
    assert ei.value.category == "validation" and "overflows" in str(ei.value)
    v = np.array([np.nan])
    with pytest.raises(P.HEError):
        P.call("hg_encode", ctx, v.ctypes.data_as(P.f64p), v.size, ctx.L, 2.0 ** 30, pt)
    v = np.zeros(4096 // 2 + 1)
    with pytest.raises(P.HEError) as ei:
        P.call("hg_encode", ctx, v.ctypes.data_as(P.f64p), v.size, ctx.L, 2.0 ** 30, pt)
    assert ei.value.category == "capacity"
