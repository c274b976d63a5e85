"""GPU decode (k_decode_crt + the conjugate FFT, hg_encode.cu) against the host restatement of
CrtReconstructor::to_centered_double + SlotEncoder::coeffs_to_values (ring.hpp:438-480,
encoder.hpp:80-89, ckks_backend.hpp:493-505) and against the oracle's decrypt: bit-identical
doubles for arbitrary residues (every multiword branch: values above Q/2, one limb, 16 limbs),
every ring degree including the split-FFT path (N > 8192), and partial slot counts."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [(4096, [30, 30, 30], 30), (8192, [36, 26, 26, 26, 36], 26), (16384, [50, 30, 30, 30, 50], 30),
         (32768, [30] * 16, 30), (2048, [40, 30, 40], 30)]


def _decode(P, ctx, pt, level, scale, count, gpu):
    out = np.zeros(max(count, 1), dtype=np.float64)
    P.call("hg_set_gpu_decode", 1 if gpu else 0)
    try:
        P.call("hg_decode", ctx, pt, level, scale, count, out.ctypes.data_as(P.f64p))
    finally:
        P.call("hg_set_gpu_decode", 1)
    return out[:count]


@pytest.mark.parametrize("n,bits,sb", CASES)
def test_gpu_decode_matches_host_decode(n, bits, sb, cuda_ok):
    import torch

    import paper_1810_10121_b200 as P

    ctx = P.Context(n, bits, sb, security=0)
    rng = np.random.default_rng(n + len(bits))
    primes = ctx.primes
    for level in sorted({0, 1, ctx.L}):
        nl = level + 1
        # arbitrary residues (a uniformly random value mod Q: both signs, full magnitude), and a
        # small-magnitude plaintext (the usual case: a few limbs of headroom)
        big = np.stack([rng.integers(0, int(primes[i]), n, dtype=np.uint64) for i in range(nl)])
        small_v = rng.integers(-(1 << 40), 1 << 40, n)
        small = np.stack([(small_v % int(primes[i])).astype(np.uint64) for i in range(nl)])
        for words in (big, small):
            pt = torch.from_numpy(words.reshape(-1).view(np.int64).copy()).cuda()
            # hg_decode expects NTT form: transform the coefficient-domain rows forward first
            P.call("hg_ntt_forward", ctx, pt, nl, nl)
            for count in (n // 2, 1, 77):
                got = _decode(P, ctx, pt, level, 2.0 ** sb, count, True)
                want = _decode(P, ctx, pt, level, 2.0 ** sb, count, False)
                assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), f"n={n} level={level} count={count}"


def test_gpu_decrypt_matches_oracle(cuda_ok):
    import torch

    import paper_1810_10121_b200 as P
    from oracle import oracle as O

    n, bits, sb = 4096, [36, 26, 26, 36], 26
    ctx = P.Context(n, bits, sb, security=0)
    keys = P.Keys(ctx, 5)
    octx = O.Context(n, bits, sb)
    okeys = O.Keys(octx, 5)
    L = ctx.L
    rng = np.random.default_rng(2)
    cts = []
    for it in range(3):
        pt = octx.encode(rng.uniform(-4, 4, n // 2), L, octx.scale)
        cts.append(octx.encrypt(okeys, pt, L, 11 + it))
    x = torch.from_numpy(np.concatenate(cts).view(np.int64)).cuda()
    for count in (n // 2, 5):
        out = np.zeros(3 * count, dtype=np.float64)
        P.call("hg_decrypt", ctx, keys, x, 3, 2, L, octx.scale, count, out.ctypes.data_as(P.f64p))
        for it in range(3):
            want = octx.decrypt(okeys, cts[it], L, octx.scale, count)
            assert np.array_equal(out[it * count:(it + 1) * count].view(np.uint64), np.asarray(want).view(np.uint64))
