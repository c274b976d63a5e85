"""Pin the C restatement oracle against the reference's own known answers and
against golden vectors produced by the reference itself (oracle/_ref).  CPU only."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests import golden_util as G


def test_frozen_negacyclic_product():
    # test_ring.cpp:129-142: (1+2x+3x^2+4x^3)(5+6x+7x^2+8x^3) mod (x^4+1, 97)
    assert list(O.schoolbook(97, [1, 2, 3, 4], [5, 6, 7, 8])) == [41, 61, 2, 60]
    assert list(O.schoolbook(97, [0, 0, 0, 1], [0, 0, 1, 0])) == [0, 96, 0, 0]


def test_frozen_crt():
    # test_ring.cpp:159-166
    assert O.crt_centered([97, 113], [53, 28]) == 5000.0
    assert O.crt_centered([97, 113], [7, 51]) == -3000.0
    assert O.crt_centered([97, 113], [0, 0]) == 0.0
    assert O.crt_centered([97, 113], [96, 112]) == -1.0


def test_frozen_encoder():
    # test_ckks.cpp:95-110
    c = O.encode_values(4, [1.0, 2.0])
    r = math.sqrt(2.0) / 4.0
    np.testing.assert_allclose(c, [1.5, -r, 0.0, r], atol=1e-12)
    back = O.decode_coeffs(4, c, 2)
    np.testing.assert_allclose(back, [1.0, 2.0], atol=1e-12)


def test_context_pinned_shape():
    # test_ring.cpp:187-196 default context: 8192, seven 30-bit primes
    ctx = O.Context(8192, [30] * 7, 30)
    assert ctx.L == 6
    assert all(int(q) % 16384 == 1 for q in ctx.primes)
    assert all(int(ctx.primes[i]) < int(ctx.primes[i - 1]) for i in range(1, 7))


def test_survey_primes():
    # SURVEY §8(d) probe values from the reference's generate_ntt_primes
    assert list(map(int, O.Context(8192, [40, 30, 40]).primes)) == [1099511480321, 1073692673, 1099510890497]
    assert list(map(int, O.Context(8192, [36, 26, 26, 26, 26, 26, 36], 26).primes)) == [
        68719230977, 67043329, 66994177, 66961409, 66813953, 66551809, 68718428161]


def test_ntt_roundtrip_and_schoolbook():
    ctx = O.Context(64, [30])
    q = int(ctx.primes[0])
    rng = np.random.default_rng(3)
    for _ in range(5):
        a = rng.integers(0, q, 64, dtype=np.uint64)
        b = rng.integers(0, q, 64, dtype=np.uint64)
        assert np.array_equal(ctx.intt(0, ctx.ntt(0, a)), a)
        fa, fb = ctx.ntt(0, a), ctx.ntt(0, b)
        prod = np.array([(int(x) * int(y)) % q for x, y in zip(fa, fb)], dtype=np.uint64)
        assert np.array_equal(ctx.intt(0, prod), O.schoolbook(q, a, b))


@pytest.mark.parametrize("name", G.PRIM_CASES)
def test_oracle_matches_reference_goldens(name):
    g = G.load_prims(name)
    mine = G.oracle_prims(name)
    missing = [k for k in g["arrays"] if k not in mine]
    assert not missing, missing
    bad = [k for k, v in g["arrays"].items() if G.sha(mine[k]) != v["sha256"]]
    assert not bad, f"oracle differs from reference on {bad}"
