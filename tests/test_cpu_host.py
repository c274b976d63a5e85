"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
the Python-side Rng/builders reproduce the reference streams, and the
reference's error behaviour is mirrored where no GPU is needed."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "hegpu.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes

    import paper_1810_10121_b200 as P

    lib = ctypes.CDLL(P.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes binding covers the whole header
    P.lib()


def test_library_is_sm100a():
    import subprocess

    import paper_1810_10121_b200 as P

    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out[:400]


def test_no_gpu_errors_loudly():
    """Without a device the product raises (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1810_10121_b200 as P

    with pytest.raises(P.HEError) as e:
        P.Context(1024, [30, 30, 30], 30, security=0)
    assert e.value.category == "cuda"


def test_python_rng_matches_reference_rng():
    from oracle import oracle as O
    from paper_1810_10121_b200 import graphs

    for seed in (0, 1, 42, 2 ** 63 + 5):
        a, b = graphs.Rng(seed), O.Rng(seed)
        for _ in range(50):
            assert a.next() == b.next()
        for _ in range(50):
            assert a.gaussian() == b.gaussian()
    r = graphs.Rng(9)
    blk = r.next_block(257)
    r2 = graphs.Rng(9)
    assert all(int(blk[i]) == r2.next() for i in range(257))


def test_fork_labels():
    from paper_1810_10121_b200 import graphs

    # fork is const: forking twice with the same label gives the same stream
    r = graphs.Rng(7)
    assert r.fork("inputs").next() == r.fork("inputs").next()
    assert r.fork("inputs").next() != r.fork("input").next()
    assert r.fork(3).next() == r.fork(3).next()


@pytest.mark.parametrize("cfg,shape", [("c1", (8, 64)), ("c3", (8, 1, 28, 28)), ("c4", (8, 3, 32, 32)),
                                       ("c5", (8, 784))])
def test_builders_shapes_and_json(cfg, shape):
    import json

    from paper_1810_10121_b200 import graphs

    g, x, ctxp = graphs.build({"config": cfg, "batch": 8, "seed": 1})
    assert x.shape == shape
    s = json.dumps(g)
    assert json.loads(s)["format_version"] == 1
    ids = [n["id"] for n in g["nodes"]]
    assert ids == sorted(ids) and len(ids) == len(set(ids))
    if cfg == "c3":
        assert np.all((x * 255.0) == np.round(x * 255.0))  # pixels are k/255


def test_config5_weight_mix():
    from paper_1810_10121_b200 import graphs

    w = graphs.sparse_pm1_tensor(graphs.Rng(11), (200, 100), 0.05)
    z = np.mean(w == 0.0)
    pm = np.mean(np.abs(w) == 1.0)
    assert 0.55 < z < 0.65 and 0.07 < pm < 0.13


def test_golden_fixtures_are_small():
    gdir = os.path.join(ROOT, "tests", "golden")
    total = sum(os.path.getsize(os.path.join(d, f)) for d, _, fs in os.walk(gdir) for f in fs)
    assert total < 2_000_000
