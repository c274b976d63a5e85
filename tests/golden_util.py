"""Helpers shared by the oracle and GPU parity tests: golden fixtures and the
oracle-side recomputation of every primitive the reference harness dumps."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")

PRIM_CASES = ["n1024_30x3", "n1024_36_26x2_36", "n2048_50_30_50", "n8192_40_30_40", "n4096_30x4",
              "n16384_50_30x2_50", "n16384_30x8", "n32768_30x16", "n16384_50_30x7_50",
              # config 2's remaining (N, L) shapes
              "n4096_30x8", "n4096_30x16", "n8192_30x4", "n8192_30x8", "n8192_30x16", "n16384_30x4",
              "n16384_30x16", "n32768_30x4", "n32768_30x8"]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_prims(name: str) -> dict:
    with open(os.path.join(GOLDEN, f"prims_{name}.json")) as f:
        return json.load(f)


def load_net(name: str) -> dict:
    with open(os.path.join(GOLDEN, f"net_{name}.json")) as f:
        return json.load(f)


def harness_values(seed_vals: int, slots: int):
    """v1, v2 of ref_harness prims: Rng(77).uniform(-1, 1), slots each."""
    from oracle.oracle import Rng

    r = Rng(seed_vals)
    out = []
    for _ in range(2):
        v = np.empty(slots)
        for i in range(slots):
            u = (r.next() >> 11) * 2.0 ** -53
            v[i] = -1.0 + 2.0 * u
        out.append(v)
    return out


def oracle_prims(name: str) -> dict:
    """Recompute, with the C restatement, every array ref_harness prims dumps."""
    from oracle import oracle as O

    g = load_prims(name)
    n, sb, bits, key_seed = g["n"], g["scale_bits"], g["bits"], g["key_seed"]
    ctx = O.Context(n, bits, sb)
    L = ctx.L
    out = {"primes": ctx.primes.copy()}
    ins, intts = O.uniform_limb(1234, ctx.primes, n)
    for i in range(L + 1):
        out[f"ntt_in_{i}"] = ins[i]
        out[f"ntt_fwd_{i}"] = ctx.ntt(i, ins[i])
        out[f"intt_in_{i}"] = intts[i]
        out[f"ntt_inv_{i}"] = ctx.intt(i, intts[i])
    keys = O.Keys(ctx, key_seed)
    out["sk"], out["pk_b"], out["pk_a"] = keys.secret, keys.pk_b, keys.pk_a
    for r in range(keys.rows):
        out[f"relin_b_{r}"] = keys.relin_b[r]
        out[f"relin_a_{r}"] = keys.relin_a[r]
    slots = n // 2
    v1, v2 = harness_values(77, slots)
    out["v1"], out["v2"] = v1, v2
    scale = ctx.scale
    pt1 = ctx.encode(v1, L, scale)
    pt2 = ctx.encode(v2, L, scale)
    out["pt1"] = pt1
    c1 = ctx.encrypt(keys, pt1, L, 1001)
    c2 = ctx.encrypt(keys, pt2, L, 1002)
    out["ct1"], out["ct2"] = c1, c2
    out["zero_lm1"] = ctx.encrypt_zero(keys, L - 1, 2002)
    out["add"] = ctx.add(L, c1, c2)
    out["sub"] = ctx.sub(L, c1, c2)
    out["neg"] = ctx.negate(L, c1)
    ap = c1.copy()
    ap[: ctx.words(L)] = ctx.add(L, c1[: ctx.words(L)], pt2)
    out["add_plain"] = ap
    mp = ctx.mul_plain(L, c1, pt2)
    out["mul_plain"] = mp
    out["mul_plain_rescale"] = ctx.rescale(L, mp)
    prod = ctx.multiply_relin(keys, L, c1, c2)
    out["mul_relin"] = prod
    mr = ctx.rescale(L, prod)
    out["mul_relin_rescale"] = mr
    out["mul_relin_rescale_coeff"] = ctx.to_coeff(mr, L - 1)
    W = ctx.words(L)
    out["mod_switch"] = np.concatenate([c1[: W][: ctx.words(L - 1)], c1[W:][: ctx.words(L - 1)]])
    wv = [0.37, -1.25, 0.0625, 2.5, -0.75]
    xs = []
    for t in range(5):
        pt = ctx.encode(np.full(slots, 0.1 * (t + 1)), L, scale)
        xs.append(ctx.encrypt(keys, pt, L, 3000 + t))
        out[f"ws_x{t}"] = xs[-1]
    out["ws_weights"] = np.array(wv)
    out["weighted_sum"] = ctx.weighted_sum(L, xs, wv)
    cws = []
    for t in range(3):
        cws.append(ctx.encrypt(keys, ctx.encode_constant(wv[t], L, scale), L, 4000 + t))
        out[f"wsc_w{t}"] = cws[-1]
    out["weighted_sum_cipher"] = ctx.weighted_sum_cipher(keys, L, xs[:3], cws)
    out["dec_ct1"] = ctx.decrypt(keys, c1, L, scale, slots)
    mr_scale = scale * scale / float(ctx.primes[L])
    out["dec_mul_relin_rescale"] = ctx.decrypt(keys, mr, L - 1, mr_scale, slots)
    out["enc_coeffs_v1"] = O.encode_values(n, v1)
    return out
