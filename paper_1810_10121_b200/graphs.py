"""BASELINE.json configurations as reference-format graphs (graph_io.hpp format_version 1).

The builders mirror the reference's own helpers (builders.hpp:42-94: add_param,
add_const, add_op, add_channel_bias) and draw every value from the reference's
splitmix64 Rng (common.hpp:71-122), restated here bit for bit, so the same JSON
graph and input tensor drive both the GPU executor and the CPU reference.

Conventions; recorded in DESIGN.md and the bench line:
  * keys     = generate_keys(ctx, Rng(seed).fork("keys").next())
  * weights  = Rng(seed).fork("<config>").fork("<const id>"); N(0, v) means variance v
  * inputs   = Rng(seed).fork("inputs").fork("x")
  * exec     = ExecOptions.seed = seed; EncryptedData, bypass {true, true, 0.0}
  * "{base, rescale..., special}" is the reference list coeff_mod_bits = [base, rescale..., special].
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1


def _splitmix64(state: int):
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


class Rng:
    """heg::Rng (common.hpp:79-122)."""

    def __init__(self, seed: int = 0):
        self.s = (seed ^ 0xD1B54A32D192ED03) & M64
        self.next()
        self.next()

    def next(self) -> int:
        self.s, out = _splitmix64(self.s)
        return out

    def uniform(self, lo: float = None, hi: float = None) -> float:
        u = float(self.next() >> 11) * (2.0 ** -53)
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def uniform_int(self, n: int) -> int:
        return self.next() % n

    def next_block(self, k: int) -> np.ndarray:
        """The next k outputs at once: splitmix64 is a counter (state += golden), so
        output i is mix(state + (i+1) golden) -- vectorised, bit-identical to k next() calls."""
        with np.errstate(over="ignore"):
            st = np.uint64(self.s) + np.arange(1, k + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
            z = (st ^ (st >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        self.s = (self.s + k * 0x9E3779B97F4A7C15) & M64
        return z

    def gaussian(self) -> float:
        u1 = self.uniform()
        u2 = self.uniform()
        while u1 <= 1e-300:
            u1 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586476925286766559 * u2)

    def fork(self, label) -> "Rng":
        if isinstance(label, str):
            h = 0xCBF29CE484222325
            for c in label.encode():
                h = ((h ^ c) * 0x100000001B3) & M64
            label = h
        _, mixed = _splitmix64(self.s)
        mixed ^= (label * 0x9E3779B97F4A7C15 + 0x165667B19E3779F9) & M64
        return Rng(mixed)


# ---- graph helpers (builders.hpp:42-94) ----

class G:
    def __init__(self, name: str):
        self.name = name
        self.nodes = []

    def param(self, id_, shape):
        self.nodes.append({"id": id_, "op": "Parameter", "inputs": [], "attrs": {"shape": list(shape)}})

    def const(self, id_, arr: np.ndarray):
        self.nodes.append({"id": id_, "op": "Constant", "inputs": [],
                           "data": {"shape": list(arr.shape), "values": [float(v) for v in arr.reshape(-1)]}})

    def op(self, id_, op, inputs, **attrs):
        n = {"id": id_, "op": op, "inputs": list(inputs)}
        if attrs:
            n["attrs"] = attrs
        self.nodes.append(n)

    def channel_bias(self, base, bias: np.ndarray, target, channel_axis: int) -> str:
        axes = [a for a in range(len(target)) if a != channel_axis]
        target = list(target)
        target[0] = -1
        self.const(base, bias)
        self.op(base + "_bcast", "Broadcast", [base], shape=target, axes=axes)
        return base + "_bcast"

    def json(self, outputs) -> dict:
        return {"format_version": 1, "name": self.name, "nodes": sorted(self.nodes, key=lambda n: n["id"]),
                "outputs": list(outputs)}


def gaussian_tensor(rng: Rng, shape, variance: float) -> np.ndarray:
    sd = math.sqrt(variance)
    return np.array([rng.gaussian() * sd for _ in range(int(np.prod(shape)))], dtype=np.float64).reshape(shape)


def uniform_tensor(rng: Rng, shape, lo: float, hi: float) -> np.ndarray:
    u = (rng.next_block(int(np.prod(shape))) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (lo + (hi - lo) * u).reshape(shape)


def sparse_pm1_tensor(rng: Rng, shape, variance: float) -> np.ndarray:
    """Config 5 weights: u<0.6 -> 0; u<0.7 -> +/-1 (sign next()&1); else N(0, variance)."""
    sd = math.sqrt(variance)
    out = np.empty(int(np.prod(shape)))
    for i in range(out.size):
        u = rng.uniform()
        if u < 0.6:
            out[i] = 0.0
        elif u < 0.7:
            out[i] = 1.0 if (rng.next() & 1) else -1.0
        else:
            out[i] = rng.gaussian() * sd
    return out.reshape(shape)


def pixel_tensor(rng: Rng, shape) -> np.ndarray:
    k = rng.next_block(int(np.prod(shape))) % np.uint64(256)
    return (k.astype(np.float64) / 255.0).reshape(shape)


# ---- BASELINE configurations ----

CONTEXTS = {
    "c1": {"n": 8192, "bits": [40, 30, 40], "scale_bits": 30, "security": 128},
    "c3": {"n": 8192, "bits": [36, 26, 26, 26, 26, 26, 36], "scale_bits": 26, "security": 128},
    "c4": {"n": 16384, "bits": [50] + [30] * 7 + [50], "scale_bits": 30, "security": 128},
    "c5": {"n": 16384, "bits": [50] + [30] * 5 + [50], "scale_bits": 30, "security": 128},
}


def config1(seed: int, batch: int):
    wr = Rng(seed).fork("config1")
    g = G("config1_dot")
    g.param("x", [1, 64])
    g.const("w", gaussian_tensor(wr.fork("w"), (64, 16), 0.25))
    g.op("dot", "Dot", ["x", "w"])
    b = g.channel_bias("b", gaussian_tensor(wr.fork("b"), (16,), 0.1), [1, 16], 1)
    g.op("out", "Add", ["dot", b])
    x = uniform_tensor(Rng(seed).fork("inputs").fork("x"), (batch, 64), -1.0, 1.0)
    return g.json(["out"]), x


def config3(seed: int, batch: int):
    wr = Rng(seed).fork("config3")
    g = G("config3_cryptonets")
    g.param("x", [1, 1, 28, 28])
    g.op("pad", "Pad", ["x"], pad_below=[0, 0, 0, 0], pad_above=[0, 0, 1, 1])
    g.const("w1", gaussian_tensor(wr.fork("w1"), (5, 1, 5, 5), 1.0 / 25))
    g.op("conv1", "Convolution", ["pad", "w1"], stride=2)
    g.op("act1", "PolyAct", ["conv1"], a=1.0, b=0.0, c=0.0)
    g.op("flat", "Reshape", ["act1"], shape=[-1, 845])
    g.const("w2", gaussian_tensor(wr.fork("w2"), (845, 100), 1.0 / 845))
    g.op("fc1", "Dot", ["flat", "w2"])
    g.op("act2", "PolyAct", ["fc1"], a=1.0, b=0.0, c=0.0)
    g.const("w3", gaussian_tensor(wr.fork("w3"), (100, 10), 1.0 / 100))
    g.op("logits", "Dot", ["act2", "w3"])
    x = pixel_tensor(Rng(seed).fork("inputs").fork("x"), (batch, 1, 28, 28))
    return g.json(["logits"]), x


def config4(seed: int, batch: int):
    wr = Rng(seed).fork("config4")
    g = G("config4_convnet")
    g.param("x", [1, 3, 32, 32])
    g.op("pad1", "Pad", ["x"], pad_below=[0, 0, 1, 1], pad_above=[0, 0, 1, 1])
    g.const("w1", gaussian_tensor(wr.fork("w1"), (16, 3, 3, 3), 1.0 / 27))
    g.op("conv1", "Convolution", ["pad1", "w1"], stride=1)
    g.op("act1", "PolyAct", ["conv1"], a=1.0, b=0.0, c=0.0)
    g.op("pool1", "AvgPool", ["act1"], window=[2, 2], stride=2)
    g.op("pad2", "Pad", ["pool1"], pad_below=[0, 0, 1, 1], pad_above=[0, 0, 1, 1])
    g.const("w2", gaussian_tensor(wr.fork("w2"), (32, 16, 3, 3), 1.0 / 144))
    g.op("conv2", "Convolution", ["pad2", "w2"], stride=1)
    g.op("act2", "PolyAct", ["conv2"], a=1.0, b=0.0, c=0.0)
    g.op("pool2", "AvgPool", ["act2"], window=[2, 2], stride=2)
    g.op("flat", "Reshape", ["pool2"], shape=[-1, 2048])
    g.const("w3", gaussian_tensor(wr.fork("w3"), (2048, 10), 1.0 / 2048))
    g.op("logits", "Dot", ["flat", "w3"])
    x = uniform_tensor(Rng(seed).fork("inputs").fork("x"), (batch, 3, 32, 32), 0.0, 1.0)
    return g.json(["logits"]), x


def config4_small(seed: int, batch: int):
    """Config 4's layer chain and context (N=16384, {50, 30x7, 50}, L=8: conv K=27 and K=144, x^2
    relinearisations at levels 7 and 4, AvgPool at 6 and 3, Dense at 2) on 3x8x8 images, so the
    reference finishes in about a minute on the host; same weights draw as config 4 with the
    Dense fan-in 32*2*2 = 128."""
    wr = Rng(seed).fork("config4")
    g = G("config4_convnet_8x8")
    g.param("x", [1, 3, 8, 8])
    g.op("pad1", "Pad", ["x"], pad_below=[0, 0, 1, 1], pad_above=[0, 0, 1, 1])
    g.const("w1", gaussian_tensor(wr.fork("w1"), (16, 3, 3, 3), 1.0 / 27))
    g.op("conv1", "Convolution", ["pad1", "w1"], stride=1)
    g.op("act1", "PolyAct", ["conv1"], a=1.0, b=0.0, c=0.0)
    g.op("pool1", "AvgPool", ["act1"], window=[2, 2], stride=2)
    g.op("pad2", "Pad", ["pool1"], pad_below=[0, 0, 1, 1], pad_above=[0, 0, 1, 1])
    g.const("w2", gaussian_tensor(wr.fork("w2"), (32, 16, 3, 3), 1.0 / 144))
    g.op("conv2", "Convolution", ["pad2", "w2"], stride=1)
    g.op("act2", "PolyAct", ["conv2"], a=1.0, b=0.0, c=0.0)
    g.op("pool2", "AvgPool", ["act2"], window=[2, 2], stride=2)
    g.op("flat", "Reshape", ["pool2"], shape=[-1, 128])
    g.const("w3", gaussian_tensor(wr.fork("w3"), (128, 10), 1.0 / 128))
    g.op("logits", "Dot", ["flat", "w3"])
    x = uniform_tensor(Rng(seed).fork("inputs").fork("x"), (batch, 3, 8, 8), 0.0, 1.0)
    return g.json(["logits"]), x


def config5(seed: int, batch: int):
    wr = Rng(seed).fork("config5")
    g = G("config5_mlp")
    g.param("x", [1, 784])
    g.const("w1", sparse_pm1_tensor(wr.fork("w1"), (784, 1024), 0.05))
    g.op("fc1", "Dot", ["x", "w1"])
    g.op("act1", "PolyAct", ["fc1"], a=1.0, b=0.0, c=0.0)
    g.const("w2", sparse_pm1_tensor(wr.fork("w2"), (1024, 1024), 0.05))
    g.op("fc2", "Dot", ["act1", "w2"])
    g.op("act2", "PolyAct", ["fc2"], a=1.0, b=0.0, c=0.0)
    g.const("w3", sparse_pm1_tensor(wr.fork("w3"), (1024, 10), 0.05))
    g.op("fc3", "Dot", ["act2", "w3"])
    x = uniform_tensor(Rng(seed).fork("inputs").fork("x"), (batch, 784), 0.0, 1.0)
    return g.json(["fc3"]), x


def mini(seed: int, batch: int):
    """Small graph covering every GPU node kernel (test-only; N=2048)."""
    wr = Rng(seed).fork("mini")
    g = G("mini_all_ops")
    g.param("x", [1, 2, 6, 6])
    g.op("pad", "Pad", ["x"], pad_below=[0, 0, 1, 0], pad_above=[0, 0, 0, 1])
    w1 = gaussian_tensor(wr.fork("w1"), (3, 2, 3, 3), 1.0 / 18)
    w1.reshape(-1)[[0, 5, 9]] = [0.0, 1.0, -1.0]  # bypass terms inside general sums
    g.const("w1", w1)
    g.op("conv", "Convolution", ["pad", "w1"], stride=1)
    bias = g.channel_bias("b1", gaussian_tensor(wr.fork("b1"), (3,), 0.1), [1, 3, 5, 5], 1)
    g.op("conv_b", "Add", ["conv", bias])
    g.op("act", "PolyAct", ["conv_b"], a=1.0, b=0.0, c=0.0)
    g.op("pool", "AvgPool", ["act"], window=[2, 2], stride=1)
    g.op("smp", "ScaledMeanPool", ["pool"], window=[2, 2], stride=2)
    g.op("neg", "Negate", ["smp"])
    g.op("flat", "Reshape", ["neg"], shape=[-1, 12])
    w2 = gaussian_tensor(wr.fork("w2"), (12, 4), 1.0 / 12)
    w2[0, :] = 0.0
    w2[1, 1] = 1.0
    g.const("w2", w2)
    g.op("fc", "Dot", ["flat", "w2"])
    g.const("k", np.array([0.5, -0.25, 2.0, 1.5]))
    g.op("kb", "Broadcast", ["k"], shape=[-1, 4], axes=[0])
    g.op("sub", "Subtract", ["fc", "kb"])
    g.const("m", np.array([0.75, -1.5, 0.125, 3.0]))
    g.op("mb", "Broadcast", ["m"], shape=[-1, 4], axes=[0])
    g.op("mul", "Multiply", ["sub", "mb"])
    x = uniform_tensor(Rng(seed).fork("inputs").fork("x"), (batch, 2, 6, 6), -1.0, 1.0)
    return g.json(["mul", "fc"]), x


def pmodel(seed: int, batch: int):
    """Paradigm coverage graph (test-only; N=2048): Conv + channel bias, x^2, Dot + bias.  Run under
    EncryptedModel (data in the clear, constants encrypted) and EncryptedBoth (both encrypted)."""
    wr = Rng(seed).fork("pmodel")
    g = G("paradigm_conv_dot")
    g.param("x", [1, 1, 5, 5])
    g.const("w1", gaussian_tensor(wr.fork("w1"), (2, 1, 3, 3), 1.0 / 9))
    g.op("conv", "Convolution", ["x", "w1"], stride=1)
    bias = g.channel_bias("b1", gaussian_tensor(wr.fork("b1"), (2,), 0.1), [1, 2, 3, 3], 1)
    g.op("conv_b", "Add", ["conv", bias])
    g.op("act", "PolyAct", ["conv_b"], a=1.0, b=0.0, c=0.0)
    g.op("flat", "Reshape", ["act"], shape=[-1, 18])
    g.const("w2", gaussian_tensor(wr.fork("w2"), (18, 3), 1.0 / 18))
    g.op("fc", "Dot", ["flat", "w2"])
    g.const("b2", gaussian_tensor(wr.fork("b2"), (3,), 0.1))
    g.op("b2b", "Broadcast", ["b2"], shape=[-1, 3], axes=[0])
    g.op("out", "Add", ["fc", "b2b"])
    x = uniform_tensor(Rng(seed).fork("inputs").fork("x"), (batch, 1, 5, 5), -1.0, 1.0)
    return g.json(["out"]), x


def ops2(seed: int, batch: int):
    """Second coverage graph (test-only; N=2048): BatchNormInference, Sum, Negate and a
    Concat that promotes a batch-column constant to fresh encryptions."""
    wr = Rng(seed).fork("ops2")
    g = G("ops2_bn_sum_concat")
    g.param("x", [1, 2, 4, 4])
    g.const("gamma", np.array([1.5, 0.75]))
    g.const("beta", np.array([0.25, 0.0]))
    g.const("mean", np.array([0.1, 0.0]))
    g.const("var", np.array([2.0, 0.5]))
    g.op("bn", "BatchNormInference", ["x", "gamma", "beta", "mean", "var"], epsilon=1e-5)
    g.op("sq", "PolyAct", ["bn"], a=1.0, b=0.0, c=0.0)
    g.op("s", "Sum", ["sq"], axes=[3])
    g.op("ns", "Negate", ["s"])
    g.const("k", gaussian_tensor(wr.fork("k"), (2, 3), 0.5))
    g.op("kb", "Broadcast", ["k"], shape=[-1, 2, 3], axes=[0])
    g.op("cat", "Concat", ["s", "ns", "kb"], axis=2)
    g.op("flat", "Reshape", ["cat"], shape=[-1, 22])
    g.const("w", gaussian_tensor(wr.fork("w"), (22, 3), 1.0 / 22))
    g.op("fc", "Dot", ["flat", "w"])
    x = uniform_tensor(Rng(seed).fork("inputs").fork("x"), (batch, 2, 4, 4), -1.0, 1.0)
    return g.json(["fc", "cat"]), x


def wide(seed: int, batch: int):
    """Prime-width coverage graph (test-only): a 96-term Dot (the tensor-core GEMM's K >= 64
    range), x^2 and a small Dot, run in contexts whose primes fall outside the GEMM's 4..7-byte,
    < 2^55 range (<= 24-bit and >= 55-bit primes: the IMAD GEMM and the 64-bit lane)."""
    wr = Rng(seed).fork("wide")
    g = G("wide_primes")
    g.param("x", [1, 96])
    g.const("w1", gaussian_tensor(wr.fork("w1"), (96, 8), 1.0 / 96))
    g.op("fc1", "Dot", ["x", "w1"])
    g.op("act", "PolyAct", ["fc1"], a=1.0, b=0.0, c=0.0)
    g.const("w2", gaussian_tensor(wr.fork("w2"), (8, 4), 1.0 / 8))
    g.op("fc2", "Dot", ["act", "w2"])
    x = uniform_tensor(Rng(seed).fork("inputs").fork("x"), (batch, 96), -1.0, 1.0)
    return g.json(["fc2", "fc1"]), x


def ops3(seed: int, batch: int):
    """Third coverage graph (test-only; N=2048): Reverse and Slice of ciphertexts; a weight built
    by constant folding through Convolution, AvgPool, BatchNormInference, Reverse, Concat, Sum,
    Add and Multiply (eval.hpp:127-265); a convolution whose weights hold exact 0 and +/-1 inside
    general sums; PolyAct with general coefficients; and a Dot without general terms (one column
    all-zero: the empty sum is a fresh zero; two pass-through-only columns), so it stays at the
    input level (runtime.hpp:553-568).  Run with optimized_addition on and off."""
    wr = Rng(seed).fork("ops3")
    g = G("ops3_rearrange_fold")
    g.param("x", [1, 2, 6, 6])
    g.op("rev", "Reverse", ["x"], axes=[3])
    g.op("sl", "Slice", ["rev"], begin=[0, 0, 1, 0], end=[batch, 2, 6, 5])
    g.const("c0", gaussian_tensor(wr.fork("c0"), (1, 2, 6, 6), 0.5))
    g.const("k", gaussian_tensor(wr.fork("k"), (2, 2, 3, 3), 0.1))
    g.op("cf", "Convolution", ["c0", "k"], stride=1)
    g.op("cp", "AvgPool", ["cf"], window=[2, 2], stride=2)
    g.const("gamma", np.array([1.25, 0.5]))
    g.const("beta", np.array([0.1, -0.2]))
    g.const("mean", np.array([0.05, 0.0]))
    g.const("var", np.array([1.5, 0.75]))
    g.op("bn", "BatchNormInference", ["cp", "gamma", "beta", "mean", "var"], epsilon=1e-5)
    g.op("bnr", "Reverse", ["bn"], axes=[1])
    g.op("cc", "Concat", ["bn", "bnr"], axis=0)
    g.const("s5", gaussian_tensor(wr.fork("s5"), (2, 2, 3, 2), 0.05))
    g.op("s4", "Sum", ["s5"], axes=[2])
    g.op("s1", "Reshape", ["s4"], shape=[2, 2, 2, 1])
    g.op("s1b", "Concat", ["s1", "s1"], axis=3)
    g.op("wa", "Add", ["cc", "s1b"])
    mask = np.ones((2, 2, 2, 2))
    pm = np.zeros((2, 2, 2, 2))
    for i, (pos, v) in enumerate([((0, 0, 0, 1), 0.0), ((0, 1, 1, 0), 1.0), ((1, 0, 1, 1), -1.0), ((1, 1, 0, 0), 0.0)]):
        mask[pos] = 0.0
        pm[pos] = v
    g.const("mask", mask)
    g.const("pm", pm)
    g.op("wm", "Multiply", ["wa", "mask"])
    g.op("w1", "Add", ["wm", "pm"])
    g.op("conv", "Convolution", ["sl", "w1"], stride=1)
    g.op("act", "PolyAct", ["conv"], a=0.5, b=-0.25, c=0.125)
    g.op("flat", "Reshape", ["act"], shape=[-1, 32])
    wd = np.zeros((32, 3))
    wd[3, 1], wd[17, 1], wd[30, 2] = 1.0, -1.0, 1.0
    g.const("wd", wd)
    g.op("fc", "Dot", ["flat", "wd"])
    x = uniform_tensor(Rng(seed).fork("inputs").fork("x"), (batch, 2, 6, 6), -1.0, 1.0)
    return g.json(["fc", "act"]), x


CONFIGS = {"c1": config1, "c3": config3, "c4": config4, "c4s": config4_small, "c5": config5}
MINI_CONTEXT = {"n": 2048, "bits": [45, 30, 30, 30, 30, 45], "scale_bits": 30, "security": 0}


def key_seed(seed: int) -> int:
    return Rng(seed).fork("keys").next()


def build(spec: dict):
    """spec: {"config": "c1"|"c3"|"c4"|"c5"|"mini", "batch": B, "seed": s} -> (graph, x, ctx params)."""
    cfg = spec["config"]
    if cfg in ("mini", "ops2", "ops3", "pmodel", "wide"):
        g, x = {"mini": mini, "ops2": ops2, "ops3": ops3, "pmodel": pmodel, "wide": wide}[cfg](spec["seed"],
                                                                                              spec["batch"])
        ctxp = dict(MINI_CONTEXT)
    else:
        g, x = CONFIGS[cfg](spec["seed"], spec["batch"])
        ctxp = dict(CONTEXTS["c4" if cfg == "c4s" else cfg])
    for k in ("bits", "scale_bits"):  # context overrides (prime-width coverage)
        if k in spec:
            ctxp[k] = spec[k]
    if "n" in spec:  # reduced ring for fast parity tests (same primes bit sizes)
        ctxp["n"] = spec["n"]
        ctxp["security"] = 0
    return g, x, ctxp


def _spec(config, batch, seed=1, **kw):
    d = {"config": config, "batch": batch, "seed": seed, "key_seed": key_seed(seed), "exec_seed": seed}
    d.update(kw)
    return d


GOLDEN_NETS = {
    "mini": _spec("mini", 16, seed=3),
    "ops2": _spec("ops2", 16, seed=4),
    "ops3": _spec("ops3", 16, seed=8),
    # the same graph with optimized_addition off: zero weights become fresh-zero terms
    "ops3_na": _spec("ops3", 16, seed=8, bypass={"optimized_addition": False}),
    # mini with both bypass shortcuts off: every term is a real product
    "mini_nb": _spec("mini", 16, seed=3, bypass={"optimized_addition": False, "optimized_multiply": False}),
    "pmodel_m": _spec("pmodel", 16, seed=5, paradigm="encrypted-model"),
    "pmodel_b": _spec("pmodel", 16, seed=5, paradigm="encrypted-both"),
    "mini_b": _spec("mini", 16, seed=3, paradigm="encrypted-both"),
    "c1": _spec("c1", 4096),
    "c3_n2048": _spec("c3", 64, n=2048),
    "c5_n2048": _spec("c5", 64, n=2048),
    "c4_n2048": _spec("c4", 32, n=2048),
    # config 4's full context and chain (N=16384, {50, 30x7, 50}) on 3x8x8 images
    "c4s": _spec("c4s", 8192),
    # primes outside the tensor-core GEMM's range: <= 24-bit and 56/60-bit limbs
    "wide_p20": _spec("wide", 16, seed=6, bits=[24, 20, 20, 24], scale_bits=20),
    "wide_p56": _spec("wide", 16, seed=6, bits=[56, 36, 36, 56]),
    "wide_p60": _spec("wide", 16, seed=6, bits=[60, 40, 40, 60]),
    "c3": _spec("c3", 4096),
    "c5": _spec("c5", 8192),
    # config 4 at full size (8192 images of 3x32x32): the reference run needs ~65 GB of RAM, so this
    # golden is produced on a GPU-box host (HG_GOLDEN_OUT=gpurun_out make_golden.py nets c4)
    "c4": _spec("c4", 8192),
}
