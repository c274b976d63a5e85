"""Generate the committed golden fixtures from the REFERENCE itself.

Runs oracle/_ref/ref_harness (the unmodified hegraph headers compiled by
oracle/Makefile) and records SHA-256 digests (plus metadata) of every array it
dumps.  Run here, where /root/reference exists:

    python tests/golden/make_golden.py prims      # primitive goldens (seconds)
    python tests/golden/make_golden.py nets       # network goldens (minutes)

The outputs (tests/golden/*.json) are small and committed; the GPU box never
needs the reference.
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")
# where the fixtures are written (HG_GOLDEN_OUT lets a GPU-box host with more RAM produce a golden
# into gpurun_out/, e.g. the full config-4 net, whose reference run needs ~65 GB)
OUT = os.environ.get("HG_GOLDEN_OUT", HERE)

PRIM_CASES = {
    # name: (n, scale_bits, bits, key_seed)
    "n1024_30x3": (1024, 30, [30, 30, 30], 7),
    "n1024_36_26x2_36": (1024, 26, [36, 26, 26, 36], 11),
    "n2048_50_30_50": (2048, 30, [50, 30, 50], 13),
    "n8192_40_30_40": (8192, 30, [40, 30, 40], 5),
    "n4096_30x4": (4096, 30, [30, 30, 30, 30], 17),
    "n16384_50_30x2_50": (16384, 30, [50, 30, 30, 50], 19),
    # BASELINE config 2 (primitive sweep) shapes: 30-bit chains, L = 7 and L = 15, up to N = 2^15
    "n16384_30x8": (16384, 30, [30] * 8, 29),
    "n32768_30x16": (32768, 30, [30] * 16, 23),
    # the rest of config 2's (N, L) grid: L + 1 30-bit primes for N = 2^12 .. 2^15, L = 3 / 7 / 15
    "n4096_30x8": (4096, 30, [30] * 8, 37),
    "n4096_30x16": (4096, 30, [30] * 16, 41),
    "n8192_30x4": (8192, 30, [30] * 4, 43),
    "n8192_30x8": (8192, 30, [30] * 8, 47),
    "n8192_30x16": (8192, 30, [30] * 16, 53),
    "n16384_30x4": (16384, 30, [30] * 4, 59),
    "n16384_30x16": (16384, 30, [30] * 16, 61),
    "n32768_30x4": (32768, 30, [30] * 4, 67),
    "n32768_30x8": (32768, 30, [30] * 8, 71),
    # BASELINE config 4's context: N = 2^14, {50, 30x7, 50} (L = 8, D = 4 digits for the 50-bit limbs)
    "n16384_50_30x7_50": (16384, 30, [50] + [30] * 7 + [50], 31),
}


def load_dump(d: str) -> dict:
    with open(os.path.join(d, "index.json")) as f:
        idx = json.load(f)
    blob = np.fromfile(os.path.join(d, "blob.bin"), dtype=np.uint8)
    out = {}
    for k, v in idx.items():
        if isinstance(v, dict) and "offset" in v and "dtype" in v:
            dt = np.uint64 if v["dtype"] == "u64" else np.float64
            raw = blob[v["offset"]: v["offset"] + 8 * v["count"]]
            out[k] = raw.view(dt).copy()
        else:
            out[k] = v
    return out


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_prims(only=None):
    for name, (n, sb, bits, key_seed) in PRIM_CASES.items():
        if only and name not in only:
            continue
        with tempfile.TemporaryDirectory() as d:
            subprocess.check_call([HARNESS, "prims", d, str(n), str(sb), ",".join(map(str, bits)), str(key_seed)])
            dump = load_dump(d)
        g = {"n": n, "scale_bits": sb, "bits": bits, "key_seed": key_seed, "arrays": {}, "meta": {}}
        for k, v in dump.items():
            if isinstance(v, np.ndarray):
                g["arrays"][k] = {"sha256": sha(v), "count": int(v.size),
                                  "dtype": "u64" if v.dtype == np.uint64 else "f64"}
                if v.size <= 64:
                    g["arrays"][k]["values"] = [int(x) for x in v] if v.dtype == np.uint64 else [float(x) for x in v]
            else:
                g["meta"][k] = v
        # a few leading words of the big arrays help debugging without bloating the repo
        for k in ("ct1", "mul_relin_rescale", "weighted_sum", "ntt_fwd_0"):
            g["arrays"][k]["head"] = [int(x) for x in dump[k][:8]]
        for k in ("dec_ct1", "dec_mul_relin_rescale"):
            g["arrays"][k]["head"] = [float(x) for x in dump[k][:16]]
        with open(os.path.join(OUT, f"prims_{name}.json"), "w") as f:
            json.dump(g, f, indent=1)
        print("wrote", name)


def make_nets(which=None):
    from paper_1810_10121_b200 import graphs  # product-side builders (pure Python, no GPU)

    for name, spec in graphs.GOLDEN_NETS.items():
        if which and name not in which:
            continue
        g, x, ctxp = graphs.build(spec)
        with tempfile.TemporaryDirectory() as d:
            gp = os.path.join(d, "graph.json")
            xp = os.path.join(d, "x.f64")
            with open(gp, "w") as f:
                json.dump(g, f)
            x.astype(np.float64).tofile(xp)
            pre = os.path.join(d, "out")
            subprocess.check_call([HARNESS, "net", gp, xp, str(spec["batch"]), str(ctxp["n"]), str(ctxp["scale_bits"]),
                                   ",".join(map(str, ctxp["bits"])), str(ctxp["security"]), str(spec["key_seed"]),
                                   str(spec["exec_seed"]), str(spec.get("threads", os.cpu_count())), pre] +
                                  ([f"--paradigm={spec['paradigm']}"] if "paradigm" in spec else []) +
                                  (["--no-opt-add"] if not spec.get("bypass", {}).get("optimized_addition", True)
                                   else []) +
                                  (["--no-opt-mult"] if not spec.get("bypass", {}).get("optimized_multiply", True)
                                   else []))
            with open(pre + ".json") as f:
                res = json.load(f)
            cts = np.fromfile(pre + ".ct.bin", dtype=np.uint64)
            outs = {}
            off = 0
            for o in res["outputs"]:
                vals = np.fromfile(pre + "." + o["id"] + ".f64", dtype=np.float64)
                digs = []
                for e in o["elements"]:
                    words = e["size"] * (e["level"] + 1) * ctxp["n"]
                    digs.append(sha(cts[off: off + words]))
                    off += words
                outs[o["id"]] = {"shape": o["shape"], "elements": o["elements"], "ct_sha256": digs,
                                 "values_sha256": sha(vals), "values_head": [float(v) for v in vals[:64]],
                                 "values_absmax": float(np.abs(vals).max())}
                np.save(os.path.join(OUT, f"net_{name}_{o['id']}_values.npy"), vals[: min(vals.size, 64 * 16)])
            golden = {"spec": spec, "ctx": ctxp, "profile": res["profile"], "outputs": outs,
                      "ref_execute_ms": res["execute_ms"], "threads": res["threads"]}
            with open(os.path.join(OUT, f"net_{name}.json"), "w") as f:
                json.dump(golden, f, indent=1)
            print("wrote net", name, "execute_ms", res["execute_ms"])


# The reference's own HEGK / HEGC files (keyio.hpp) for the GPU key/ciphertext I/O tests:
# N=1024, primes {30, 30}, keys seed 7, one encryption (seed 11) of 512 seeded slot values,
# plus the reference's decrypt of it.
IO_CASE = {"dir": "io_n1024", "n": 1024, "scale_bits": 30, "bits": [30, 30], "key_seed": 7, "enc_seed": 11}


def make_io():
    d = os.path.join(HERE, IO_CASE["dir"])
    os.makedirs(d, exist_ok=True)
    subprocess.check_call([HARNESS, "io", d, str(IO_CASE["n"]), str(IO_CASE["scale_bits"]),
                           ",".join(map(str, IO_CASE["bits"])), str(IO_CASE["key_seed"]), str(IO_CASE["enc_seed"])])
    with open(os.path.join(d, "case.json"), "w") as f:
        json.dump(IO_CASE, f, indent=1)
    print("wrote", d)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "prims"
    if what == "prims":
        make_prims(sys.argv[2:] or None)
    elif what == "nets":
        make_nets(sys.argv[2:] or None)
    elif what == "io":
        make_io()
