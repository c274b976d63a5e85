"""BASELINE config 2: ciphertext primitive sweep on one B200.

N in {4096, 8192, 16384, 32768}; L in {3, 7, 15} 30-bit NTT-friendly primes
plus one 30-bit special prime (coeff_mod_bits = [30] * (L + 1)),
batches of 1 .. 16384 ciphertexts (capped by a memory budget).  Ops, each
through the C-ABI (include/hegpu.h) on device-resident operands:

  ntt_fwd / ntt_inv       all 2(L+1) limb rows of every ciphertext
  add                     ct + ct                          (CkksBackend::add)
  mul_plain               ct x full plaintext              (multiply_plain)
  mul_plain_rescale       ... + rescale                    (multiply_plain_rescale)
  mul_const_rescale       ct x encode_constant weight + rescale (weighted_sum, one term)
  mul_relin               ct x ct + relinearise            (multiply)
  mul_relin_rescale       ct x ct + relinearise + rescale  (multiply_rescale)
  square_relin_rescale    fused x^2 (PolyAct)              (multiply_rescale(x, x))

Reported per (N, L, op, B): ops/s, achieved algorithmic GB/s and modmul/s, and
their fractions of the measured HBM copy bandwidth (MEASURED_PEAKS.json) and of
the register-only 32-bit Shoup modmul peak measured live on this GPU.  The
algorithmic counts are SURVEY §8(d)'s.  Timing: CUDA events on the launching
stream, after warm-up, median of 3 repeats.  Operands smaller than the 126 MB
L2 stay cache-resident between repeats (marked "l2_resident").

Usage:  python tools/prim_sweep.py [--quick] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 2**20


def main():
    import torch

    import paper_1810_10121_b200 as P

    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="a few points only")
    ap.add_argument("--out", default=None)
    ap.add_argument("--budget-gb", type=float, default=48.0, help="device bytes for operands per point")
    ap.add_argument("--ns", default="4096,8192,16384,32768")
    ap.add_argument("--ls", default="3,7,15")
    args = ap.parse_args()

    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        with open(pk) as f:
            peaks = json.load(f)
    hbm = float(peaks.get("hbm_gbs", 6552.6))
    out = open(args.out, "w") if args.out else None

    def emit(rec):
        s = json.dumps(rec)
        print(s, flush=True)
        if out:
            out.write(s + "\n")
            out.flush()

    ns = [int(v) for v in args.ns.split(",")]
    ls = [int(v) for v in args.ls.split(",")]
    batches = [1, 4, 16, 64, 256, 1024, 4096, 16384]
    if args.quick:
        ns, ls, batches = [8192, 32768], [3, 15], [16, 256]
    stream = torch.cuda.current_stream()
    peak32 = None

    for n in ns:
        for L in ls:
            bits = [30] * (L + 1)
            ctx = P.Context(n, bits, 30, security=0)
            keys = P.Keys(ctx, 1)
            if peak32 is None:
                peak32 = ctx.modmul_peak(False)
                emit({"kind": "peaks", "hbm_gbs": hbm, "modmul32_per_s": peak32,
                      "modmul64_per_s": ctx.modmul_peak(True), "gpu": torch.cuda.get_device_name()})
            nl, logn = L + 1, int(math.log2(n))
            W = nl * n  # words per poly
            ct_bytes = 2 * W * 8
            ntt_mm = (n // 2) * logn
            rows = ctx.relin_rows  # sum_i D_i over all nl limbs
            resc_mm = lambda polys: polys * (nl * ntt_mm + (nl - 1) * n)  # noqa: E731  INTT top + (nl-1) NTT + mul
            # worst case per item: a, b, out3, out2 ≈ 9 polys + relin scratch (c2, 2 accum) ≈ 12 polys
            bmax = int(args.budget_gb * 1e9 // (6 * ct_bytes))
            for B in [b for b in batches if b <= bmax]:
                g = torch.Generator(device="cuda").manual_seed(B)
                # uniform residues in [0, q) per limb (the op's cost does not depend on the values)
                q = torch.tensor([int(v) for v in ctx.primes], dtype=torch.int64, device="cuda")

                def rand_ct(items, polys=2):
                    r = torch.randint(0, 2**62, (items, polys, nl, n), generator=g, device="cuda",
                                      dtype=torch.int64)
                    return (r % q.view(1, 1, nl, 1)).reshape(-1).contiguous()

                a, b = rand_ct(B), rand_ct(B)
                pt = rand_ct(1, 1)
                o2 = torch.empty(B * 2 * W, dtype=torch.int64, device="cuda")
                o2b = torch.empty(B * 2 * W, dtype=torch.int64, device="cuda")
                r2 = torch.empty(B * 2 * (nl - 1) * n, dtype=torch.int64, device="cuda")
                w1 = torch.tensor([int(v) for v in ctx.primes], dtype=torch.int64, device="cuda")
                w1 = (torch.full((B, nl), 12345, dtype=torch.int64, device="cuda") % w1).reshape(-1).contiguous()
                idx = torch.arange(B, dtype=torch.int32, device="cuda")
                keybytes = rows * 2 * W * 8
                ops = {
                    "ntt_fwd": (lambda: P.ntt(ctx, a, B * 2 * nl, nl), B * 2 * nl,
                                2 * B * 2 * W * 8, B * 2 * nl * ntt_mm),
                    "ntt_inv": (lambda: P.ntt(ctx, a, B * 2 * nl, nl, inverse=True), B * 2 * nl,
                                2 * B * 2 * W * 8, B * 2 * nl * ntt_mm),
                    "add": (lambda: P.call("hg_add", ctx, a, b, o2, B * 2 * W, nl), B,
                            3 * B * ct_bytes, 0),
                    "mul_plain": (lambda: P.call("hg_multiply_plain", ctx, a, pt, o2, B, 2, nl, 0), B,
                                  2 * B * ct_bytes + W * 8, B * 2 * W),
                    "mul_plain_rescale": (lambda: (P.call("hg_multiply_plain", ctx, a, pt, o2, B, 2, nl, 0),
                                                   P.call("hg_rescale", ctx, o2, r2, B * 2, nl)), B,
                                          2 * B * ct_bytes + W * 8 + B * ct_bytes * (nl - 1) // nl,
                                          B * 2 * W + resc_mm(2 * B)),
                    "mul_const_rescale": (lambda: P.call("hg_weighted_sum", ctx, a, idx, w1, r2, B, 1, 1, nl), B,
                                          B * ct_bytes + B * ct_bytes * (nl - 1) // nl,
                                          B * 2 * W + resc_mm(2 * B)),
                    "mul_relin": (lambda: P.call("hg_multiply_relin", ctx, keys, a, b, o2, B, nl), B,
                                  3 * B * ct_bytes + keybytes,
                                  B * (4 * W + nl * ntt_mm + rows * nl * ntt_mm + 2 * rows * W)),
                    "mul_relin_rescale": (lambda: (P.call("hg_multiply_relin", ctx, keys, a, b, o2, B, nl),
                                                   P.call("hg_rescale", ctx, o2, r2, B * 2, nl)), B,
                                          2 * B * ct_bytes + B * ct_bytes * (nl - 1) // nl + keybytes,
                                          B * (4 * W + nl * ntt_mm + rows * nl * ntt_mm + 2 * rows * W)
                                          + resc_mm(2 * B)),
                    "square_relin_rescale": (lambda: P.call("hg_square_relin_rescale", ctx, keys, a, r2, B, nl), B,
                                             B * ct_bytes + B * ct_bytes * (nl - 1) // nl + keybytes,
                                             B * (3 * W + nl * ntt_mm + rows * nl * ntt_mm + 2 * rows * W)
                                             + resc_mm(2 * B)),
                }
                for name, (fn, units, abytes, amm) in ops.items():
                    try:
                        fn()
                        torch.cuda.synchronize()
                    except P.HEError as e:
                        emit({"kind": "error", "n": n, "L": L, "op": name, "batch": B, "error": str(e)})
                        continue
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    one = e0.elapsed_time(e1)
                    reps = max(1, min(200, int(20.0 / max(one, 1e-3))))
                    ts = []
                    for _ in range(3):
                        e0.record(stream)
                        for _ in range(reps):
                            fn()
                        e1.record(stream)
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1) / reps)
                    ms = statistics.median(ts)
                    sec = ms / 1e3
                    gbs = abytes / sec / 1e9
                    mms = amm / sec
                    emit({"kind": "point", "n": n, "L": L, "op": name, "batch": B, "ms": ms,
                          "ops_per_s": (units / sec), "unit": "limb NTTs/s" if name.startswith("ntt") else "ct ops/s",
                          "alg_gbs": gbs, "hbm_frac": gbs / hbm, "alg_gmodmul_s": mms / 1e9,
                          "modmul_frac": (mms / peak32) if amm else 0.0,
                          "roofline_frac": max(gbs / hbm, (mms / peak32) if amm else 0.0),
                          "l2_resident": 3 * B * ct_bytes < L2_BYTES})
                del a, b, o2, o2b, r2, pt
                torch.cuda.empty_cache()
            keys.close()
            ctx.close()
    if out:
        out.close()


if __name__ == "__main__":
    main()
