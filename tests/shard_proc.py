"""One rank of a multi-process sharded graph run (tests/test_gpu_shard_procs.py): the C++
executor computes this rank's Dot/Conv blocks and calls back at every gather point; the
callback exchanges the ranks' item ranges over torch.distributed (gloo, host memory) -- the
real sharded executor across processes, with a host collective standing in for NCCL where one
GPU per rank is not available.  Prints one JSON line per rank with the output digests.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port P \\
        tests/shard_proc.py <golden net name>
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from tests import golden_util as G  # noqa: E402

_rt = ctypes.CDLL("libcudart.so.12")
_rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]


def _copy(dst, src, nbytes, kind):  # 1 = H2D, 2 = D2H
    rc = _rt.cudaMemcpy(ctypes.c_void_p(dst), ctypes.c_void_p(src), ctypes.c_size_t(nbytes), kind)
    assert rc == 0, f"cudaMemcpy failed ({rc})"


def main():
    import paper_1810_10121_b200 as P
    from paper_1810_10121_b200 import graphs

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    name = sys.argv[1]
    gold = G.load_net(name)
    spec = gold["spec"]
    graph, x, ctxp = graphs.build(spec)
    ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
    keys = P.Keys(ctx, spec["key_seed"])
    plan = P.Plan(ctx, keys, graph, spec["batch"], spec["exec_seed"])
    if "paradigm" in spec or "bypass" in spec:
        plan.set_options(paradigm=spec.get("paradigm"), bypass=spec.get("bypass"))
    gathers = []

    def gather(tid, dev, item_words, ranges):
        ib = item_words * 8
        mine = ranges[rank]
        own = b"".join(_d2h(dev + b * ib, (e - b) * ib) for b, e in mine)
        parts = [None] * world
        dist.all_gather_object(parts, own)
        for r in range(world):
            if r == rank:
                continue
            off = 0
            blob = parts[r]
            for b, e in ranges[r]:
                n = (e - b) * ib
                buf = np.frombuffer(blob, dtype=np.uint8, count=n, offset=off)
                _copy(dev + b * ib, buf.ctypes.data, n, 1)
                off += n
        gathers.append(tid)

    def _d2h(ptr, n):
        buf = np.empty(n, dtype=np.uint8)
        _copy(buf.ctypes.data, ptr, n, 2)
        return buf.tobytes()

    plan.set_gather(rank, world, gather)
    plan.bind_input("x", x)
    plan.run()
    res = {"rank": rank, "world": world, "gathers": gathers, "outputs": {}}
    prof = plan.profile()
    res["counts_equal"] = (prof["bypass"] == gold["profile"]["bypass"] and prof["ct_ops"] == gold["profile"]["ct_ops"])
    for oid, want in gold["outputs"].items():
        elems, level, _ = plan.output_info(oid)
        words = plan.output_ciphertexts(oid)
        d = torch.from_numpy(words.view(np.int64)).cuda()
        P.ntt(ctx, d, elems * 2 * (level + 1), level + 1, inverse=True)
        coeff = d.cpu().numpy().view(np.uint64).reshape(elems, -1)
        bad = [e for e in range(elems) if G.sha(coeff[e]) != want["ct_sha256"][e]]
        res["outputs"][oid] = {"bad": bad, "values_equal": G.sha(plan.output(oid)) == want["values_sha256"]}
    plan.close()
    print("RESULT " + json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
