"""Clear-value (fp64) model of the executor's output sharding, for CPU tests.

Mirrors hg_exec.cpp's multi-rank rules on plain numbers instead of ciphertexts:
  * Dot / Convolution compute only this rank's block of outputs, chosen by the
    executor's own partition rule (hg_shard_partition through the C-ABI);
  * x^2 (PolyAct a=1,b=0,c=0) and Reshape keep the shard;
  * every other consumer, and every graph output, first all-gathers the tensor:
    each rank broadcasts its own element ranges in place (what the NCCL
    transport does with grouped ncclBroadcast calls).
A tensor is an array [elements][batch]; elements a rank does not own are NaN
until gathered, so a missing exchange cannot go unnoticed."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10121_b200 as P  # noqa: E402


def coalesce(els):
    out = []
    for e in sorted(els):
        if out and out[-1][1] == e:
            out[-1][1] += 1
        else:
            out.append([e, e + 1])
    return [tuple(r) for r in out]


def contraction_layout(groups, mg, world, out_index):
    """Per rank: its partition block and its coalesced output-element ranges."""
    blocks, ranges = [], []
    for r in range(world):
        g0, g1, m0, m1 = P.shard_partition(groups, mg, world, r)
        blocks.append((g0, g1, m0, m1))
        ranges.append(coalesce([out_index(g, m) for g in range(g0, g1) for m in range(m0, m1)]))
    return blocks, ranges


class ShardedEval:
    def __init__(self, graph, batch, rank, world, gather):
        """gather(array, ranges_by_rank) -> array with every element filled (collective)."""
        self.nodes = {n["id"]: n for n in graph["nodes"]}
        self.outputs = graph["outputs"]
        self.batch, self.rank, self.world, self.gather_fn = batch, rank, world, gather
        self.gathers = 0

    def _order(self):
        seen, order = set(), []

        def visit(i):
            if i in seen:
                return
            seen.add(i)
            for j in self.nodes[i].get("inputs", []):
                visit(j)
            order.append(i)

        for i in sorted(self.nodes):
            visit(i)
        return order

    def _full(self, v):
        if v["ranges"] is not None and self.world > 1:
            v["data"] = self.gather_fn(v["data"], v["ranges"])
            self.gathers += 1
        v["ranges"] = None
        return v

    def run(self, x):
        vals = {}
        for i in self._order():
            n = self.nodes[i]
            op = n["op"]
            a = n.get("attrs", {})
            if op == "Parameter":
                vals[i] = {"data": x.reshape(self.batch, -1).T.copy(), "shape": list(x.shape[1:]), "ranges": None}
                continue
            if op == "Constant":
                vals[i] = {"const": np.array(n["data"]["values"]).reshape(n["data"]["shape"])}
                continue
            ins = [vals[j] for j in n["inputs"]]
            keeps = op == "Reshape" or (op == "PolyAct" and a.get("a") == 1.0 and a.get("b") == 0.0
                                         and a.get("c") == 0.0)
            if not keeps:
                ins = [self._full(v) if "data" in v else v for v in ins]
            vals[i] = getattr(self, "_" + op)(n, ins)
        return {o: self._full(vals[o])["data"] for o in self.outputs}

    # ---- ops ----
    def _Reshape(self, n, ins):
        shape = n["attrs"]["shape"][1:]
        return {"data": ins[0]["data"], "shape": list(shape), "ranges": ins[0]["ranges"]}

    def _PolyAct(self, n, ins):
        d = ins[0]["data"]
        return {"data": d * d, "shape": ins[0]["shape"], "ranges": ins[0]["ranges"]}

    def _Pad(self, n, ins):
        lo, hi = n["attrs"]["pad_below"][1:], n["attrs"]["pad_above"][1:]
        shp = ins[0]["shape"]
        d = ins[0]["data"].reshape(shp + [self.batch])
        d = np.pad(d, [(l, h) for l, h in zip(lo, hi)] + [(0, 0)])
        return {"data": d.reshape(-1, self.batch), "shape": list(d.shape[:-1]), "ranges": None}

    def _contract(self, groups, mg, kt, out_index, x_index, w_index, xd, w, out_shape):
        blocks, ranges = contraction_layout(groups, mg, self.world, out_index)
        out = np.full((groups * mg, self.batch), np.nan)
        g0, g1, m0, m1 = blocks[self.rank]
        wf = w.reshape(-1)
        for g in range(g0, g1):
            for m in range(m0, m1):
                acc = np.zeros(self.batch)
                for t in range(kt):
                    acc = acc + wf[w_index(g, m, t)] * xd[x_index(g, t)]
                out[out_index(g, m)] = acc
        return {"data": out, "shape": out_shape, "ranges": ranges if self.world > 1 else None}

    def _Dot(self, n, ins):
        x, w = ins[0], ins[1]["const"]
        k, md = w.shape
        rows = int(np.prod(x["shape"])) // k
        return self._contract(rows, md, k, lambda g, m: g * md + m, lambda g, t: g * k + t,
                              lambda g, m, t: t * md + m, x["data"], w, [md])

    def _Convolution(self, n, ins):
        x, w = ins[0], ins[1]["const"]
        s = n["attrs"]["stride"]
        C, H, W = x["shape"][-3:]
        F, _, kh, kw = w.shape
        OH, OW = (H - kh) // s + 1, (W - kw) // s + 1
        kt = C * kh * kw

        def oi(g, f):
            return (f * OH + g // OW) * OW + g % OW

        def xi(g, t):
            oy, ox = g // OW, g % OW
            dx, dy, c = t % kw, (t // kw) % kh, t // (kw * kh)
            return (c * H + oy * s + dy) * W + ox * s + dx

        return self._contract(OH * OW, F, kt, oi, xi, lambda g, f, t: f * kt + t, x["data"], w, [F, OH, OW])


# ---- world_size-N worker over torch.distributed (gloo on CPU) ----

def small_mlp(seed=5):
    """c5-shaped MLP at toy size: sparse +-1 / zero / Gaussian weights, x^2 between."""
    from paper_1810_10121_b200 import graphs

    wr = graphs.Rng(seed).fork("mlp")
    g = graphs.G("mlp_toy")
    g.param("x", [1, 24])
    g.const("w1", graphs.sparse_pm1_tensor(wr.fork("w1"), (24, 17), 0.05))
    g.op("fc1", "Dot", ["x", "w1"])
    g.op("act1", "PolyAct", ["fc1"], a=1.0, b=0.0, c=0.0)
    g.const("w2", graphs.sparse_pm1_tensor(wr.fork("w2"), (17, 9), 0.05))
    g.op("fc2", "Dot", ["act1", "w2"])
    return g.json(["fc2"])


def _graph(name, batch):
    from paper_1810_10121_b200 import graphs

    if name == "mlp":
        g = small_mlp()
        x = graphs.uniform_tensor(graphs.Rng(9).fork("x"), (batch, 24), 0.0, 1.0)
        return g, x
    return graphs.CONFIGS[name](3, batch)


def main():
    import argparse
    import json

    import torch
    import torch.distributed as dist

    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int)
    ap.add_argument("--world", type=int)
    ap.add_argument("--port", type=int)
    ap.add_argument("--graph", default="c3")
    ap.add_argument("--batch", type=int, default=2)
    a = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{a.port}", rank=a.rank, world_size=a.world)

    def gather(arr, ranges):
        t = torch.from_numpy(arr)
        for r, rr in enumerate(ranges):
            for b, e in rr:
                dist.broadcast(t[b:e], src=r)  # in place, like the NCCL transport's grouped broadcasts
        return arr

    g, x = _graph(a.graph, a.batch)
    sharded = ShardedEval(g, a.batch, a.rank, a.world, gather)
    got = sharded.run(x)
    want = ShardedEval(g, a.batch, 0, 1, None).run(x)
    ok = all(np.array_equal(got[o], want[o]) and not np.isnan(got[o]).any() for o in want)
    print(json.dumps({"rank": a.rank, "ok": bool(ok), "gathers": sharded.gathers}), flush=True)
    dist.destroy_process_group()
    raise SystemExit(0 if ok else 1)


if __name__ == "__main__":
    main()
