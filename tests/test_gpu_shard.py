"""Output-sharded execution checked on one GPU: W plans of the
same graph run as an in-process shard group (hg_group_run) -- every Dot/Conv
computes only its rank's block, x^2 runs on the shard, tensors are gathered
where a consumer needs all elements.  Every rank's outputs must equal the
reference's bit for bit (the same golden fixtures as test_gpu_exec), with the
reference's ExecProfile counts."""
import os

import numpy as np
import pytest

from tests import golden_util as G

pytestmark = pytest.mark.gpu

CASES = [("mini", 2), ("ops2", 2), ("ops3", 2), ("ops3_na", 3), ("c1", 2), ("c1", 3), ("c3_n2048", 2), ("c3_n2048", 4),
         ("c5_n2048", 3), ("c4_n2048", 4), ("c4s", 4), ("c3", 8),
         # encrypted-weight contractions (EncryptedModel / EncryptedBoth) sharded by outputs
         ("pmodel_m", 2), ("pmodel_b", 2), ("pmodel_b", 3), ("mini_b", 2)]


def _available(name):
    return os.path.exists(os.path.join(G.GOLDEN, f"net_{name}.json"))


@pytest.mark.parametrize("name,world", [c for c in CASES if _available(c[0])])
def test_shard_group_bit_exact(name, world, cuda_ok):
    import torch

    import paper_1810_10121_b200 as P
    from paper_1810_10121_b200 import graphs

    gold = G.load_net(name)
    spec = gold["spec"]
    graph, x, ctxp = graphs.build(spec)
    ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
    keys = P.Keys(ctx, spec["key_seed"])
    plans = [P.Plan(ctx, keys, graph, spec["batch"], spec["exec_seed"]) for _ in range(world)]
    for p in plans:
        if "paradigm" in spec or "bypass" in spec:
            p.set_options(paradigm=spec.get("paradigm"), bypass=spec.get("bypass"))
        p.bind_input("x", x)
    for _ in range(2):  # the second run reuses the per-rank node caches
        P.group_run(plans)
    ref = gold["profile"]
    for r, plan in enumerate(plans):
        prof = plan.profile()
        assert prof["bypass"] == ref["bypass"] and prof["ct_ops"] == ref["ct_ops"], (r, prof)
        assert prof["peak_elements"] == ref["peak_elements"]
        for oid, want in gold["outputs"].items():
            elems, level, _ = plan.output_info(oid)
            words = plan.output_ciphertexts(oid)
            d = torch.from_numpy(words.view(np.int64)).cuda()
            P.ntt(ctx, d, elems * 2 * (level + 1), level + 1, inverse=True)
            coeff = d.cpu().numpy().view(np.uint64).reshape(elems, -1)
            bad = [e for e in range(elems) if G.sha(coeff[e]) != want["ct_sha256"][e]]
            assert not bad, f"{name} world {world} rank {r}/{oid}: ciphertexts {bad[:8]} differ"
            assert G.sha(plan.output(oid)) == want["values_sha256"]
    for p in plans:
        p.close()


def test_single_rank_comm_is_unsharded(cuda_ok):
    """hg_plan_set_comm with world 1 (a real NCCL id is not needed) keeps the plain path."""
    import paper_1810_10121_b200 as P
    from paper_1810_10121_b200 import graphs

    gold = G.load_net("c1")
    spec = gold["spec"]
    graph, x, ctxp = graphs.build(spec)
    ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
    keys = P.Keys(ctx, spec["key_seed"])
    plan = P.Plan(ctx, keys, graph, spec["batch"], spec["exec_seed"])
    plan.set_comm(0, 1)
    plan.bind_input("x", x)
    plan.run()
    for oid, want in gold["outputs"].items():
        assert G.sha(plan.output(oid)) == want["values_sha256"]
    plan.close()
