"""The NCCL transport of the output-sharded executor (hg_plan_set_comm) on one GPU:
a one-rank communicator runs the transport's own all-gather-v (grouped in-place broadcasts of
item ranges).  A one-GPU box cannot host two ranks, so this is the part of the NCCL path that
can execute here: the library loads, the communicator initialises, the grouped broadcasts are
well-formed and leave the buffer intact."""
import pytest

pytestmark = pytest.mark.gpu


def test_nccl_transport_one_rank_selftest(cuda_ok):
    import torch  # noqa: F401  (loads the process's libnccl, the one the transport dlopens)

    import paper_1810_10121_b200 as P

    ctx = P.Context(4096, [30, 30, 30], 30, security=0)
    for ranges, words in [(1, 2 * 3 * 4096), (7, 2 * 3 * 4096), (33, 512)]:
        P.call("hg_comm_selftest", ctx, ranges, words)
    assert len(P.comm_unique_id()) == 128
