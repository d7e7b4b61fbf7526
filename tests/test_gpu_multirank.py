"""Bit-identity across world sizes (north_star: "bit-identical at 1, 2, 4 and 8
GPUs") exercised on ONE GPU: G processes share cuda:0 and talk over gloo
(NCCL refuses two ranks on one device).  The product code path is the same as
with NCCL except the collective transport; the step root (which commits every
operator output of every shard, the combined gradient and the AdamW update)
must equal the single-process root for every G."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tiny, q, combine="sliced"):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2502_19405_b200.gpt2 import GPT2Config, GPT2Step
        cfg = GPT2Config.tiny() if tiny else GPT2Config()
        st = GPT2Step(cfg, rank=rank, world=world, combine=combine, p2p_sync="host")
        st.set_tokens(0)
        st.run()
        root, _ = st.step_root()
        loss = st.loss()
        # the updated parameters themselves must be identical on every rank
        pdig = st.digests_host.numpy()[st.tensors[st.adam_out["wte"][0]].slot].tobytes()
        q.put((rank, root.hex(), loss, pdig.hex()))
    except Exception:  # report instead of leaving the parent waiting on the queue
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc(), None, None))
        raise
    finally:
        dist.destroy_process_group()


def _run(world, tiny, combine="sliced"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, tiny, q, combine)) for r in range(world)]
    for p in ps:
        p.start()
    res = []
    for _ in ps:
        r = q.get(timeout=900)
        assert not str(r[1]).startswith("ERROR"), f"rank {r[0]} failed:\n{r[1]}"
        res.append(r)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(res)


@pytest.fixture(scope="module")
def tiny_single():
    return _run(1, True)[0]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_tiny_step_root_identical_across_world_sizes(world, tiny_single):
    for rank, root, loss, pdig in _run(world, True):
        assert root == tiny_single[1], f"world {world} rank {rank}: step root differs"
        assert loss == tiny_single[2]
        assert pdig == tiny_single[3]


@pytest.fixture(scope="module")
def full_single():
    return _run(1, False)[0]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_full_gpt2_step_root_equals_world1(world, full_single):
    """the full GPT-2 124M step (every operator output committed) gives the G = 1 root
    with its 8 shards spread over 2, 4 and 8 rank processes"""
    for rank, root, loss, pdig in _run(world, False):
        assert root == full_single[1], f"rank {rank}: full GPT-2 step root differs between G=1 and G={world}"
        assert pdig == full_single[3]


@pytest.mark.parametrize("world", [2, 4])
def test_tiny_step_root_p2p_combine(world, tiny_single):
    """R-TREE_S through the fused peer-memory kernel (CUDA IPC between the rank
    processes, P2P loads / stores) gives the single-process root."""
    for rank, root, loss, pdig in _run(world, True, combine="p2p"):
        assert root == tiny_single[1], f"p2p world {world} rank {rank}: step root differs"
        assert pdig == tiny_single[3]
