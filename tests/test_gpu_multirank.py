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


def _worker(rank, world, port, tiny, q, combine="sliced", sync="host", bucketed=True, zero1=False, steps=1,
            fail_rank=None):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2502_19405_b200.gpt2 import GPT2Config, GPT2Step
        if rank == fail_rank:   # a rank whose peer-memory mapping fails
            import paper_2502_19405_b200 as R

            def _fail(*a, **k):
                raise RuntimeError("injected IPC open failure")
            R.repops_ipc_open = _fail
        cfg = GPT2Config.tiny() if tiny else GPT2Config()
        st = GPT2Step(cfg, rank=rank, world=world, combine=combine, p2p_sync=sync, zero1=zero1)
        if fail_rank is not None:
            assert st.combine == "sliced" and st.p2p is None and f"rank {fail_rank}" in st.combine_fallback
        st.bucketed = bucketed
        for t in range(steps):   # several steps: the next step starts from the updated state
            st.set_tokens(t)
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


def _run(world, tiny, combine="sliced", sync="host", bucketed=True, zero1=False, steps=1, fail_rank=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, tiny, q, combine, sync, bucketed, zero1, steps,
                                            fail_rank))
          for r in range(world)]
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


def test_tiny_step_root_p2p_whole_gradient(tiny_single):
    """the un-bucketed peer-memory combine (one bucket) gives the same root"""
    for rank, root, loss, pdig in _run(2, True, combine="p2p", bucketed=False):
        assert root == tiny_single[1]


def test_tiny_step_root_p2p_device_flags_across_processes(tiny_single):
    """the device-side signal / wait protocol (release / acquire on IPC-mapped flags,
    system scope) between two rank PROCESSES -- the transport bench.py uses at N > 1.
    On one GPU the two contexts time-slice, so every wait completes only after the
    other process's context gets the GPU: slow, but it must complete without a
    timeout and give the single-process root."""
    for rank, root, loss, pdig in _run(2, True, combine="p2p", sync="device"):
        assert root == tiny_single[1], f"device-flag p2p rank {rank}: step root differs"
        assert pdig == tiny_single[3]


@pytest.mark.parametrize("world", [2, 4])
def test_full_gpt2_step_root_p2p_bucketed(world, full_single):
    """full GPT-2 124M step with the per-layer bucketed peer-memory combine (13 buckets
    overlapping the backward on a comm stream) at G = 2, 4: the G = 1 root"""
    for rank, root, loss, pdig in _run(world, False, combine="p2p"):
        assert root == full_single[1], f"bucketed p2p G={world} rank {rank}: full step root differs"
        assert pdig == full_single[3]


@pytest.mark.parametrize("world", [2, 4])
def test_tiny_zero1_three_steps_root_equals_replicated(world):
    """ZeRO-1 (optimizer state partitioned by parameter tensor, owner-only AdamW + commit,
    parameters broadcast, replicated digests exchanged by owner) over 3 steps: every
    step's root equals the single-process replicated run's"""
    single = _run(1, True, steps=3)[0]
    for rank, root, loss, pdig in _run(world, True, combine="p2p", zero1=True, steps=3):
        assert root == single[1], f"ZeRO-1 G={world} rank {rank}: step-3 root differs"
        assert loss == single[2]
        assert pdig == single[3]


@pytest.mark.parametrize("world", [2, 8])
def test_full_gpt2_zero1_root_equals_world1(world, full_single):
    for rank, root, loss, pdig in _run(world, False, combine="p2p", zero1=True):
        assert root == full_single[1], f"ZeRO-1 full G={world} rank {rank}: step root differs"


# ---------------------------------------------------------------- config 2: M-split GEMM
MSPLIT_N = (1024, 2048)


def _msplit_worker(rank, world, port, q):
    """rank r computes the R-GEMM rows [r n/G, (r+1) n/G) with the full K (P:584-591:
    only order-insensitive dimensions are split) and commits the slab's data root
    (CommitPlan mode 1); the G slab roots are all-gathered and joined by
    verde_digest_from_subroots -- bench.py's config-2 digest path."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2502_19405_b200 as R
        from paper_2502_19405_b200.dist import all_gather_rows
        out = []
        for n in MSPLIT_N:
            A, B = synth.gemm_inputs(n, "msplit")
            rows = n // world
            Cs = R.repops_gemm(torch.from_numpy(np.ascontiguousarray(A[rank * rows:(rank + 1) * rows])).cuda(),
                               torch.from_numpy(B).cuda())
            roots = torch.zeros((1, 32), dtype=torch.uint8, device="cuda")
            R.CommitPlan([Cs], roots, modes=[1]).run()
            parts = all_gather_rows(roots, world).cpu().numpy()
            sub = b"".join(parts[r, 0].tobytes() for r in range(world))
            dig = R.verde_digest_from_subroots(sub, R.F32, (n, n), n * n * 4)
            # the slab bits themselves, gathered, for the oracle comparison on rank 0
            full = all_gather_rows(Cs, world).reshape(n, n).cpu().numpy() if n == MSPLIT_N[0] else None
            out.append((dig.hex(), None if full is None else full.tobytes()))
        q.put((rank, out))
    except Exception:
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def _run_msplit(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_msplit_worker, args=(r, world, port, q)) for r in range(world)]
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
    return sorted(res, key=lambda r: r[0])


@pytest.fixture(scope="module")
def msplit_single():
    import numpy as np

    import oracle
    import synth
    res = _run_msplit(1)[0][1]
    # G = 1 against the oracle: the full product's bits and the tensor digest
    n = MSPLIT_N[0]
    A, B = synth.gemm_inputs(n, "msplit")
    ref = oracle.gemm(A, B)
    assert np.frombuffer(res[0][1], np.uint32).tobytes() == ref.view(np.uint32).tobytes()
    assert bytes.fromhex(res[0][0]) == oracle.commit_tensor(ref)
    return res


@pytest.mark.parametrize("world", [2, 4, 8])
def test_msplit_gemm_digest_identical_across_world_sizes(world, msplit_single):
    import numpy as np

    import oracle
    for rank, out in _run_msplit(world):
        for (dig, full), (dig1, full1), n in zip(out, msplit_single, MSPLIT_N):
            assert dig == dig1, f"G={world} rank {rank} n={n}: joined slab digest differs from G=1"
            if full is not None:
                assert full == full1, f"G={world} rank {rank}: gathered slabs differ from G=1"
                C = np.frombuffer(full, np.float32).reshape(n, n)
                assert bytes.fromhex(dig) == oracle.commit_tensor(C)


def test_p2p_setup_failure_falls_back_on_every_rank(tiny_single):
    """one rank cannot map a peer's CUDA IPC buffer: every rank learns it (the setup agrees
    over the process group), falls back to the NCCL-style sliced transport of the same
    R-TREE_S, and the step root is the single-process one"""
    for rank, root, loss, pdig in _run(2, True, combine="p2p", fail_rank=1):
        assert root == tiny_single[1], f"rank {rank}: step root differs after the fallback"
