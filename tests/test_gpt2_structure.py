"""CPU tests of the GPT-2 step's host logic: the Verde node graph (reading R13)
is identical for every world size and rank (the step root can only be
G-invariant if the graph is), it is topologically ordered, and the multi-GPU
combine / digest-gather logic (paper_2502_19405_b200.dist) reproduces the
single-GPU tree over S shards on a world_size-2 gloo group."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from paper_2502_19405_b200 import dist as D
from paper_2502_19405_b200.gpt2 import OP, REPLICATED, GPT2Config, GPT2Step


@pytest.fixture(scope="module")
def ref_graph():
    return GPT2Step(GPT2Config(), structure_only=True)


def test_full_config_sizes(ref_graph):
    st = ref_graph
    assert st.P == 124_439_808  # GPT-2 small parameter count
    assert len(st.nodes) == 3212  # R29: one ATTENTION + one ATTENTION_BWD node per (shard, layer)
    assert len(GPT2Step(GPT2Config(), structure_only=True, attn_nodes="primitive").nodes) == 3596
    assert st.n_slots == st.rep_slots + 8 * st.shard_slots


@pytest.mark.parametrize("world", [2, 4, 8])
def test_graph_identical_for_every_world_and_rank(ref_graph, world):
    for rank in range(world):
        st = GPT2Step(GPT2Config(), rank=rank, world=world, structure_only=True)
        assert np.array_equal(st.node_blob, ref_graph.node_blob)
        assert np.array_equal(st.node_offs, ref_graph.node_offs)
        assert np.array_equal(st.node_slots, ref_graph.node_slots)
        assert np.array_equal(st.node_soffs, ref_graph.node_soffs)


def test_graph_is_topological_and_single_producer(ref_graph):
    st = ref_graph
    seen = set()
    for nd in st.nodes:
        for t in nd.inputs:
            assert st.tensors[t].producer < nd.index, (nd.name, st.tensors[t].name)
        for t in nd.outputs:
            assert t not in seen
            seen.add(t)
    assert len(seen) == len(st.tensors)
    # node order: params, then per shard, then tree, then AdamW (R13)
    shards = [nd.shard for nd in st.nodes]
    per = [s for s in shards if s != REPLICATED]
    assert per == sorted(per)
    assert st.nodes[0].op == OP["PARAM_IN"] and st.nodes[-1].op == OP["ADAMW"]
    # every parameter has exactly one final per-shard gradient producer per shard
    trees = [nd for nd in st.nodes if nd.op == OP["TREE_SUM"]]
    assert len(trees) == len(st.specs)
    for nd in trees:
        assert len(nd.inputs) == 8
        assert [st.nodes[st.tensors[t].producer].shard for t in nd.inputs] == list(range(8))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_llama_tp_graph_identical_for_every_degree(world):
    from paper_2502_19405_b200.llama import LlamaConfig, LlamaPrefill
    ref = LlamaPrefill(LlamaConfig(), structure_only=True)
    assert len(ref.nodes) == 2480  # R26 ROPE_TABLES node; R29: one ATTENTION node per (layer, block)
    for rank in range(world):
        st = LlamaPrefill(LlamaConfig(), rank=rank, world=world, structure_only=True)
        assert np.array_equal(st.node_blob, ref.node_blob) and np.array_equal(st.node_slots, ref.node_slots)
    # 8,030,261,248 parameters (Llama-3-8B)
    import synth as S
    specs = S.llama_param_specs(32, 4096, 32, 8, 128, 14336, 128256)
    assert sum(int(np.prod(s)) for _, s, _ in specs) == 8_030_261_248


def test_shard_block_rules():
    assert D.shard_block(3, 4, 8) == (6, 2)
    with pytest.raises(ValueError):
        D.shard_block(0, 3, 8)


# ---------------------------------------------------------------- gloo world_size 2
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_tree(parts, out):
    r = torch.from_numpy(oracle.tree_sum([p.numpy() for p in parts]))
    if out is not None:
        out.copy_(r)
        return out
    return r


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S = 8
        s0, per = D.shard_block(rank, world, S)
        parts = [torch.from_numpy(synth.uniform(1000 + s, 5003, 4.0)) for s in range(S)]
        parts[0][:3] = torch.tensor([2.0 ** 24, 1.0, 1.0])
        parts[4][:3] = torch.tensor([1.0, 1.0, 2.0 ** 24])
        got = D.dp_tree_combine(parts[s0:s0 + per], world, _oracle_tree)
        got2 = D.dp_tree_combine_sliced(parts[s0:s0 + per], world, _oracle_tree)
        assert got2.numpy().tobytes() == got.numpy().tobytes()
        # digest table: replicated region + shard regions; each rank fills its own
        rep, ss = 3, 5
        table = torch.zeros((rep + S * ss, 32), dtype=torch.uint8)
        table[:rep] = 7
        for s in range(s0, s0 + per):
            table[rep + s * ss: rep + (s + 1) * ss] = s + 1
        D.gather_shard_digests(table, rep, ss, s0, per, world)
        q.put((rank, got.numpy().tobytes(), table.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_dp_combine_and_digest_gather(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    S = 8
    parts = [synth.uniform(1000 + s, 5003, 4.0) for s in range(S)]
    parts[0][:3] = [2.0 ** 24, 1.0, 1.0]
    parts[4][:3] = [1.0, 1.0, 2.0 ** 24]
    ref = oracle.tree_sum(parts).tobytes()
    expect = np.zeros((3 + S * 5, 32), np.uint8)
    expect[:3] = 7
    for s in range(S):
        expect[3 + s * 5: 3 + (s + 1) * 5] = s + 1
    for rank, tree_bytes, table_bytes in res:
        assert tree_bytes == ref, f"rank {rank}: tree differs from the single-process R-TREE_S"
        assert table_bytes == expect.tobytes(), f"rank {rank}: digest table gather wrong"


def test_p2p_slices_partition_and_align():
    """the peer-memory combine's slices are disjoint, cover [0, n) and start on float4 boundaries"""
    for world in (1, 2, 4, 8):
        for n in (0, 1, 3, 4, 5, 31, 4096, 100003, 124439808):
            sl = [D.p2p_slice(r, world, n) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == n
            for (lo, hi), (lo2, _) in zip(sl, sl[1:]):
                assert hi == lo2 and lo <= hi
            assert all(lo % 4 == 0 or lo == n for lo, _ in sl)


def test_combine_transport_validation():
    """host-side validation of the gradient-combine transports (no GPU needed)"""
    with pytest.raises(ValueError):
        GPT2Step(GPT2Config.tiny(), structure_only=True, combine="allreduce")  # NCCL reductions are never used
    with pytest.raises(ValueError):
        D.P2PTreeCombine(1000, 0, 3)   # world must be a power of two <= 8 (aligned R-TREE_S subtrees)
    with pytest.raises(ValueError):
        D.P2PTreeCombine(1000, 0, 16)
    # the structure (node graph, slots) does not depend on the transport
    a = GPT2Step(GPT2Config.tiny(), structure_only=True, combine="sliced")
    b = GPT2Step(GPT2Config.tiny(), structure_only=True, combine="p2p")
    assert np.array_equal(a.node_blob, b.node_blob) and np.array_equal(a.node_slots, b.node_slots)


def test_zero1_ownership_partition():
    """ZeRO-1 ownership: every parameter tensor has exactly one owner, the same on every
    rank, and the compact optimizer-state buffers hold exactly the owned tensors"""
    from paper_2502_19405_b200.gpt2 import GPT2Config, GPT2Step
    for world in (2, 4, 8):
        steps = [GPT2Step(GPT2Config(), rank=r, world=world, structure_only=True, zero1=True) for r in range(world)]
        owners = [st.owner for st in steps]
        assert all(o == owners[0] for o in owners)
        owned = [set(st.owned) for st in steps]
        assert set().union(*owned) == {n for n, _, _ in steps[0].specs}
        assert sum(len(o) for o in owned) == len(steps[0].specs)
        assert sum(st.P_own for st in steps) == steps[0].P
        # greedy balance: no rank exceeds the largest tensor plus the ideal share
        wte = 50257 * 768
        assert max(st.P_own for st in steps) <= max(wte, steps[0].P // world + wte)
