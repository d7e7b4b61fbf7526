"""Config 4 (Llama-3-8B-shaped FP32 prefill, tensor-parallel N split): kernel
parity of the Llama operators, whole-pass parity of a tiny Llama against the
oracle (every committed tensor, 0 ULP, and its digest), bit-identity of the
pass's Merkle root for G = 1, 2, 4, 8 (processes sharing one GPU over gloo),
and sampled referee recomputes of the full-size pass."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from oracle import llama_prefill as olp

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def test_llama_kernels_parity():
    import paper_2502_19405_b200 as R
    x = synth.uniform(1, (77, 4096), 3.0)
    w = synth.uniform(2, 4096)
    y, rs = oracle.rmsnorm(x, w)
    gy, grs = R.repops_rmsnorm(dev(x), dev(w))
    assert np.array_equal(bits(gy.cpu()), bits(y)) and np.array_equal(bits(grs.cpu()), bits(rs))
    g = np.concatenate([synth.uniform(3, 100003, 30.0), np.float32([0, -0.0, 200, -200, np.inf, -np.inf, np.nan])])
    u = synth.uniform(4, g.size, 2.0)
    assert np.array_equal(bits(R.repops_swiglu(dev(g), dev(u)).cpu()), bits(oracle.swiglu(g, u)))
    T, H, hd = 96, 6, 128
    q = synth.uniform(5, (T, H * hd + 32))  # ld > H*hd
    cos, sin = synth.rope_tables(T, hd)
    ref = oracle.rope(np.ascontiguousarray(q[:, :H * hd]), cos, sin, H, hd)
    got = R.repops_rope(dev(q)[:, :H * hd], dev(cos), dev(sin), H, hd, out=torch.empty(T, H * hd, device="cuda"))
    assert np.array_equal(bits(got.cpu()), bits(ref))
    table = synth.uniform(6, (500, 33))
    idx = synth.integers(7, 41, 500)
    assert np.array_equal(bits(R.repops_gather_rows(dev(table), dev(idx)).cpu()), bits(table[idx]))
    for seed, scale, n in ((11, 1.0, 1000003), (12, 0.034641016151377546, 4097), (2 ** 63 + 5, 3.0, 77)):
        t = torch.empty(n, device="cuda")
        R.repops_fill_uniform(t, seed, scale)
        assert np.array_equal(bits(t.cpu()), bits(synth.uniform(seed, n, scale)))


@pytest.fixture(scope="module")
def tiny_llama():
    from paper_2502_19405_b200.llama import LlamaConfig, LlamaPrefill
    cfg = LlamaConfig.tiny()
    st = LlamaPrefill(cfg)
    st.load_weights()
    st.set_tokens()
    st.run()
    root = st.device_root()
    ref, W = olp.run_prefill(cfg)
    return cfg, st, root, ref, W


def test_tiny_llama_every_tensor_bit_exact(tiny_llama):
    cfg, st, root, ref, W = tiny_llama
    table = st.digests.cpu().numpy()
    n = 0
    for t in st.tensors:
        if t.name.startswith("param/"):
            name = t.name.split("/", 1)[1]
            assert table[t.slot].tobytes() == oracle.commit_tensor(W[name]), t.name
            continue
        r = np.ascontiguousarray(ref[t.name])
        g = t.view.cpu().numpy()
        assert g.shape == r.reshape(g.shape).shape
        if g.dtype == np.float32:
            bad = np.flatnonzero(bits(g).ravel() != bits(r).ravel())
            assert bad.size == 0, f"{t.name}: {bad.size}/{g.size} elements differ"
        else:
            assert np.array_equal(g.ravel(), r.ravel())
        code = 2 if r.dtype == np.int32 else 1
        assert table[t.slot].tobytes() == oracle.commit_tensor(r.reshape(g.shape), code), t.name
        n += 1
    assert n > 150


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2502_19405_b200.llama import LlamaConfig, LlamaPrefill
        st = LlamaPrefill(LlamaConfig.tiny(), rank=rank, world=world)
        st.load_weights()
        st.set_tokens()
        st.run()
        q.put((rank, st.device_root().hex(), st.logits.cpu().numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_tiny_llama_root_identical_across_tp_degrees(world, tiny_llama):
    cfg, st, root, ref, W = tiny_llama
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    per = cfg.nb // world
    for rank, rt, logits in res:
        assert rt == root.hex(), f"TP degree {world}, rank {rank}: root differs from G=1"
        mine = np.frombuffer(logits, np.float32).reshape(per, cfg.seq, cfg.vocab // cfg.nb)
        for j in range(per):
            assert np.array_equal(bits(mine[j]), bits(ref[f"b{rank * per + j}/logits"]))


def test_full_llama_prefill_sampled_referee():
    """Full config-4 pass on one GPU; the oracle recomputes sampled outputs one by one
    from the pass's own (committed) inputs -- Verde Case 3 at full size."""
    from paper_2502_19405_b200.llama import LlamaConfig, LlamaPrefill
    cfg = LlamaConfig()
    st = LlamaPrefill(cfg)
    st.load_weights()
    st.set_tokens()
    st.run()
    root = st.device_root()
    assert len(root) == 32
    a = st.act[0]
    T, d, hd, qh = cfg.seq, cfg.d, cfg.hd, cfg.qh
    x0 = st.x[0].cpu().numpy()
    # RMSNorm rows of layer 0
    w = synth.llama_param("l0.attn_norm", (d,), "g")
    rows = [0, 1, 777, T - 1]
    y, rs = oracle.rmsnorm(x0[rows], w)
    assert np.array_equal(bits(a["xn"].cpu().numpy()[rows]), bits(y))
    # sampled QKV outputs of block 3 (full K = 4096 fold each)
    xn = a["xn"].cpu().numpy()
    wq = synth.llama_param("l0.wq", (d, cfg.n_head * hd), "w")
    qkv3 = a["qkv"][3].cpu().numpy()
    rng = np.random.default_rng(5)
    for i, j in zip(rng.integers(0, T, 12), rng.integers(0, qh * hd, 12)):
        r = oracle.gemm_element(xn, np.ascontiguousarray(wq[:, 3 * qh * hd:4 * qh * hd]), int(i), int(j))
        assert bits(qkv3[i, j]) == bits(r), (i, j)
    # attention (R29: one operator) of block 3, head 1, recomputed for sampled query rows
    # from the committed RoPE'd Q/K and V: scores, causal softmax, PV over all T keys
    qk3 = a["qk"][3].cpu().numpy()
    v3 = np.ascontiguousarray(qkv3[:, (qh + 1) * hd:])
    k3 = np.ascontiguousarray(qk3[:, qh * hd:(qh + 1) * hd])
    o3 = a["o"][3].cpu().numpy()
    scale = float(np.float32(1.0 / np.sqrt(hd)))
    for i in (0, 5, 1000, T - 1):
        q_row = np.ascontiguousarray(qk3[i:i + 1, hd:2 * hd])
        s_row = oracle.gemm(q_row, k3, transB=True, epi=2, scale=scale)
        p_row = np.zeros((1, T), np.float32)
        p_row[0, :i + 1] = oracle.softmax(np.ascontiguousarray(s_row[:, :i + 1]))[0]
        assert np.array_equal(bits(o3[i, hd:2 * hd]), bits(oracle.gemm(p_row, v3)[0])), i
    # SwiGLU elements of the last layer, block 7
    al = st.act[cfg.n_layer - 1]
    g = al["g"][7].cpu().numpy()[:64]
    u = al["u"][7].cpu().numpy()[:64]
    assert np.array_equal(bits(al["a"][7].cpu().numpy()[:64]), bits(oracle.swiglu(g, u)))


def test_llama_fused_probs_root_equals_unfused(monkeypatch):
    """a Llama-shaped prefill with hd = 128 (the full model's head dim) through the fused
    scores + softmax kernel commits the same attention outputs as the causal-skip scores
    R-GEMM + R-SOFTMAX path: identical pass roots"""
    from paper_2502_19405_b200.llama import LlamaConfig, LlamaPrefill
    cfg = LlamaConfig(n_layer=2, d=2048, n_head=16, n_kv=8, hd=128, ffn=256, vocab=512, seq=256)
    roots = []
    for flag in ("1", "0"):
        monkeypatch.setenv("REPOPS_ATTN_PROBS_LLAMA", flag)
        st = LlamaPrefill(cfg)
        assert st.attn_probs == (flag == "1")
        st.load_weights()
        st.set_tokens()
        st.run()
        roots.append(st.device_root())
        del st
        torch.cuda.empty_cache()
    assert roots[0] == roots[1]
