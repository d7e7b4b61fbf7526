"""Exercise every librepops.so kernel on tiny shapes -- the workload for compute-sanitizer
(memcheck / racecheck / synccheck).  Sections (argv[1], comma separated):
  gemm     every R-GEMM tile configuration, 4 layouts, ragged + full tiles, batched, gemm_tn
  rowops   sums, softmax (+ causal, long rows), LayerNorm, cross entropy, R-SEQ folds
  elem     software math, GELU, dropout, conversions, embedding, AdamW, tree, transposes
  commit   SHA-256 commit plans (multi-pass reduce), root plan, chunk leaves
  attn     fused attention forward
  steps    tiny GPT-2 step (aux + commit side streams), MLP step, tiny Llama prefill
  p2p      peer-memory combine + device signal / wait flags with virtual ranks on streams
Exits 0 when every section ran; the sanitizer decides on errors."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_19405_b200 as R  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gemm():
    for (M, N, K) in ((33, 70, 19), (64, 128, 32), (130, 129, 40)):
        A, B = synth.gemm_inputs((M, N, K), "san")
        for ta in (0, 1):
            for tb in (0, 1):
                Ai = dev(A.T.copy() if ta else A)
                Bi = dev(B.T.copy() if tb else B)
                for cfg in range(R.gemm_num_cfgs()):
                    R.repops_gemm(Ai, Bi, transA=bool(ta), transB=bool(tb), cfg=cfg)
                R.repops_gemm(Ai, Bi, transA=bool(ta), transB=bool(tb), epi=R.EPI_BIAS, bias=dev(synth.uniform(3, N)))
    q = dev(synth.uniform(9, (2 * 32, 3 * 32)))
    S = torch.empty((2 * 2 * 32, 32), device="cuda")
    R.repops_gemm_strided_batched(q, q, S, M=32, N=32, K=16, lda=96, ldb=96, ldc=32, sA=(32 * 96, 16),
                                  sB=(32 * 96, 16), sC=(2 * 32 * 32, 32 * 32), batch=(2, 2), transB=True,
                                  epi=R.EPI_SCALE, scale=0.25, offB=32)
    A = dev(synth.uniform(4, (1024, 1024)))
    R.repops_gemm(A, A)  # NN through the transposed-A path (stream-ordered temporary)


def rowops():
    for cols in (1, 129, 4097, 9000):
        x = dev(synth.uniform(cols, (5, cols)))
        R.repops_sum_rows(x)
        y = R.repops_softmax(x)
        R.repops_softmax_backward(y, x, scale=0.5)
        if cols <= 4096:  # LayerNorm rows (<= 4096 columns, the kernels' limit)
            g = dev(synth.uniform(1, cols))
            ly, mu, rs = R.repops_layernorm(x, g, g)
            R.repops_layernorm_backward(x, x, g, mu, rs)
            R.repops_layernorm_backward_params(x, x, mu, rs, nseg=5)
        R.repops_cross_entropy(x, torch.zeros(5, dtype=torch.int32, device="cuda"), scale=0.5,
                               loss=torch.empty(5, device="cuda"), dlogits=torch.empty_like(x), V=cols)
    x = dev(synth.uniform(7, (4 * 64, 64)))
    R.repops_softmax(x, causal=True)
    x = dev(synth.uniform(7, (2 * 512, 512)))
    R.repops_softmax(x, causal=True)
    R.repops_sum_cols_seq(dev(synth.uniform(8, (64, 33))), nseg=4)
    R.repops_rmsnorm(dev(synth.uniform(8, (6, 96))), dev(synth.uniform(9, 96)))


def elem():
    x = dev(synth.uniform(11, 4099, 4.0))
    for f in (R.repops_exp, R.repops_log, R.repops_tanh, R.repops_rsqrt, R.repops_gelu, R.repops_sin, R.repops_cos,
              R.repops_erf, R.repops_gelu_erf, R.repops_relu):
        f(x)
    R.repops_gelu_backward(x, x)
    R.repops_gelu_erf_backward(x, x)
    R.repops_relu_backward(x, x)
    R.repops_add(x, x)
    R.repops_rand_uniform(1, 2, 4099)
    y, m = R.repops_dropout(x, 0.25, 3, 4)
    R.repops_dropout_backward(x, 0.25, 3, 4)
    X = dev(synth.uniform(12, (67, 45)))
    R.repops_transpose(X)
    R.repops_tree_sum([x, x, x, x])
    p, g = x.clone(), x.clone()
    R.repops_adamw(p, g, torch.zeros_like(p), torch.zeros_like(p), 1, 1e-3, 0.9, 0.95, 1e-8, 0.1, True)
    wte, wpe = dev(synth.uniform(13, (50, 16))), dev(synth.uniform(14, (8, 16)))
    tok = torch.randint(0, 50, (16,), dtype=torch.int32, device="cuda")
    x0 = R.repops_embedding(tok, wte, wpe, 8)
    R.repops_embedding_backward(tok[:8].contiguous(), x0[:8].contiguous(), 8, torch.zeros_like(wte),
                                torch.zeros_like(wpe))
    for dt in (torch.bfloat16, torch.float16):
        h = R.repops_convert(X, dt)
        R.repops_convert(h, torch.float32)


def commit():
    ts = [dev(synth.uniform(20 + i, n)) for i, n in enumerate((1, 1023, 1024 * 300 + 7, 4096 * 1025))]
    R.verde_commit_tensors(ts)
    d = torch.zeros((len(ts), 32), dtype=torch.uint8, device="cuda")
    plan = R.CommitPlan(ts, d)
    plan.run()
    R.verde_chunk_leaves(ts[2])
    torch.cuda.synchronize()


def attn():
    T, hd, H = 128, 64, 2
    if not R.repops_attention_fwd_supported(T, hd):
        return
    qkv = dev(synth.uniform(30, (T, 3 * H * hd)))
    d = H * hd
    att = torch.empty((T, d), device="cuda")
    S = torch.empty((H * T, T), device="cuda")
    P = torch.empty((H * T, T), device="cuda")
    R.repops_attention_fwd(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, 2 * d, (1, H), att, d, (T * d, hd), S=S, P=P,
                           sp=(H * T * T, T * T), scale=0.125, causal=True)


def steps():
    from paper_2502_19405_b200.gpt2 import GPT2Config, GPT2Step
    from paper_2502_19405_b200.llama import LlamaConfig, LlamaPrefill
    from paper_2502_19405_b200.mlp import MLPConfig, MLPStep
    st = GPT2Step(GPT2Config.tiny())
    st.set_tokens(0)
    st.run()
    st.device_root()
    st.step_root()
    m = MLPStep(MLPConfig())
    m.run()
    lp = LlamaPrefill(LlamaConfig.tiny())
    lp.load_weights()
    lp.set_tokens()
    lp.run()
    lp.device_root()


def p2p():
    from paper_2502_19405_b200.dist import p2p_slice
    G, n = 4, 4099
    streams = [torch.cuda.Stream() for _ in range(G)]
    partial = [dev(synth.uniform(40 + r, n)) for r in range(G)]
    grad = [torch.zeros(n, device="cuda") for _ in range(G)]
    flags = [torch.zeros(2 * G, dtype=torch.int32, device="cuda") for _ in range(G)]
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    # all signals are enqueued before any wait, so the protocol completes even if the
    # sanitizer serialises the launches
    for r in range(G):
        R.repops_p2p_signal([f[:G] for f in flags], r, 1, stream=streams[r])
    for r in range(G):
        with torch.cuda.stream(streams[r]):
            R.repops_p2p_wait(flags[r][:G], G, 1, 20000, status, stream=streams[r])
            lo, hi = p2p_slice(r, G, n)
            R.repops_p2p_tree_combine(partial, lo, hi, grad, stream=streams[r], status=status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0


SECTIONS = dict(gemm=gemm, rowops=rowops, elem=elem, commit=commit, attn=attn, steps=steps, p2p=p2p)

if __name__ == "__main__":
    torch.cuda.set_device(0)
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(SECTIONS)
    for nm in names:
        SECTIONS[nm]()
        torch.cuda.synchronize()
        print(f"section {nm}: ok", flush=True)
