"""GPU parity: every kernel of librepops.so against the CPU oracle, element by
element as raw uint32 bit patterns (tolerance 0 ULP, north_star), on seeded
synthetic inputs from `synth`, through the C ABI (the Python binding only
marshals arguments).  Sizes span several tiles plus ragged tails; edge cases
(empty, K = 0, K tails, -0, NaN/Inf, long rows) are included."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

R = None


def setup_module(_):
    global R
    import paper_2502_19405_b200 as mod
    R = mod


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def assert_bits(gpu, ref, what=""):
    g = np.ascontiguousarray(gpu, dtype=np.float32).view(np.uint32)
    r = np.ascontiguousarray(ref, dtype=np.float32).view(np.uint32)
    assert g.shape == r.shape, (what, g.shape, r.shape)
    bad = np.flatnonzero(g.ravel() != r.ravel())
    assert bad.size == 0, f"{what}: {bad.size} of {g.size} differ; first at {bad[:5]}: " \
                          f"gpu {g.ravel()[bad[:3]]} oracle {r.ravel()[bad[:3]]}"


# ------------------------------------------------------------------ GEMM
GEMM_SHAPES = [(1, 1, 1), (7, 5, 3), (128, 128, 128), (129, 257, 33), (300, 200, 1000), (64, 96, 17),
               (513, 130, 7), (5, 700, 256)]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
@pytest.mark.parametrize("tA,tB", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_parity(M, N, K, tA, tB):
    A, B = synth.gemm_inputs((M, N, K), "gp")
    Ain = np.ascontiguousarray(A.T) if tA else A
    Bin = np.ascontiguousarray(B.T) if tB else B
    ref = oracle.gemm(Ain, Bin, transA=bool(tA), transB=bool(tB))
    for cfg in (None, 0, 1, 19):
        got = R.repops_gemm(dev(Ain), dev(Bin), transA=bool(tA), transB=bool(tB), cfg=cfg)
        assert_bits(host(got), ref, f"gemm {M}x{N}x{K} tA{tA} tB{tB} cfg{cfg}")


@pytest.mark.parametrize("K", [7, 16, 1005])
@pytest.mark.parametrize("tA,tB", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_full_tiles_ragged_k_every_cfg(K, tA, tB):
    # M, N multiples of every tile shape -> the predicate-free full-tile loads,
    # with a ragged last K tile taking the bounded path (no zero padding, R2)
    M, N = 256, 512
    A, B = synth.gemm_inputs((M, N, K), "gk")
    Ain = np.ascontiguousarray(A.T) if tA else A
    Bin = np.ascontiguousarray(B.T) if tB else B
    ref = oracle.gemm(Ain, Bin, transA=bool(tA), transB=bool(tB))
    assert R.gemm_num_cfgs() >= 20
    for cfg in range(R.gemm_num_cfgs()):  # every tile configuration, XP and BK = 32 variants included
        got = R.repops_gemm(dev(Ain), dev(Bin), transA=bool(tA), transB=bool(tB), cfg=cfg)
        assert_bits(host(got), ref, f"gemm {M}x{N}x{K} tA{tA} tB{tB} cfg{cfg}")


@pytest.mark.parametrize("tA,tB", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_ragged_every_cfg(tA, tB):
    # ragged M / N / K tails on every configuration (the bounded-load paths)
    M, N, K = 197, 301, 77
    A, B = synth.gemm_inputs((M, N, K), "gr")
    Ain = np.ascontiguousarray(A.T) if tA else A
    Bin = np.ascontiguousarray(B.T) if tB else B
    ref = oracle.gemm(Ain, Bin, transA=bool(tA), transB=bool(tB))
    for cfg in range(R.gemm_num_cfgs()):
        got = R.repops_gemm(dev(Ain), dev(Bin), transA=bool(tA), transB=bool(tB), cfg=cfg)
        assert_bits(host(got), ref, f"gemm {M}x{N}x{K} tA{tA} tB{tB} cfg{cfg}")


@pytest.mark.parametrize("K", [16, 48, 96, 1024])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_tn_kernel_full_tiles(K, epi):
    # gemm_tn.cu (cfg 20: BK 32 when K % 32 == 0, else 16; cfg 21: BK 16), A^T stored,
    # several 128 x 128 tiles and rasterisation groups; bias / scale epilogues
    M, N = 384, 640
    A, B = synth.gemm_inputs((M, N, K), "gtn")
    At = np.ascontiguousarray(A.T)
    bias = synth.uniform(31, N)
    ref = oracle.gemm(At, B, transA=True, epi=epi, bias=bias if epi == 1 else None, scale=0.375)
    for cfg in (None, 20, 21, 22, 23):
        got = R.repops_gemm(dev(At), dev(B), transA=True, epi=epi, bias=dev(bias) if epi == 1 else None,
                            scale=0.375, cfg=cfg)
        assert_bits(host(got), ref, f"gemm_tn K{K} epi{epi} cfg{cfg}")


@pytest.mark.parametrize("M,N,K", [(301, 200, 77), (50257 // 16, 768, 513), (129, 131, 32), (5, 7, 3),
                                   (1000, 130, 1)])
def test_gemm_tn_kernel_ragged_edges(M, N, K):
    # ragged M / N edge tiles (zero-filled bounded copies, guarded epilogue) and a ragged
    # last K tile (short loop, no padding) in gemm_tn.cu, e.g. the LM wgrad's M = vocab
    # and the LM dgrad's K = vocab; 16-byte aligned padded rows (ld % 4 == 0)
    A, B = synth.gemm_inputs((M, N, K), "gtr")
    At = np.ascontiguousarray(A.T)
    lda, ldb = (M + 3) // 4 * 4 + 4, (N + 3) // 4 * 4
    Ab = np.full((K, lda), np.nan, np.float32)
    Ab[:, :M] = At
    Bb = np.full((K, ldb), np.nan, np.float32)
    Bb[:, :N] = B
    ref = oracle.gemm(At, B, transA=True)
    for cfg in (None, 20, 21, 22, 23):
        got = R.repops_gemm(dev(Ab)[:, :M], dev(Bb)[:, :N], transA=True, cfg=cfg)
        assert_bits(host(got), ref, f"gemm_tn ragged {M}x{N}x{K} cfg{cfg}")


def test_gemm_tn_kernel_batched_and_strided_output():
    # the GPT-2 per-shard weight-gradient layout: a batch of A^T B whose outputs sit at a
    # large stride inside one buffer with ldc > N (the step's [S, P] gradient rows)
    Bsz, M, N, K = 3, 256, 384, 64
    ldc, sc = N + 64, M * (N + 64) + 100
    A = synth.uniform(41, (Bsz, K, M))
    Bm = synth.uniform(42, (Bsz, K, N))
    C = torch.zeros(Bsz * sc, device="cuda")
    R.repops_gemm_strided_batched(dev(A), dev(Bm), C, M=M, N=N, K=K, lda=M, ldb=N, ldc=ldc, sA=(K * M, 0),
                                  sB=(K * N, 0), sC=(sc, 0), batch=(Bsz, 1), transA=True)
    got = host(C)
    for b in range(Bsz):
        blk = got[b * sc:b * sc + M * ldc].reshape(M, ldc)
        assert_bits(blk[:, :N], oracle.gemm(A[b], Bm[b], transA=True), f"batched gemm_tn {b}")
        assert np.all(blk[:, N:].view(np.uint32) == 0), "wrote outside the C tile"


def test_copy2d_batched_places_blocks_bit_exactly():
    # tensor-parallel block placement (Llama gathers): nb blocks of rows x w into column
    # ranges of one matrix, float4 and scalar paths, every bit pattern preserved (NaN payloads)
    for nb, rows, w in ((8, 33, 12), (3, 17, 5)):
        src = synth.uniform(81 + w, (nb, rows, w))
        src.view(np.uint32)[0, 1, :2] = [0x7FA00001, 0xFFC00002]   # NaN payloads travel unchanged
        full = torch.zeros((rows, nb * w), device="cuda")
        R.repops_copy2d_batched(dev(src), full, rows, w, w, rows * w, nb * w, w, nb)
        ref = np.concatenate([src[b] for b in range(nb)], axis=1)
        assert np.array_equal(host(full).view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("M,N,K,tA", [(256, 384, 96, 1), (4096 // 8, 3072 // 4, 768 // 4, 1), (130, 200, 77, 1),
                                      (64, 96, 40, 0)])
@pytest.mark.parametrize("post", [1, 2])
def test_gemm_post_fused_gelu(M, N, K, tA, post):
    # R-GEMM with GELU (post 1) or GELU backward at X (post 2) fused into the epilogue:
    # C and C2 equal the GEMM followed by the separate elementwise launch, and the oracle
    # (A^T kernel shapes fused; the others -- ragged / NN -- take the unfused fallback)
    A, B = synth.gemm_inputs((M, N, K), "gpost")
    A = (A * np.float32(2.0)).astype(np.float32)
    X = synth.uniform(91, (M, N), 4.0)
    bias = synth.uniform(92, N)
    Ain = np.ascontiguousarray(A.T) if tA else A
    epi = 1 if post == 1 else 0
    C, C2 = R.repops_gemm_post(dev(Ain), dev(B), post, torch.empty((M, N), device="cuda"),
                               X=dev(X) if post == 2 else None, transA=bool(tA), epi=epi,
                               bias=dev(bias) if epi else None)
    refC = oracle.gemm(Ain, B, transA=bool(tA), epi=epi, bias=bias if epi else None)
    assert_bits(host(C), refC, "fused GEMM C")
    ref2 = oracle.gelu(refC) if post == 1 else oracle.gelu_backward(X, refC)
    assert_bits(host(C2), ref2, f"fused GEMM C2 post {post}")


# ------------------------------------------------------------------ causal structure (f4)
def test_gemm_causal_skip_scores():
    # causal 1: tiles strictly above the diagonal are not written; every other output
    # equals the full R-GEMM (scores with the 1/sqrt(hd) epilogue, batched heads)
    T, hd, H = 384, 64, 3
    q = synth.uniform(51, (H, T, hd))
    k = synth.uniform(52, (H, T, hd))
    S = torch.full((H, T, T), float("nan"), device="cuda")
    R.repops_gemm_strided_batched(dev(q), dev(k), S, M=T, N=T, K=hd, lda=hd, ldb=hd, ldc=T, sA=(T * hd, 0),
                                  sB=(T * hd, 0), sC=(T * T, 0), batch=(H, 1), transB=True, epi=R.EPI_SCALE,
                                  scale=0.125, causal=1)
    got = host(S)
    for h in range(H):
        ref = oracle.gemm(q[h], k[h], transB=True, epi=2, scale=0.125)
        low = np.tril(np.ones((T, T), bool))
        assert_bits(got[h][low], ref[low], f"causal scores head {h}")
    # the causal softmax of the partially written scores equals the softmax of the full ones
    P = host(R.repops_softmax(S.view(-1, T), causal=True)).reshape(H, T, T)
    for h in range(H):
        assert_bits(P[h], oracle.softmax(oracle.gemm(q[h], k[h], transB=True, epi=2, scale=0.125), causal=True),
                    f"softmax after skipped tiles, head {h}")


def _causal_pv_case(T, hd, H, seed, specials):
    P = np.tril(synth.uniform(seed, (H, T, T)) * np.float32(0.5) + np.float32(0.5)).astype(np.float32)
    P[:, np.triu_indices(T, 1)[0], np.triu_indices(T, 1)[1]] = 0.0  # exactly +0 above the diagonal
    V = synth.uniform(seed + 1, (H, T, hd))
    if specials:
        # columns 0..7 of head 0: every V negative with |v| < 1/2, and rows whose probabilities
        # are 2^-149: each fma(2^-149, v, -0) rounds to -0, so those accumulators are -0
        V[0, :, :8] = (-np.abs(V[0, :, :8]) * np.float32(0.49)).astype(np.float32)
        for r in (0, 5, 64, 70):
            P[0, r, :r + 1] = np.float32(2.0 ** -149)
        V[0, 200, 4] = 0.0                      # a +0 in the skipped range: -0 + +0 -> +0
        V[0, 300, 5] = -0.0                     # a -0 (sign bit set): -0 survives
        V[1, 250, 6] = np.inf                   # non-finite in the skipped range -> NaN
        V[1, 260, 7] = np.nan
    return P, V


@pytest.mark.parametrize("specials", [False, True])
def test_gemm_causal_probabilities_exact(specials):
    # causal 2: each tile's K fold stops at its last row; the skipped fma(+0, v, acc) terms
    # are applied from the suffix flags -- bits equal the oracle's full K fold, including
    # -0 accumulators and non-finite V in the skipped range
    T, hd, H = 320, 64, 2
    P, V = _causal_pv_case(T, hd, H, 61, specials)
    Vd = dev(V)
    fl = R.repops_causal_suffix_flags(Vd, T, hd, hd, (T * hd, 0), (H, 1))
    for cfg in (None,):
        O = torch.empty((H, T, hd), device="cuda")
        R.repops_gemm_strided_batched(dev(P), Vd, O, M=T, N=hd, K=T, lda=T, ldb=hd, ldc=hd, sA=(T * T, 0),
                                      sB=(T * hd, 0), sC=(T * hd, 0), batch=(H, 1), causal=2, kflags=fl, ldf=hd,
                                      sF=((T + 1) * hd, 0))
        got = host(O)
        for h in range(H):
            assert_bits(got[h], oracle.gemm(P[h], V[h]), f"causal PV head {h} specials={specials}")
    if specials:
        ref0 = oracle.gemm(P[0], V[0])
        assert np.any(ref0.view(np.uint32) == 0x80000000)       # the -0 case is exercised
        assert np.isnan(oracle.gemm(P[1], V[1])).any()          # and the non-finite case


def test_causal_suffix_flags_definition():
    K, N = 77, 9
    B = synth.uniform(71, (K, N))
    B[10, 0] = np.inf
    B[:, 1] = -np.abs(B[:, 1]) - np.float32(0.5)
    B[40, 2] = -0.0
    B[:, 3] = 0.0
    B[60, 4] = np.nan
    got = host(R.repops_causal_suffix_flags(dev(B), K, N, N, (0, 0), (1, 1)))[0]
    u = B.view(np.uint32)
    for k in range(K + 1):
        nf = ((u[k:] & 0x7F800000) == 0x7F800000).any(axis=0)
        neg = (u[k:] >> 31).astype(bool).all(axis=0) if k < K else np.ones(N, bool)
        assert np.array_equal(got[k], nf.astype(np.uint8) | (neg.astype(np.uint8) << 1)), k


def _subnormal_operands(M, N, K, tag):
    """operands whose products and partial sums fall in the binary32 subnormal range
    (|x| < 2^-126), so every fma in the K fold rounds with gradual underflow (R9)"""
    A, B = synth.gemm_inputs((M, N, K), tag)
    A = (A * np.float32(2.0 ** -66)).astype(np.float32)      # normal operands ...
    B = (B * np.float32(2.0 ** -66)).astype(np.float32)      # ... subnormal products
    A[::3] = (A[::3] * np.float32(2.0 ** -64)).astype(np.float32)  # subnormal operands in every third row
    A[1, :] = np.float32(2.0 ** -149)                        # the smallest subnormal
    B[:, 2] = -np.float32(2.0 ** -126)                       # the smallest normal
    return A, B


@pytest.mark.parametrize("tA,tB", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_subnormal_operands_and_products(tA, tB):
    M, N, K = 130, 257, 96
    A, B = _subnormal_operands(M, N, K, "gsub")
    assert np.count_nonzero((np.abs(A) < 2.0 ** -126) & (A != 0)) > 1000
    ref = oracle.gemm(A, B)
    tiny = np.abs(ref) < 2.0 ** -126
    assert np.count_nonzero(tiny & (ref != 0)) > M * N // 4  # most results are themselves subnormal
    Ain = np.ascontiguousarray(A.T) if tA else A
    Bin = np.ascontiguousarray(B.T) if tB else B
    ref = oracle.gemm(Ain, Bin, transA=bool(tA), transB=bool(tB))
    for cfg in (None, 0, 3, 6, 10, 19):
        got = R.repops_gemm(dev(Ain), dev(Bin), transA=bool(tA), transB=bool(tB), cfg=cfg)
        assert_bits(host(got), ref, f"subnormal gemm tA{tA} tB{tB} cfg{cfg}")
    # an FTZ implementation would flush these: the oracle result is not the flushed one
    flushed = np.where(np.abs(A) < 2.0 ** -126, np.float32(0), A).astype(np.float32)
    assert not np.array_equal(oracle.gemm(flushed, B).view(np.uint32), oracle.gemm(A, B).view(np.uint32))


def _oracle_rows(args):
    A, B, r0, r1 = args
    return oracle.gemm(A[r0:r1], B)


def oracle_gemm_parallel(A, B, blocks=None):
    """the oracle's full R-GEMM split across host processes by output rows (rows are
    independent, so the bits equal one oracle call)"""
    import multiprocessing as mp
    import os
    n = A.shape[0]
    procs = max(1, min(os.cpu_count() or 1, 64))
    blocks = blocks or procs * 2
    step = (n + blocks - 1) // blocks
    jobs = [(A, B, r, min(n, r + step)) for r in range(0, n, step)]
    with mp.get_context("fork").Pool(procs) as pool:
        return np.concatenate(pool.map(_oracle_rows, jobs))


@pytest.mark.slow
def test_gemm_full_matrix_nn_4096_cfg10():
    # config 2's 4096 point, NN, in the configuration the cost model picks for it (cfg 10,
    # the XP shared-memory transpose): every one of the 16.8 M outputs against the oracle
    n = 4096
    A, B = synth.gemm_inputs(n, "bench")
    got = host(R.repops_gemm(dev(A), dev(B), cfg=10))
    ref = oracle_gemm_parallel(A, B)
    assert_bits(got, ref, "4096 NN cfg10 full matrix")
    assert_bits(host(R.repops_gemm(dev(A), dev(B))), ref, "4096 NN default cfg full matrix")


def test_gemm_epilogues_and_edge_cases():
    A, B = synth.gemm_inputs((70, 90, 45), "ge")
    bias = synth.uniform(5, 90)
    ref = oracle.gemm(A, B, epi=1, bias=bias)
    assert_bits(host(R.repops_gemm(dev(A), dev(B), epi=R.EPI_BIAS, bias=dev(bias))), ref, "bias")
    ref = oracle.gemm(A, B, epi=2, scale=0.125)
    assert_bits(host(R.repops_gemm(dev(A), dev(B), epi=R.EPI_SCALE, scale=0.125)), ref, "scale")
    # K = 0: C = epi(+0)
    Z = R.repops_gemm(torch.empty((3, 0), device="cuda"), torch.empty((0, 4), device="cuda"))
    assert np.all(host(Z).view(np.uint32) == 0)
    # underflow to -0 inside the K fold: K tail must not be zero padded
    a = np.array([[-2.0 ** -80, 2.0 ** -80, 0.0]], np.float32)
    b = np.array([[2.0 ** -80], [0.0], [0.0]], np.float32)
    ref = oracle.gemm(a[:, :2], b[:2])
    assert_bits(host(R.repops_gemm(dev(a[:, :2].copy()), dev(b[:2].copy()))), ref, "neg-zero")
    # NaN / Inf propagate and NaN is canonical
    A2 = A.copy()
    A2[3, 4] = np.inf
    A2[5, 6] = np.nan
    B2 = B.copy()
    B2[7, 8] = 0.0
    ref = oracle.gemm(A2, B2)
    assert_bits(host(R.repops_gemm(dev(A2), dev(B2))), ref, "nan/inf")


def test_gemm_unaligned_leading_dims():
    A, B = synth.gemm_inputs((67, 45, 131), "gu")
    # view with ld = 133 (not a multiple of 4) and an offset start
    big = np.zeros((67, 134), np.float32)
    big[:, 1:132] = A
    tA = dev(big)[:, 1:132]
    ref = oracle.gemm(A, B)
    assert_bits(host(R.repops_gemm(tA, dev(B))), ref, "unaligned")


def test_gemm_strided_batched_attention_layout():
    # QK^T per (sequence, head) inside a packed QKV buffer, as in the GPT-2 step
    Bsz, T, H, hd = 2, 96, 3, 16
    D = H * hd
    qkv = synth.uniform(9, (Bsz * T, 3 * D))
    S = torch.empty((Bsz * H * T, T), device="cuda")
    q = dev(qkv)
    R.repops_gemm_strided_batched(q, q, S, M=T, N=T, K=hd, lda=3 * D, ldb=3 * D, ldc=T,
                                  sA=(T * 3 * D, hd), sB=(T * 3 * D, hd), sC=(H * T * T, T * T),
                                  batch=(Bsz, H), transB=True, epi=R.EPI_SCALE, scale=0.25, offA=0, offB=D)
    got = host(S)
    for b in range(Bsz):
        for h in range(H):
            Q = qkv[b * T:(b + 1) * T, h * hd:(h + 1) * hd]
            K = qkv[b * T:(b + 1) * T, D + h * hd:D + (h + 1) * hd]
            ref = oracle.gemm(Q, K, transB=True, epi=2, scale=0.25)
            assert_bits(got[(b * H + h) * T:(b * H + h + 1) * T], ref, f"batch {b},{h}")


@pytest.mark.parametrize("n", [1024, 2048, 4096, 8192])
def test_gemm_full_size_sampled(n):
    # BASELINE config 2 sizes in the launch configuration bench.py times; the
    # oracle recomputes sampled elements one by one (full K fold each)
    A, B = synth.gemm_inputs(n, "bench")
    got = host(R.repops_gemm(dev(A), dev(B)))
    rng = np.random.default_rng(n)
    idx = [(0, 0), (n - 1, n - 1), (n - 1, 0), (0, n - 1)] + [tuple(x) for x in rng.integers(0, n, (60, 2))]
    for i, j in idx:
        r = oracle.gemm_element(A, B, i, j)
        assert got[i, j].view(np.uint32) == np.float32(r).view(np.uint32), (i, j)


# ------------------------------------------------------------------ reductions
@pytest.mark.parametrize("cols", [1, 5, 127, 128, 129, 768, 4095, 4096, 4097, 50257, 3 * 4096 + 11])
def test_sum_rows_parity(cols):
    x = synth.uniform(synth.seed_for("sr", cols), (9, cols), 3.0)
    x[0, :min(cols, 3)] = -0.0
    ref = oracle.sum_rows(x)
    assert_bits(host(R.repops_sum_rows(dev(x))), ref, f"sum_rows {cols}")


def test_sum_rows_order_pins_on_gpu():
    x = np.ones((1, 4098), np.float32)
    x[0, 0] = 2.0 ** 24
    assert host(R.repops_sum_rows(dev(x)))[0] == 16781282.0
    y = np.zeros((1, 66), np.float32)
    y[0, 0], y[0, 1], y[0, 65] = 2.0 ** 24, 1, 1
    assert host(R.repops_sum_rows(dev(y)))[0] == 16777218.0


def test_sum_cols_seq_parity():
    x = synth.uniform(3, (512 * 4, 333))
    ref = oracle.sum_cols_seq(x, nseg=4)
    assert_bits(host(R.repops_sum_cols_seq(dev(x), nseg=4)), ref, "seq")


@pytest.mark.parametrize("nparts", [1, 2, 4, 8])
def test_tree_sum_parity(nparts):
    parts = [synth.uniform(50 + i, 100003) for i in range(nparts)]
    ref = oracle.tree_sum(parts)
    assert_bits(host(R.repops_tree_sum([dev(p) for p in parts])), ref, f"tree {nparts}")


# ------------------------------------------------------------------ row operators
@pytest.mark.parametrize("rows,cols,causal", [(37, 5, False), (2 * 512, 512, True), (64, 512, False),
                                              (2048, 2048, True), (6, 4096, False), (3, 4097, False),
                                              (3 * 5000, 5000, True),
                                              (2, 50257, False), (4096 * 2, 4096, True)])
def test_softmax_parity(rows, cols, causal):
    if rows * cols > 2 ** 25:
        rows = (2 ** 25 // cols) // cols * cols or cols
    x = synth.uniform(synth.seed_for("sm", rows, cols), (rows, cols), 6.0)
    ref = oracle.softmax(x, causal=causal)
    assert_bits(host(R.repops_softmax(dev(x), causal=causal)), ref, f"softmax {rows}x{cols} c{causal}")


def test_softmax_special_values():
    x = synth.uniform(4, (6, 300), 2.0)
    x[0, 5] = np.nan
    x[1, :] = -np.inf
    x[2, 7] = np.inf
    x[3, :] = 0.0
    x[3, 9] = -0.0
    x[4, 3] = -np.inf
    ref = oracle.softmax(x)
    assert_bits(host(R.repops_softmax(dev(x))), ref, "softmax specials")


@pytest.mark.parametrize("rows,cols", [(96, 512), (13, 77), (4, 5000)])
def test_softmax_backward_parity(rows, cols):
    y = oracle.softmax(synth.uniform(7, (rows, cols), 3.0))
    dy = synth.uniform(8, (rows, cols))
    ref = oracle.softmax_backward(y, dy, scale=0.125)
    assert_bits(host(R.repops_softmax_backward(dev(y), dev(dy), scale=0.125)), ref, "softmax bwd")


@pytest.mark.parametrize("rows,cols", [(64, 768), (33, 100), (5, 4096), (3, 1)])
def test_layernorm_parity(rows, cols):
    x = synth.uniform(1, (rows, cols), 2.0)
    g = synth.uniform(2, cols)
    b = synth.uniform(3, cols)
    y, mean, rstd = oracle.layernorm(x, g, b)
    gy, gm, gr = R.repops_layernorm(dev(x), dev(g), dev(b))
    assert_bits(host(gy), y, "ln y")
    assert_bits(host(gm), mean, "ln mean")
    assert_bits(host(gr), rstd, "ln rstd")
    dy = synth.uniform(4, (rows, cols))
    dres = synth.uniform(5, (rows, cols))
    dx = oracle.layernorm_backward(dy, x, g, mean, rstd, dres=dres)
    assert_bits(host(R.repops_layernorm_backward(dev(dy), dev(x), dev(g), gm, gr, dres=dev(dres))), dx, "ln dx")
    dx0 = oracle.layernorm_backward(dy, x, g, mean, rstd)
    assert_bits(host(R.repops_layernorm_backward(dev(dy), dev(x), dev(g), gm, gr)), dx0, "ln dx nores")
    if rows % 1 == 0:
        nseg = 1 if rows % 4 else 4
        dgm, dbt = oracle.layernorm_backward_params(dy, x, mean, rstd, nseg=nseg)
        gdg, gdb = R.repops_layernorm_backward_params(dev(dy), dev(x), gm, gr, nseg=nseg)
        assert_bits(host(gdg), dgm, "dgamma")
        assert_bits(host(gdb), dbt, "dbeta")


@pytest.mark.parametrize("rows,V", [(8, 4), (16, 1000), (6, 50257), (3, 4097), (2, 55000)])
def test_cross_entropy_parity(rows, V):
    x = synth.uniform(11, (rows, V), 8.0)
    lab = synth.integers(12, rows, V)
    loss, d = oracle.cross_entropy(x, lab, scale=2.0 ** -12)
    gl, gd = R.repops_cross_entropy(dev(x), dev(lab), scale=2.0 ** -12)
    assert_bits(host(gl), loss, "ce loss")
    assert_bits(host(gd), d, "ce grad")
    # in place (dlogits aliasing logits), padded leading dimension
    ld = V + 47
    xp = np.zeros((rows, ld), np.float32)
    xp[:, :V] = x
    t = dev(xp)
    gl2, _ = R.repops_cross_entropy(t, dev(lab), scale=2.0 ** -12, dlogits=t, V=V)
    assert_bits(host(gl2), loss, "ce loss padded")
    assert_bits(host(t)[:, :V], d, "ce grad in place")
    # 16-byte aligned padded rows (the GPT-2 logits layout, ld = V rounded up to 64):
    # the shared-memory-row kernel, in place and out of place
    ld = (V + 63) // 64 * 64
    xp = np.zeros((rows, ld), np.float32)
    xp[:, :V] = x
    t = dev(xp)
    out = torch.zeros_like(t)
    gl3, _ = R.repops_cross_entropy(t, dev(lab), scale=2.0 ** -12, dlogits=out, V=V)
    assert_bits(host(gl3), loss, "ce loss aligned")
    assert_bits(host(out)[:, :V], d, "ce grad aligned")
    gl4, _ = R.repops_cross_entropy(t, dev(lab), scale=2.0 ** -12, dlogits=t, V=V)
    assert_bits(host(gl4), loss, "ce loss aligned in place")
    assert_bits(host(t)[:, :V], d, "ce grad aligned in place")


# ------------------------------------------------------------------ elementwise / math
def _sweep(stride, lo=0, hi=2 ** 32):
    return np.arange(lo, hi, stride, dtype=np.uint64).astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("name", ["exp", "log", "tanh", "rsqrt"])
def test_math_sweep_all_floats(name):
    # a stride-1009 sweep of ALL 2^32 bit patterns (NaNs, infs, subnormals, both signs)
    x = _sweep(1009)
    x = np.concatenate([x, np.float32([0.0, -0.0, np.inf, -np.inf, np.nan, 88.72283172607422,
                                       88.72283935546875, -104.0, -103.99999, 89.0, 1.17549435e-38])])
    ref = getattr(oracle, name)(x)
    got = getattr(R, "repops_" + name)(dev(x))
    assert_bits(host(got), ref, name)


def test_gelu_parity():
    x = np.concatenate([synth.uniform(1, 1000003, 8.0), np.float32([0, -0.0, 30, -30, np.nan, np.inf, -np.inf])])
    assert_bits(host(R.repops_gelu(dev(x))), oracle.gelu(x), "gelu")
    dy = synth.uniform(2, x.size)
    assert_bits(host(R.repops_gelu_backward(dev(x), dev(dy))), oracle.gelu_backward(x, dy), "gelu bwd")


def test_erf_and_exact_gelu_parity():
    # R27: a stride-1009 sweep of all 2^32 patterns plus the branch boundaries (1, 2, 10)
    x = np.concatenate([_sweep(1009), synth.uniform(3, 500003, 6.0),
                        np.float32([0, -0.0, 1.0, -1.0, np.nextafter(np.float32(1), np.float32(2)), 2.0,
                                    np.nextafter(np.float32(2), np.float32(0)), 10.0, -10.0, 9.999999,
                                    np.nan, np.inf, -np.inf, 1e-40, -1e-40])])
    assert_bits(host(R.repops_erf(dev(x))), oracle.erf(x), "erf")
    g = np.concatenate([synth.uniform(4, 1000003, 8.0), np.float32([0, -0.0, 30, -30, np.nan, np.inf, -np.inf])])
    assert_bits(host(R.repops_gelu_erf(dev(g))), oracle.gelu_erf(g), "gelu_erf")
    dy = synth.uniform(5, g.size)
    assert_bits(host(R.repops_gelu_erf_backward(dev(g), dev(dy))), oracle.gelu_erf_backward(g, dy), "gelu_erf bwd")


def test_add_parity():
    a = synth.uniform(1, 100001)
    b = synth.uniform(2, 100001)
    a[:3] = [-0.0, np.nan, np.inf]
    b[:3] = [-0.0, 1.0, -np.inf]
    assert_bits(host(R.repops_add(dev(a), dev(b))), oracle.add(a, b), "add")


def test_embedding_parity():
    V, T, Cc, ntok = 1000, 64, 96, 256
    wte = synth.uniform(1, (V, Cc))
    wpe = synth.uniform(2, (T, Cc))
    tok = synth.integers(3, ntok, 50)  # many repeats
    x0 = oracle.embedding(tok, wte, wpe, T)
    assert_bits(host(R.repops_embedding(dev(tok), dev(wte), dev(wpe), T)), x0, "emb fwd")
    dx0 = synth.uniform(4, (ntok, Cc))
    inc_te = synth.uniform(5, (V, Cc))
    inc_pe = synth.uniform(6, (T, Cc))
    rte, rpe = oracle.embedding_backward(tok, dx0, T, inc_te, inc_pe)
    gte, gpe = dev(inc_te), dev(inc_pe)
    R.repops_embedding_backward(dev(tok), dev(dx0), T, gte, gpe)
    assert_bits(host(gte), rte, "emb bwd wte")
    assert_bits(host(gpe), rpe, "emb bwd wpe")


def test_adamw_parity():
    n = 100003
    p, g = synth.uniform(1, n), synth.uniform(2, n)
    m, v = synth.uniform(3, n, 0.01), np.abs(synth.uniform(4, n, 0.001))
    for step, decay in ((1, True), (7, False), (1000, True)):
        rp, rm, rv = oracle.adamw(p, g, m, v, step, 6e-4, 0.9, 0.95, 1e-8, 0.1, decay)
        tp, tm, tv = dev(p), dev(m), dev(v)
        R.repops_adamw(tp, dev(g), tm, tv, step, 6e-4, 0.9, 0.95, 1e-8, 0.1, decay)
        assert_bits(host(tp), rp, "adam p")
        assert_bits(host(tm), rm, "adam m")
        assert_bits(host(tv), rv, "adam v")


def test_sin_cos_and_rope_tables_exact():
    x = np.concatenate([synth.uniform(51, 200003, 3000.0), synth.uniform(52, 1001, 1e7),
                        np.float32([0.0, -0.0, np.inf, -np.inf, np.nan, 8192.0, 8192.5, 16777215.0, 3e7,
                                    np.pi / 4, -np.pi / 4, 1e-40])])
    assert_bits(host(R.repops_sin(dev(x))), oracle.sin(x), "sin")
    assert_bits(host(R.repops_cos(dev(x))), oracle.cos(x), "cos")
    inv = (500000.0 ** (-np.arange(0, 128, 2, dtype=np.float64) / 128)).astype(np.float32)
    c, s_ = R.repops_rope_tables(dev(inv), 2048)
    rc, rs = oracle.rope_tables_from_inv_freq(inv, 2048)
    assert_bits(host(c), rc, "rope cos")
    assert_bits(host(s_), rs, "rope sin")


def test_adamw_segments_equals_per_tensor_launches():
    sizes = [5, 768, 3, 4097, 64, 1, 1000]
    start = np.concatenate([[0], np.cumsum(sizes)])
    decay = [1, 0, 1, 1, 0, 0, 1]
    n = int(start[-1])
    p, g = synth.uniform(61, n, 0.05), synth.uniform(62, n, 0.01)
    m, v = synth.uniform(63, n, 0.001), np.abs(synth.uniform(64, n, 1e-4))
    for step in (1, 7):
        a = [dev(t) for t in (p, g, m, v)]
        R.repops_adamw_segments(a[0], a[1], a[2], a[3], start, decay, step, 6e-4, 0.9, 0.95, 1e-8, 0.1)
        b = [dev(t) for t in (p, g, m, v)]
        for k in range(len(sizes)):
            sl = slice(int(start[k]), int(start[k + 1]))
            R.repops_adamw(b[0][sl], b[1][sl], b[2][sl], b[3][sl], step, 6e-4, 0.9, 0.95, 1e-8, 0.1, decay[k])
        for x, y in zip(a, b):
            assert np.array_equal(host(x).view(np.uint32), host(y).view(np.uint32))


def test_relu_and_backward_exact():
    x = np.concatenate([synth.uniform(41, 100003, 3.0),
                        np.float32([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45])])
    g = synth.uniform(42, x.size, 2.0)
    assert_bits(host(R.repops_relu(dev(x))), oracle.relu(x), "relu")
    assert_bits(host(R.repops_relu_backward(dev(x), dev(g))), oracle.relu_backward(x, g), "relu_backward")


@pytest.mark.parametrize("rows,cols", [(1, 1), (64, 64), (130, 67), (256, 1000), (4096, 77)])
def test_transpose_exact(rows, cols):
    # data movement only: y = x^T bit for bit, contiguous (16-byte path) and strided views
    x = synth.uniform(31, (rows, cols + 5))
    xs = np.ascontiguousarray(x[:, :cols])
    got = R.repops_transpose(dev(xs))
    assert np.array_equal(host(got).view(np.uint32), xs.T.view(np.uint32))
    big = torch.zeros((cols, rows + 8), device="cuda")
    R.repops_transpose(dev(x)[:, 1:cols + 1], out=big[:, 3:rows + 3])  # misaligned views: scalar path
    b = host(big)
    assert np.array_equal(b[:, 3:rows + 3].view(np.uint32), x[:, 1:cols + 1].T.view(np.uint32))
    assert np.all(b[:, :3] == 0) and np.all(b[:, rows + 3:] == 0)


# ------------------------------------------------------------------ Verde commitments
def test_commit_parity_and_batching():
    shapes = [(0,), (1,), (1023,), (1024,), (1025,), (3, 4096), (257, 1000), (4096 * 70 + 3,), (5, 7, 11)]
    arrs = [synth.uniform(synth.seed_for("cm", s), s) for s in shapes]
    refs = [oracle.commit_tensor(a) for a in arrs]
    ts = [dev(a) for a in arrs]
    ws = R.CommitWorkspace()
    digs = host(R.verde_commit_tensors(ts, ws=ws))
    for i, r in enumerate(refs):
        assert digs[i].tobytes() == r, shapes[i]
    # one at a time gives the same digests
    for t, r in zip(ts, refs):
        assert host(R.verde_commit_tensor(t, ws=ws)).tobytes() == r


def test_commit_reduce_group_boundaries():
    """chunk counts around the reduce kernel's 8-node thread blocks and 1024-node CTA
    groups (ragged last block, ragged last group, one node over) match the oracle's
    RFC 6962 tree"""
    counts = [2, 3, 7, 8, 9, 15, 17, 1023, 1024, 1025, 1031, 2047, 2049, 8 * 1024 + 3]
    arrs = [synth.uniform(900 + c, c * 1024 - (c % 3) * 7) for c in counts]   # c chunks, last one short
    ts = [dev(a) for a in arrs]
    digs = host(R.verde_commit_tensors(ts, ws=R.CommitWorkspace()))
    for i, a in enumerate(arrs):
        assert digs[i].tobytes() == oracle.commit_tensor(a), counts[i]


def test_commit_large_tensor_multi_pass():
    # > 256*256 leaves -> three reduce passes (logits-sized tensors)
    a = synth.uniform(77, 256 * 256 * 1024 + 12345)  # 268 MB
    t = dev(a)
    got = host(R.verde_commit_tensor(t)).tobytes()
    assert got == oracle.commit_tensor(a)
    R.repops_flip_bit(t, 12345678, 0)
    b = a.copy()
    b.view(np.uint32)[12345678] ^= 1
    got2 = host(R.verde_commit_tensor(t)).tobytes()
    assert got2 == oracle.commit_tensor(b) and got2 != got


def _dirty_ref(rows, row_bytes, nbytes):
    nch = (nbytes + 4095) // 4096
    f = np.zeros(nch, np.uint8)
    for r in rows:
        for c in range(r * row_bytes // 4096, ((r + 1) * row_bytes - 1) // 4096 + 1):
            if c < nch:
                f[c] = 1
    return f


@pytest.mark.parametrize("shape", [(50257, 768), (1000, 100), (37, 1024), (5, 3)])
def test_incremental_commit_equals_full(shape):
    """verde_dirty_chunks flags exactly the 4 KiB chunks the given rows meet (rows straddling
    chunk edges, duplicates, first / last row); an incremental commit (clean chunk leaves taken
    from an earlier commit's leaves_out) of the tensor with those rows rewritten has the full
    commit's digest, which is the oracle's; with no rows it is the base digest"""
    R_, Cc = shape
    a = synth.uniform(synth.seed_for("inc", shape), shape)
    t = dev(a)
    nb = a.nbytes
    nch = (nb + 4095) // 4096
    leaves = torch.empty(nch * 32, dtype=torch.uint8, device="cuda")
    dig = torch.zeros((2, 32), dtype=torch.uint8, device="cuda")
    R.CommitPlan([t], [dig[0]], incremental={0: dict(leaves_out=leaves)}).run()
    assert host(dig[0]).tobytes() == oracle.commit_tensor(a)
    rng = np.random.default_rng(R_)
    rows = sorted(set([0, R_ - 1, R_ // 2, R_ // 2] + rng.integers(0, R_, min(40, R_)).tolist()))
    rows_l = rows + rows[:3]                                   # duplicates
    b = a.copy()
    b[rows] += np.float32(1.0)
    t.copy_(torch.from_numpy(b))
    dirty = torch.full((nch,), 7, dtype=torch.uint8, device="cuda")
    rr = torch.tensor(rows_l, dtype=torch.int32, device="cuda")
    R.verde_dirty_chunks(rr, Cc * 4, nb, dirty)
    assert np.array_equal(host(dirty), _dirty_ref(rows_l, Cc * 4, nb))
    plan = R.CommitPlan([t], [dig[1]], incremental={0: dict(base_leaves=leaves, dirty=dirty)})
    plan.run()
    assert host(dig[1]).tobytes() == oracle.commit_tensor(b) == host(R.verde_commit_tensor(t)).tobytes()
    R.verde_dirty_chunks(None, Cc * 4, nb, dirty, all_chunks=True)   # full re-hash mode
    assert int(host(dirty).min()) == 1
    plan.run()
    assert host(dig[1]).tobytes() == oracle.commit_tensor(b)
    R.verde_dirty_chunks(rr[:0], Cc * 4, nb, dirty)                 # no rows: every leaf reused
    assert int(host(dirty).max()) == 0
    t.copy_(torch.from_numpy(a))
    plan.run()
    assert host(dig[1]).tobytes() == oracle.commit_tensor(a)


def test_incremental_commit_rejects():
    t = torch.zeros(2048, device="cuda")
    d = torch.zeros(32, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        R.CommitPlan([t], [d], incremental={0: dict(base_leaves=torch.zeros(64, dtype=torch.uint8,
                                                                              device="cuda"))})
    with pytest.raises(ValueError):   # leaves_out too small for 2 chunks
        R.CommitPlan([t], [d], incremental={0: dict(leaves_out=torch.zeros(32, dtype=torch.uint8, device="cuda"))})


# ------------------------------------------------------------------ peer-memory combine (f1)
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_p2p_tree_combine_equals_tree_sum(G):
    """the fused combine over any slicing gives repops_tree_sum's bits (and the oracle's)
    in every output buffer; unaligned slices take the scalar path"""
    from paper_2502_19405_b200.dist import p2p_slice
    n = 100003
    parts_h = [synth.uniform(700 + q, n) for q in range(G)]
    parts = [dev(p) for p in parts_h]
    ref = oracle.tree_sum(parts_h)
    assert_bits(host(R.repops_tree_sum(parts)), ref, "tree_sum")
    outs = [torch.full((n,), float("nan"), device="cuda") for _ in range(G)]
    for r in range(G):
        lo, hi = p2p_slice(r, G, n)
        R.repops_p2p_tree_combine(parts, lo, hi, outs)
    for q in range(G):
        assert_bits(host(outs[q]), ref, f"out {q}")
    outs2 = [torch.zeros(n, device="cuda") for _ in range(G)]
    for lo, hi in ((0, 7), (7, 1001), (1001, n)):   # unaligned slice starts
        R.repops_p2p_tree_combine(parts, lo, hi, outs2)
    for q in range(G):
        assert_bits(host(outs2[q]), ref, f"unaligned out {q}")


@pytest.mark.parametrize("G", [2, 4])
def test_p2p_flag_protocol_virtual_ranks(G):
    """the device signal / wait protocol of P2PTreeCombine with G virtual ranks in one
    process, each on its own stream (so their kernels run concurrently): 3 epochs,
    every rank's gradient buffer equals the tree over all partials, no wait times out"""
    from paper_2502_19405_b200.dist import p2p_slice
    n = 65537
    streams = [torch.cuda.Stream() for _ in range(G)]
    partial = [torch.zeros(n, device="cuda") for _ in range(G)]
    grad = [torch.zeros(n, device="cuda") for _ in range(G)]
    flags = [torch.zeros(2 * G, dtype=torch.int32, device="cuda") for _ in range(G)]
    ready = [f[:G] for f in flags]
    done = [f[G:] for f in flags]
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    for epoch in (1, 2, 3):
        src = [dev(synth.uniform(800 + 10 * epoch + r, n)) for r in range(G)]
        torch.cuda.synchronize()
        for r in range(G):
            s = streams[r]
            with torch.cuda.stream(s):
                partial[r].copy_(src[r])
                R.repops_p2p_signal(ready, r, epoch, stream=s)
                R.repops_p2p_wait(ready[r], G, epoch, 10000, status, stream=s)
                lo, hi = p2p_slice(r, G, n)
                R.repops_p2p_tree_combine(partial, lo, hi, grad, stream=s, status=status)
                R.repops_p2p_signal(done, r, epoch, stream=s)
                R.repops_p2p_wait(done[r], G, epoch, 10000, status, stream=s)
        torch.cuda.synchronize()
        assert int(status.item()) == 0, "a wait timed out"
        ref = oracle.tree_sum([host(t) for t in src])
        for r in range(G):
            assert_bits(host(grad[r]), ref, f"epoch {epoch} rank {r}")


def test_p2p_wait_timeout_blocks_the_combine():
    """a peer that never signals: the bounded wait records the timeout in the status
    word and the combine launched behind it stores nothing (ADVICE: no stale partials
    reach any gradient buffer); P2P-style check() then raises"""
    G, n = 2, 4099
    flags = torch.zeros(G, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    parts = [dev(synth.uniform(900 + q, n)) for q in range(G)]
    grad = [torch.full((n,), 7.0, device="cuda") for _ in range(G)]
    R.repops_p2p_signal([flags], 0, 1)                     # only slot 0 ever signals
    R.repops_p2p_wait(flags, G, 1, 50, status)             # 50 ms, slot 1 never arrives
    R.repops_p2p_tree_combine(parts, 0, n, grad, status=status)
    torch.cuda.synchronize()
    assert int(status.item()) == 1
    for q in range(G):
        assert torch.all(grad[q] == 7.0), "combine stored after a timed-out wait"
    status.zero_()
    R.repops_p2p_tree_combine(parts, 0, n, grad, status=status)   # status clear: it runs
    assert_bits(host(grad[1]), oracle.tree_sum([host(p) for p in parts]), "after reset")


# ------------------------------------------------------------------ deterministic pseudorandomness (R28)
@pytest.mark.parametrize("n", [1, 3, 4, 4097, 1_000_003])
def test_rand_uniform_exact(n):
    for seed, stream in ((0, 0), (0x0123456789ABCDEF, 0x0000000500000007), (2 ** 64 - 1, 2 ** 64 - 1)):
        assert_bits(host(R.repops_rand_uniform(seed, stream, n)), oracle.rand_uniform(seed, stream, n),
                    f"uniform n={n} seed={seed:x}")


def test_dropout_exact_and_backward():
    x = np.concatenate([synth.uniform(901, 1_000_001, 4.0), np.float32([np.nan, np.inf, -np.inf, -0.0, 3e38])])
    dy = synth.uniform(902, x.size)
    for p in (0.0, 0.1, 0.5, 0.9, 1.0):
        ry, rm = oracle.dropout(x, p, 77, 5)
        mask = torch.empty(x.size, dtype=torch.uint8, device="cuda")
        y, _ = R.repops_dropout(dev(x), p, 77, 5, mask=mask)
        assert_bits(host(y), ry, f"dropout p={p}")
        assert np.array_equal(host(mask), rm), f"mask p={p}"
        assert_bits(host(R.repops_dropout_backward(dev(dy), p, 77, 5)), oracle.dropout_backward(dy, p, 77, 5),
                    f"dropout bwd p={p}")
    # unaligned views take the scalar path with the same bits
    xt = dev(x)
    y, _ = R.repops_dropout(xt[1:], 0.3, 5, 6)
    assert_bits(host(y), oracle.dropout(x[1:], 0.3, 5, 6)[0], "dropout unaligned")


# ------------------------------------------------------------------ R30 stored precision
def _u16(t):
    return host(t.view(torch.int16)).view(np.uint16)


@pytest.mark.parametrize("dt", ["bf16", "f16"])
def test_convert_exact_all_patterns(dt):
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16}[dt]
    x = np.concatenate([_sweep(1009), np.float32([0.0, -0.0, 65504, 65520, 65519.996, 2 ** -24, 2 ** -25,
                                                  3 * 2 ** -25, 1 + 2 ** -11, 1 + 2 ** -8, 3.3895314e38, np.nan])])
    n = _u16(R.repops_convert(dev(x), tdt))
    assert np.array_equal(n, oracle.convert(x[None], "f32", dt).ravel()), f"narrow {dt}"
    h = np.arange(2 ** 16, dtype=np.uint32).astype(np.uint16)
    w = R.repops_convert(torch.from_numpy(h.view(np.int16)).cuda().view(tdt), torch.float32)
    assert_bits(host(w), oracle.convert(h[None], dt, "f32").ravel(), f"widen {dt}")
    # 2-D strided views (leading dimensions) and a cross-format conversion
    X = dev(synth.uniform(41, 37 * 50, 100.0).reshape(37, 50))[:, 3:44]
    Y = R.repops_convert(X, tdt)
    assert np.array_equal(_u16(Y), oracle.convert(host(X).copy(), "f32", dt))
    other, odt = ("f16", torch.float16) if dt == "bf16" else ("bf16", torch.bfloat16)
    Z = R.repops_convert(Y, odt)
    assert np.array_equal(_u16(Z), oracle.convert(_u16(Y), dt, other))


@pytest.mark.parametrize("adt,bdt,cdt", [("bf16", "bf16", "bf16"), ("f16", "f16", "f32"), ("f32", "bf16", "f16"),
                                         ("f32", "f32", "f32")])
def test_gemm_ex_parity(adt, bdt, cdt):
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}
    M, N, K = 131, 257, 300
    for tA, tB in ((False, False), (True, False), (False, True)):
        A32 = synth.uniform(51, M * K).reshape((K, M) if tA else (M, K))
        B32 = synth.uniform(52, K * N).reshape((N, K) if tB else (K, N))
        A = A32 if adt == "f32" else oracle.convert(A32, "f32", adt)
        B = B32 if bdt == "f32" else oracle.convert(B32, "f32", bdt)
        bias = synth.uniform(53, N)
        ref = oracle.gemm_ex(A, adt, B, bdt, cdt, transA=tA, transB=tB, epi=1, bias=bias)

        def to_dev(a, dt):
            return dev(a) if dt == "f32" else torch.from_numpy(a.view(np.int16)).cuda().view(tdt[dt])
        C = R.repops_gemm_ex(to_dev(A, adt), to_dev(B, bdt), transA=tA, transB=tB, epi=R.EPI_BIAS, bias=dev(bias),
                             out_dtype=tdt[cdt])
        got = host(C) if cdt == "f32" else _u16(C)
        if cdt == "f32":
            assert_bits(got, ref, f"gemm_ex {adt}{bdt}{cdt} tA={tA} tB={tB}")
        else:
            assert np.array_equal(got, ref), f"gemm_ex {adt}{bdt}{cdt} tA={tA} tB={tB}"
    if (adt, bdt, cdt) == ("f32", "f32", "f32"):   # all-f32 gemm_ex is repops_gemm bit for bit
        A, B = dev(synth.uniform(54, M * K).reshape(M, K)), dev(synth.uniform(55, K * N).reshape(K, N))
        assert_bits(host(R.repops_gemm_ex(A, B)), host(R.repops_gemm(A, B)), "gemm_ex == gemm")


# ------------------------------------------------------------------ fused attention forward (f4)
def _attn_inputs(S_, H, T, hd, seed):
    d = H * hd
    return synth.uniform(seed, (S_ * T, 3 * d), 2.0)


@pytest.mark.parametrize("causal", [True, False])
def test_attention_fwd_equals_unfused_and_oracle(causal):
    """S, P and O of the fused kernel equal the three unfused calls bit for bit (every
    head of a GPT-2-shaped layer) and the oracle composition (sampled heads)"""
    S_, H, T, hd = 2, 12, 512, 64
    d = H * hd
    qkv_h = _attn_inputs(S_, H, T, hd, 31)
    qkv = dev(qkv_h)
    scale = 1.0 / np.sqrt(hd)
    Sf = torch.empty(S_ * H * T, T, device="cuda")
    Pf = torch.empty_like(Sf)
    Of = torch.empty(S_ * T, d, device="cuda")
    assert R.repops_attention_fwd_supported(T, hd)
    R.repops_attention_fwd(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, 2 * d, (S_, H), Of, d, (T * d, hd), S=Sf, P=Pf,
                           sp=(H * T * T, T * T), scale=scale, causal=causal)
    Su = torch.empty_like(Sf)
    Pu = torch.empty_like(Sf)
    Ou = torch.empty_like(Of)
    R.repops_gemm_strided_batched(qkv, qkv, Su, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T, sA=(T * 3 * d, hd),
                                  sB=(T * 3 * d, hd), sC=(H * T * T, T * T), batch=(S_, H), transB=True,
                                  epi=R.EPI_SCALE, scale=scale, offB=d)
    R.repops_softmax(Su, causal=causal, out=Pu)
    R.repops_gemm_strided_batched(Pu, qkv, Ou, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d, sA=(H * T * T, T * T),
                                  sB=(T * 3 * d, hd), sC=(T * d, hd), batch=(S_, H), offB=2 * d)
    assert_bits(host(Sf), host(Su), "S fused vs unfused")
    assert_bits(host(Pf), host(Pu), "P fused vs unfused")
    assert_bits(host(Of), host(Ou), "O fused vs unfused")
    Ph, Oh = host(Pf), host(Of)
    for s_, h in ((0, 0), (1, 11)):
        q = np.ascontiguousarray(qkv_h[s_ * T:(s_ + 1) * T, h * hd:(h + 1) * hd])
        k = np.ascontiguousarray(qkv_h[s_ * T:(s_ + 1) * T, d + h * hd:d + (h + 1) * hd])
        v = np.ascontiguousarray(qkv_h[s_ * T:(s_ + 1) * T, 2 * d + h * hd:2 * d + (h + 1) * hd])
        s_ref = oracle.gemm(q, k, transB=True, epi=2, scale=scale)
        p_ref = oracle.softmax(s_ref, causal=causal)
        o_ref = oracle.gemm(p_ref, v)
        r0 = (s_ * H + h) * T
        assert_bits(Ph[r0:r0 + T], p_ref, f"P oracle s{s_} h{h}")
        assert_bits(Oh[s_ * T:(s_ + 1) * T, h * hd:(h + 1) * hd], o_ref, f"O oracle s{s_} h{h}")


def test_attention_fwd_optional_outputs_and_shapes():
    S_, H, T, hd = 1, 2, 256, 64
    d = H * hd
    qkv = dev(_attn_inputs(S_, H, T, hd, 32))
    O1 = torch.empty(T, d, device="cuda")
    O2 = torch.empty(T, d, device="cuda")
    P = torch.empty(H * T, T, device="cuda")
    R.repops_attention_fwd(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, 2 * d, (S_, H), O1, d, (T * d, hd), P=P,
                           sp=(H * T * T, T * T), scale=0.125)
    R.repops_attention_fwd(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, 2 * d, (S_, H), O2, d, (T * d, hd),
                           scale=0.125)   # neither S nor P stored: same O
    assert_bits(host(O1), host(O2), "O with / without P")
    assert not R.repops_attention_fwd_supported(512, 128)
    assert not R.repops_attention_fwd_supported(100, 64)
    with pytest.raises(R.RepopsError):
        R.repops_attention_fwd(qkv, 100, hd, 3 * d, (T * 3 * d, hd), 0, d, 2 * d, (S_, H), O1, d, (T * d, hd))


def _unfused_attention(qkv, S_, H, T, hd, scale, causal=True):
    d = H * hd
    Su = torch.empty(S_ * H * T, T, device="cuda")
    Pu = torch.empty_like(Su)
    Ou = torch.empty(S_ * T, d, device="cuda")
    R.repops_gemm_strided_batched(qkv, qkv, Su, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T, sA=(T * 3 * d, hd),
                                  sB=(T * 3 * d, hd), sC=(H * T * T, T * T), batch=(S_, H), transB=True,
                                  epi=R.EPI_SCALE, scale=scale, offB=d)
    R.repops_softmax(Su, causal=causal, out=Pu)
    R.repops_gemm_strided_batched(Pu, qkv, Ou, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d, sA=(H * T * T, T * T),
                                  sB=(T * 3 * d, hd), sC=(T * d, hd), batch=(S_, H), offB=2 * d)
    return Pu, Ou


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
@pytest.mark.parametrize("T", [512, 256, 128])
def test_attention_fwd_causal_skip_equals_full(variant, T, monkeypatch):
    """S not stored + causal (R29 scratch scores): the fused kernel computes only the key
    chunks its rows read and applies the skipped fma(+0, V, acc) terms of the PV fold in
    closed form (R31) -- P and O bit-identical to the full unfused composition, including
    non-finite V entries in every row block's skipped suffix (each must turn that column
    of every earlier row into NaN, as the full fold does) and signed zeros there"""
    monkeypatch.setenv("REPOPS_ATTN_VARIANT", str(variant))
    S_, H, hd = 2, 12, 64
    d = H * hd
    qkv_h = _attn_inputs(S_, H, T, hd, 33 + T)
    # V of (shard 0, head 1): +inf in the last row, column 5; NaN at row T-65, column 17;
    # a column of -0 / +0 suffixes (column 30) and all-negative suffixes (column 31)
    v0 = 2 * d + 1 * hd
    qkv_h[T - 1, v0 + 5] = np.inf
    qkv_h[T - 65, v0 + 17] = np.nan
    qkv_h[T // 2:T, v0 + 30] = -0.0
    qkv_h[T // 2:T, v0 + 31] = -np.abs(qkv_h[T // 2:T, v0 + 31])
    # (shard 1, head 11): -inf at row 64 (inside the second chunk), column 63
    qkv_h[T + 64, 2 * d + 11 * hd + 63] = -np.inf
    qkv = dev(qkv_h)
    scale = 1.0 / np.sqrt(hd)
    Pf = torch.full((S_ * H * T, T), 7.0, device="cuda")   # the kernel writes every element
    Of = torch.empty(S_ * T, d, device="cuda")
    R.repops_attention_fwd(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, 2 * d, (S_, H), Of, d, (T * d, hd), P=Pf,
                           sp=(H * T * T, T * T), scale=scale, causal=True)
    Pu, Ou = _unfused_attention(qkv, S_, H, T, hd, scale)
    assert_bits(host(Pf), host(Pu), "P skip vs full")
    Oh = host(Of)
    assert_bits(Oh, host(Ou), "O skip vs full")
    assert np.isnan(Oh[:T - 1, hd + 5]).all() and np.isnan(Oh[:T - 64, hd + 17]).all()
    O2 = torch.empty_like(Of)   # neither S nor P stored
    R.repops_attention_fwd(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, 2 * d, (S_, H), O2, d, (T * d, hd),
                           scale=scale, causal=True)
    assert_bits(host(O2), Oh, "O without P")


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("T", [512, 1024, 256, 96, 32])
def test_attention_probs_equals_unfused_and_oracle(T, causal):
    """scores + softmax fused (the scores never leave shared memory; causal: only the key
    blocks a row block reads): P bit-identical to R-GEMM(SCALE) -> R-SOFTMAX for every
    (shard, head) -- T = 96 / 32 are ragged against the 256-key blocks -- and to the oracle
    on sampled heads; every element of P is written (masked +0)"""
    S_, H, hd = 2, 12 if T <= 512 else 3, 64
    d = H * hd
    qkv_h = _attn_inputs(S_, H, T, hd, 40 + T + causal)
    # large scores (exp underflow to +0 for most of a row), a -inf and a NaN score source
    qkv_h[5, 0:hd] *= 64.0
    qkv_h[T + 7, d + 3 * hd + 1] = -np.inf
    qkv_h[2, 5 * hd + 9] = np.nan
    qkv = dev(qkv_h)
    scale = 1.0 / np.sqrt(hd)
    Pf = torch.full((S_ * H * T, T), 7.0, device="cuda")
    assert R.repops_attention_probs_supported(T, hd)
    R.repops_attention_probs(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, (S_, H), Pf, (H * T * T, T * T),
                             scale=scale, causal=causal)
    Pu, _ = _unfused_attention(qkv, S_, H, T, hd, scale, causal=causal)
    Ph = host(Pf)
    assert_bits(Ph, host(Pu), "P fused vs unfused")
    for s_, h in ((0, 0), (1, H - 1)):
        q = np.ascontiguousarray(qkv_h[s_ * T:(s_ + 1) * T, h * hd:(h + 1) * hd])
        k = np.ascontiguousarray(qkv_h[s_ * T:(s_ + 1) * T, d + h * hd:d + (h + 1) * hd])
        p_ref = oracle.softmax(oracle.gemm(q, k, transB=True, epi=2, scale=scale), causal=causal)
        r0 = (s_ * H + h) * T
        assert_bits(Ph[r0:r0 + T], p_ref, f"P oracle s{s_} h{h}")


def test_attention_probs_rejects():
    qkv = torch.zeros(64, 3 * 64, device="cuda")
    P = torch.zeros(64, 64, device="cuda")
    assert not R.repops_attention_probs_supported(64, 96)
    assert not R.repops_attention_probs_supported(100, 64)
    assert not R.repops_attention_probs_supported(4096, 64)
    assert not R.repops_attention_probs_supported(4096, 128) and not R.repops_attention_probs_supported(40, 128)
    with pytest.raises(R.RepopsError):
        R.repops_attention_probs(qkv, 64, 96, 3 * 64, (0, 0), 0, 64, (1, 1), P, (0, 0))
    with pytest.raises(ValueError):
        R.repops_attention_probs(qkv, 128, 64, 3 * 64, (0, 0), 0, 64, (1, 1), P, (0, 0))  # P too small


@pytest.mark.parametrize("T", [512, 1024, 256, 96, 32])
def test_attention_dscores_equals_unfused_and_oracle(T):
    """backward scores part fused (dP kept in shared memory): dS bit-identical to
    R-GEMM(dO, V^T) -> R-SOFTMAX-BWD(P, dP, scale) for every (shard, head), with the causal
    P of the forward (+0 above the diagonal), non-finite dO / V entries (their dP columns /
    rows are inf / NaN, and the masked +0 * inf terms of the row fold give NaN), and the
    oracle on sampled heads"""
    S_, H, hd = 2, 12 if T <= 512 else 3, 64
    d = H * hd
    scale = 1.0 / np.sqrt(hd)
    qkv_h = _attn_inputs(S_, H, T, hd, 60 + T)
    h2, h4, h5 = 2 % H, 4 % H, 5 % H
    qkv_h[T - 3, 2 * d + h2 * hd + 7] = np.inf          # V of (0, h2): key T-3 -> dP column T-3 inf
    qkv_h[T + 1, 2 * d + h4 * hd + 11] = np.nan         # V of (1, h4): key 1 -> dP column 1 NaN
    dO_h = synth.uniform(61 + T, (S_ * T, d), 1.0)
    dO_h[7, h5 * hd + 3] = -np.inf                       # dO of (0, h5): row 7 -> dP row 7 inf / NaN
    qkv, dO = dev(qkv_h), dev(dO_h)
    Pu, _ = _unfused_attention(qkv, S_, H, T, hd, scale, causal=True)
    sp = (H * T * T, T * T)
    dSf = torch.full_like(Pu, 7.0)
    R.repops_attention_dscores(dO, qkv, T, hd, d, (T * d, hd), 0, 3 * d, (T * 3 * d, hd), 2 * d, Pu, sp, dSf, sp,
                               (S_, H), scale=scale)
    dPu = torch.empty_like(Pu)
    R.repops_gemm_strided_batched(dO, qkv, dPu, M=T, N=T, K=hd, lda=d, ldb=3 * d, ldc=T, sA=(T * d, hd),
                                  sB=(T * 3 * d, hd), sC=sp, batch=(S_, H), transB=True, offB=2 * d)
    dSu = torch.empty_like(Pu)
    R.repops_softmax_backward(Pu, dPu, scale=scale, out=dSu)
    dSh = host(dSf)
    assert_bits(dSh, host(dSu), "dS fused vs unfused")
    assert np.isnan(dSh[(0 * H + h5) * T + 7]).all()     # the row with -inf in dO
    Ph = host(Pu)
    for s_, h in ((0, h2), (1, h4), (1, H - 1)):
        v = np.ascontiguousarray(qkv_h[s_ * T:(s_ + 1) * T, 2 * d + h * hd:2 * d + (h + 1) * hd])
        g = np.ascontiguousarray(dO_h[s_ * T:(s_ + 1) * T, h * hd:(h + 1) * hd])
        r0 = (s_ * H + h) * T
        ref = oracle.softmax_backward(Ph[r0:r0 + T], oracle.gemm(g, v, transB=True), scale=scale)
        assert_bits(dSh[r0:r0 + T], ref, f"dS oracle s{s_} h{h}")


def test_attention_dscores_rejects():
    x = torch.zeros(64, 3 * 64, device="cuda")
    P = torch.zeros(64, 64, device="cuda")
    with pytest.raises(R.RepopsError):
        R.repops_attention_dscores(x, x, 64, 128, 3 * 64, (0, 0), 0, 3 * 64, (0, 0), 0, P, (0, 0), P, (0, 0), (1, 1))
    with pytest.raises(ValueError):   # dS too small for T = 128
        R.repops_attention_dscores(x, x, 128, 64, 3 * 64, (0, 0), 0, 3 * 64, (0, 0), 0, P, (0, 0), P, (0, 0), (1, 1))


@pytest.mark.parametrize("T,causal", [(2048, True), (256, True), (48, True), (96, False)])
def test_attention_probs_hd128_grouped_query(T, causal):
    """hd = 128 (Llama): 16-row blocks, 512-key blocks; the Llama prefill's layout -- per
    column block j a [T][(qh + 1) hd] buffer of qh query heads and one shared key head
    (K batch stride 0 across the query heads) -- P bit-identical to the causal-skip scores
    R-GEMM + R-SOFTMAX of the prefill and to the oracle on sampled heads; T = 48 is ragged
    against the 512-key blocks"""
    nbl, qh, hd = 2 if T == 2048 else 3, 4, 128
    W2 = (qh + 1) * hd
    qk_h = synth.uniform(90 + T, (nbl * T, W2), 1.0)
    qk_h[3, 0:hd] *= 40.0                            # a row whose exps mostly underflow
    qk_h[T + 5, qh * hd + 7] = np.inf                # key 5 of block 1: +-inf / NaN scores
    qk = dev(qk_h)
    scale = float(np.float32(1.0 / np.sqrt(hd)))
    sp = (qh * T * T, T * T)
    Pf = torch.full((nbl * qh * T, T), 7.0, device="cuda")
    assert R.repops_attention_probs_supported(T, hd)
    R.repops_attention_probs(qk, T, hd, W2, (T * W2, hd), 0, qh * hd, (nbl, qh), Pf, sp, scale=scale, causal=causal,
                             sk=(T * W2, 0))
    Su = torch.full_like(Pf, 5.0)
    R.repops_gemm_strided_batched(qk, qk, Su, M=T, N=T, K=hd, lda=W2, ldb=W2, ldc=T, sA=(T * W2, hd),
                                  sB=(T * W2, 0), sC=sp, batch=(nbl, qh), transB=True, epi=R.EPI_SCALE, scale=scale,
                                  offB=qh * hd, causal=1 if causal else 0)
    Pu = R.repops_softmax(Su, causal=causal)
    Ph = host(Pf)
    assert_bits(Ph, host(Pu), "P fused vs unfused (hd 128)")
    for j, h in ((0, 0), (nbl - 1, qh - 1), (1, 2)):
        q = np.ascontiguousarray(qk_h[j * T:(j + 1) * T, h * hd:(h + 1) * hd])
        k = np.ascontiguousarray(qk_h[j * T:(j + 1) * T, qh * hd:(qh + 1) * hd])
        ref = oracle.softmax(oracle.gemm(q, k, transB=True, epi=2, scale=scale), causal=causal)
        r0 = (j * qh + h) * T
        assert_bits(Ph[r0:r0 + T], ref, f"P oracle block {j} head {h}")


def test_sha256_probe_deterministic():
    """the commitment-ceiling diagnostic runs, is deterministic, and reports a rate"""
    from paper_2502_19405_b200._lib import check, lib
    out = [torch.zeros(4 * 128, dtype=torch.int32, device="cuda") for _ in range(2)]
    for o in out:
        check(lib().verde_sha256_probe(4, 10, o.data_ptr(), None), "probe")
    assert torch.equal(out[0], out[1]) and int(out[0].abs().sum()) > 0
    assert R.verde_sha256_probe_gbs(ctas_per_sm=1, iters=20) > 0


def test_ffma2_probe_deterministic():
    """the R-GEMM ceiling diagnostic runs, is deterministic, and reports a rate"""
    from paper_2502_19405_b200._lib import check, lib
    out = [torch.zeros(4 * 128, device="cuda") for _ in range(2)]
    for o in out:
        check(lib().repops_ffma2_probe(4, 10, o.data_ptr(), None), "probe")
    assert torch.equal(out[0].view(torch.int32), out[1].view(torch.int32))
    assert R.repops_ffma2_probe_tflops(ctas_per_sm=1, iters=100) > 0
