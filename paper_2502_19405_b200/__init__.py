"""B200-native RepOps / Verde hot path (arXiv 2502.19405).

Thin Python binding over librepops.so (include/repops.h).  Each function has
the name of the C entry point it calls and only marshals arguments: torch
supplies device memory and the current CUDA stream, every arithmetic step runs
in the library's CUDA kernels.  Functions take torch CUDA tensors (float32
unless stated) and return the output tensor(s).
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import Node, RepopsError, TensorDesc, check, header_symbols, lib

EPI_NONE, EPI_BIAS, EPI_SCALE = 0, 1, 2
F32, I32, U8, BF16, F16 = 1, 2, 3, 4, 5
_DT = {torch.float32: F32, torch.int32: I32, torch.uint8: U8, torch.bfloat16: BF16, torch.float16: F16}

__all__ = [
    "repops_gemm", "repops_gemm_post", "repops_gemm_strided_batched", "repops_causal_suffix_flags", "repops_copy2d_batched", "repops_sum_rows", "repops_sum_cols_seq", "repops_tree_sum",
    "repops_softmax", "repops_softmax_backward", "repops_layernorm", "repops_layernorm_backward",
    "repops_layernorm_backward_params", "repops_cross_entropy", "repops_exp", "repops_log", "repops_tanh",
    "repops_rsqrt", "repops_gelu", "repops_gelu_backward", "repops_relu", "repops_relu_backward", "repops_sin", "repops_cos", "repops_erf", "repops_gelu_erf", "repops_convert", "repops_gemm_ex",
    "repops_attention_fwd", "repops_attention_fwd_supported", "repops_attention_probs",
    "repops_attention_probs_supported", "repops_attention_dscores", "verde_dirty_chunks", "repops_rand_uniform",
    "repops_dropout", "repops_dropout_backward",
    "repops_gelu_erf_backward", "repops_rope_tables", "repops_ipc_alloc", "repops_ipc_open", "repops_ipc_close",
    "repops_ipc_free", "repops_p2p_tree_combine", "repops_p2p_signal", "repops_p2p_wait", "repops_add", "repops_embedding",
    "repops_embedding_backward", "repops_adamw", "repops_flip_bit", "verde_commit_tensor",
    "verde_commit_tensors", "verde_merkle_root", "verde_sha256", "verde_node_digest",
    "verde_first_divergence", "verde_digest_from_subroots", "launch_count", "CommitWorkspace", "CommitPlan",
    "RepopsError",
    "header_symbols", "lib", "KernelTimer", "set_timer",
]


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _p(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise RepopsError("tensor must live on a CUDA device")
    return t.data_ptr()


def _f32(t, name):
    if t.dtype != torch.float32 or not t.is_cuda:
        raise RepopsError(f"{name}: expected a float32 CUDA tensor, got {t.dtype} on {t.device}")
    return t


def _ld(t) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise RepopsError("expected a 2-D tensor with unit column stride")
    return t.stride(0)


# ------------------------------------------------------------------ live kernel timing (bench.py)
class KernelTimer:
    """Optional CUDA-event bracketing of library launches on their stream, so a
    benchmark can report a kernel family's device time inside its timed region.
    Enabled with set_timer(KernelTimer()); costs two event records per launch."""

    def __init__(self):
        self.ev = {}  # kind -> list of (start, end, work)

    def begin(self, stream=None):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream if stream is not None else torch.cuda.current_stream())
        return e

    def end(self, kind, e0, work, stream=None):
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(stream if stream is not None else torch.cuda.current_stream())
        self.ev.setdefault(kind, []).append((e0, e1, work))

    def totals(self):
        """kind -> (device ms, work units, launches); call after synchronising."""
        return {k: (sum(a.elapsed_time(b) for a, b, _ in v), sum(w for _, _, w in v), len(v))
                for k, v in self.ev.items()}

    def union_ms(self, kind, ref):
        """Length of the union of `kind`'s launch intervals (ms), measured from the event
        `ref` recorded before them: launches of one family that overlap each other on
        different streams are counted once."""
        iv = sorted((ref.elapsed_time(a), ref.elapsed_time(b)) for a, b, _ in self.ev.get(kind, []))
        tot, cur_s, cur_e = 0.0, None, None
        for s, e in iv:
            if cur_e is None or s > cur_e:
                if cur_e is not None:
                    tot += cur_e - cur_s
                cur_s, cur_e = s, e
            else:
                cur_e = max(cur_e, e)
        return tot + ((cur_e - cur_s) if cur_e is not None else 0.0)


_TIMER = None


def set_timer(t):
    global _TIMER
    _TIMER = t


# ------------------------------------------------------------------ GEMM
def repops_gemm(A, B, transA=False, transB=False, epi=EPI_NONE, bias=None, scale=1.0, out=None, stream=None,
                cfg=None):
    """R-GEMM.  A: (M,K) or (K,M) if transA; B: (K,N) or (N,K) if transB."""
    _f32(A, "A"), _f32(B, "B")
    M = A.shape[1] if transA else A.shape[0]
    K = A.shape[0] if transA else A.shape[1]
    N = B.shape[0] if transB else B.shape[1]
    Kb = B.shape[1] if transB else B.shape[0]
    if Kb != K:
        raise RepopsError(f"repops_gemm: inner dimensions differ ({K} vs {Kb})")
    if B.device != A.device:
        raise RepopsError(f"repops_gemm: A on {A.device}, B on {B.device}")
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=A.device)
    else:
        _f32(out, "out")
        if tuple(out.shape) != (M, N) or out.device != A.device:
            raise RepopsError(f"repops_gemm: out must be ({M}, {N}) on {A.device}, got {tuple(out.shape)} "
                              f"on {out.device}")
    if epi == EPI_BIAS:
        if bias is None:
            raise RepopsError("repops_gemm: EPI_BIAS needs a bias")
        _f32(bias, "bias")
        if bias.device != A.device or bias.numel() < N or (bias.dim() == 1 and bias.stride(0) != 1):
            raise RepopsError(f"repops_gemm: bias must hold >= {N} contiguous floats on {A.device}")
    args = (M, N, K, _p(A), _ld(A), int(bool(transA)), _p(B), _ld(B), int(bool(transB)), int(epi), _p(bias),
            float(scale), _p(out), _ld(out), _stream(stream))
    t0 = _TIMER.begin(stream) if _TIMER else None
    if cfg is None:
        check(lib().repops_gemm(*args), "repops_gemm")
    else:
        check(lib().repops_gemm_cfg(*args, int(cfg)), "repops_gemm_cfg")
    if t0 is not None:
        _TIMER.end("gemm", t0, 2 * M * N * K, stream)
    return out


POST_GELU, POST_GELU_BACKWARD = 1, 2


def repops_gemm_post(A, B, post, out2, X=None, transA=False, transB=False, epi=EPI_NONE, bias=None, scale=1.0,
                     out=None, stream=None):
    """R-GEMM with a fused elementwise consumer (repops.h repops_gemm_post): returns (C, C2)
    with C2 = R-GELU(C) (post = POST_GELU) or R-GELU-backward at X with dy = C."""
    _f32(A, "A"), _f32(B, "B"), _f32(out2, "out2")
    M = A.shape[1] if transA else A.shape[0]
    K = A.shape[0] if transA else A.shape[1]
    N = B.shape[0] if transB else B.shape[1]
    if (B.shape[1] if transB else B.shape[0]) != K:
        raise RepopsError(f"repops_gemm_post: inner dimensions differ ({K})")
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=A.device)
    for t, nm in ((out, "out"), (out2, "out2")) + (((X, "X"),) if post == POST_GELU_BACKWARD else ()):
        _f32(t, nm)
        if tuple(t.shape) != (M, N):
            raise RepopsError(f"repops_gemm_post: {nm} must be ({M}, {N})")
    if epi == EPI_BIAS and (bias is None or bias.numel() < N):
        raise RepopsError(f"repops_gemm_post: EPI_BIAS needs >= {N} bias values")
    t0 = _TIMER.begin(stream) if _TIMER else None
    check(lib().repops_gemm_post(M, N, K, _p(A), _ld(A), int(bool(transA)), _p(B), _ld(B), int(bool(transB)),
                                 int(epi), _p(bias), float(scale), _p(out), _ld(out), int(post), _p(X),
                                 _ld(X) if X is not None else 0, _p(out2), _ld(out2), _stream(stream)),
          "repops_gemm_post")
    if t0 is not None:
        _TIMER.end("gemm", t0, 2 * M * N * K, stream)
    return out, out2


def repops_gemm_strided_batched(A, B, C_out, M, N, K, lda, ldb, ldc, sA, sB, sC, batch, transA=False,
                                transB=False, epi=EPI_NONE, bias=None, scale=1.0, offA=0, offB=0, offC=0,
                                stream=None, causal=0, kflags=None, ldf=0, sF=(0, 0)):
    """Two-level strided batch of R-GEMMs.  sA/sB/sC = (outer, inner) element strides,
    batch = (outer, inner) counts; off* are element offsets into the storage of A/B/C.
    causal (repops_gemm_strided_batched_causal): 1 = outputs above the diagonal are not
    computed (never-read scratch scores); 2 = op(A) is +0 above the diagonal (causal
    probabilities) -- each tile's K fold stops at its last row, the skipped +0 terms applied
    exactly from kflags (repops_causal_suffix_flags of B, [K + 1][ldf] per problem)."""
    _f32(A, "A"), _f32(B, "B"), _f32(C_out, "C")
    t0 = _TIMER.begin(stream) if _TIMER else None
    args = (M, N, K, _p(A) + 4 * offA, lda, int(bool(transA)), sA[0], sA[1], _p(B) + 4 * offB, ldb,
            int(bool(transB)), sB[0], sB[1], int(epi), _p(bias), float(scale), _p(C_out) + 4 * offC, ldc, sC[0],
            sC[1], batch[0], batch[1])
    if causal:
        if causal == 2 and (kflags is None or kflags.dtype != torch.uint8):
            raise RepopsError("repops_gemm_strided_batched: causal 2 needs uint8 kflags")
        check(lib().repops_gemm_strided_batched_causal(*args, int(causal), _p(kflags), int(ldf), sF[0], sF[1],
                                                       _stream(stream)), "repops_gemm_strided_batched_causal")
    else:
        check(lib().repops_gemm_strided_batched(*args, _stream(stream)), "repops_gemm_strided_batched")
    if t0 is not None:
        _TIMER.end("gemm", t0, 2 * M * N * K * batch[0] * batch[1], stream)
    return C_out


def repops_causal_suffix_flags(B, K, N, ldb, sB, batch, out=None, ldf=None, sF=None, offB=0, stream=None):
    """uint8 [batch0 * batch1, K + 1, ldf] suffix flags of B for causal mode 2 (see repops.h)."""
    ldf = N if ldf is None else ldf
    if out is None:
        out = torch.empty((batch[0] * batch[1], K + 1, ldf), dtype=torch.uint8, device=B.device)
        sF = ((K + 1) * ldf * batch[1], (K + 1) * ldf)
    check(lib().repops_causal_suffix_flags(_p(B) + 4 * offB, K, N, ldb, sB[0], sB[1], batch[0], batch[1], _p(out),
                                           ldf, sF[0], sF[1], _stream(stream)), "repops_causal_suffix_flags")
    return out


# ------------------------------------------------------------------ fused attention (f4)
def _fits(t, off, strides, batch, rows, cols, ld):
    """the last (b0, b1) block of a strided batch lies inside t's storage"""
    last = off + (int(batch[0]) - 1) * int(strides[0]) + (int(batch[1]) - 1) * int(strides[1]) + \
        (rows - 1) * ld + cols
    return t.storage_offset() + last <= t.untyped_storage().nbytes() // 4


def repops_attention_probs_supported(T, hd):
    return bool(lib().repops_attention_probs_supported(int(T), int(hd)))


def repops_attention_probs(qkv, T, hd, ld, s, q_off, k_off, batch, P, sp, scale=1.0, causal=True, stream=None,
                           kv=None, ldk=None, sk=None):
    """Scores + softmax fused over a strided batch (element offsets / strides into the
    storage of qkv and P): P = causal R-SOFTMAX(R-GEMM(Q K^T) * scale), the scores never
    leaving shared memory -- bit-identical to repops_gemm_strided_batched(SCALE) ->
    repops_softmax.  K comes from kv (default qkv) with row stride ldk and batch strides sk
    (default ld, s; sk[1] = 0 shares one K among the inner batch, grouped-query attention)."""
    kv = qkv if kv is None else kv
    ldk = ld if ldk is None else ldk
    sk = s if sk is None else sk
    _f32(qkv, "qkv"), _f32(kv, "kv"), _f32(P, "P")
    if P.device != qkv.device or kv.device != qkv.device:
        raise ValueError("qkv, kv and P must be on one device")
    nb = int(batch[0]) * int(batch[1])
    if nb and not (_fits(qkv, q_off, s, batch, T, hd, ld) and _fits(kv, k_off, sk, batch, T, hd, ldk)
                   and _fits(P, 0, sp, batch, T, T, T)):
        raise ValueError("attention_probs: qkv, kv or P too small for the batch")
    t0 = _TIMER.begin(stream) if _TIMER else None
    check(lib().repops_attention_probs(int(T), int(hd), qkv.data_ptr() + 4 * q_off, int(ld), int(s[0]), int(s[1]),
                                       kv.data_ptr() + 4 * k_off, int(ldk), int(sk[0]), int(sk[1]), float(scale),
                                       int(bool(causal)), P.data_ptr(), int(sp[0]), int(sp[1]), int(batch[0]),
                                       int(batch[1]), _stream(stream)),
          "repops_attention_probs")
    if t0 is not None:
        _TIMER.end("gemm", t0, 2 * T * T * hd * nb, stream)
    return P


def repops_attention_dscores(dO, V, T, hd, ldo, so, o_off, ldv, sv, v_off, P, sp, dS, sd, batch, scale=1.0,
                             stream=None):
    """Attention backward, scores part, fused: dS = R-SOFTMAX-BWD(P, R-GEMM(dO, V^T)) * scale
    over a strided batch (element offsets / strides into the storage of dO, V, P, dS), the
    dP matrix never leaving shared memory -- bit-identical to repops_gemm_strided_batched ->
    repops_softmax_backward."""
    for t, n in ((dO, "dO"), (V, "V"), (P, "P"), (dS, "dS")):
        _f32(t, n)
        if t.device != dO.device:
            raise ValueError(f"{n} must be on the device of dO")
    nb = int(batch[0]) * int(batch[1])
    if nb and not (_fits(dO, o_off, so, batch, T, hd, ldo) and _fits(V, v_off, sv, batch, T, hd, ldv)
                   and _fits(P, 0, sp, batch, T, T, T) and _fits(dS, 0, sd, batch, T, T, T)):
        raise ValueError("attention_dscores: an operand is too small for the batch")
    t0 = _TIMER.begin(stream) if _TIMER else None
    check(lib().repops_attention_dscores(int(T), int(hd), dO.data_ptr() + 4 * o_off, int(ldo), int(so[0]),
                                         int(so[1]), V.data_ptr() + 4 * v_off, int(ldv), int(sv[0]), int(sv[1]),
                                         P.data_ptr(), int(sp[0]), int(sp[1]), float(scale), dS.data_ptr(),
                                         int(sd[0]), int(sd[1]), int(batch[0]), int(batch[1]), _stream(stream)),
          "repops_attention_dscores")
    if t0 is not None:
        _TIMER.end("gemm", t0, 2 * T * T * hd * nb, stream)
    return dS


def repops_attention_fwd_supported(T, hd):
    return bool(lib().repops_attention_fwd_supported(int(T), int(hd)))


def repops_attention_fwd(qkv, T, hd, ld, s, q_off, k_off, v_off, batch, O, ldo, so, S=None, P=None, sp=(0, 0),
                         scale=1.0, causal=True, stream=None):
    """Fused R-ATTN forward over a strided batch (element offsets / strides into the
    storage of qkv, O, S, P): S = R-GEMM(Q K^T) * scale, P = causal R-SOFTMAX(S),
    O = R-GEMM(P, V) -- bit-identical to the three unfused calls."""
    _f32(qkv, "qkv"), _f32(O, "O")
    base = qkv.data_ptr()
    t0 = _TIMER.begin(stream) if _TIMER else None
    check(lib().repops_attention_fwd(int(T), int(hd), base + 4 * q_off, base + 4 * k_off, base + 4 * v_off, int(ld),
                                     int(s[0]), int(s[1]), float(scale), int(bool(causal)), _p(S), _p(P),
                                     int(sp[0]), int(sp[1]), _p(O), int(ldo), int(so[0]), int(so[1]), int(batch[0]),
                                     int(batch[1]), _stream(stream)), "repops_attention_fwd")
    if t0 is not None:
        _TIMER.end("gemm", t0, 4 * T * T * hd * batch[0] * batch[1], stream)
    return O


# ------------------------------------------------------------------ R30 stored precision
_LP = {torch.float32: F32, torch.bfloat16: BF16, torch.float16: F16}


def repops_convert(x, dtype, out=None, stream=None):
    """R30: 2-D (or 1-D) x -> dtype (f32 / bf16 / f16): exact widening, RN-even narrowing."""
    if x.dtype not in _LP or dtype not in _LP:
        raise RepopsError("repops_convert: dtypes must be float32 / bfloat16 / float16")
    x2 = x if x.dim() == 2 else x.reshape(1, -1)
    if out is None:
        out = torch.empty(x.shape, dtype=dtype, device=x.device)
    o2 = out if out.dim() == 2 else out.reshape(1, -1)
    check(lib().repops_convert(_p(x2), _LP[x.dtype], x2.shape[0], x2.shape[1], _ld(x2), _p(o2), _LP[dtype],
                               _ld(o2), _stream(stream)), "repops_convert")
    return out


def repops_gemm_ex(A, B, transA=False, transB=False, epi=EPI_NONE, bias=None, scale=1.0, out=None, out_dtype=None,
                   stream=None):
    """R30: C = narrow(R-GEMM(widen(A), widen(B))); A / B / C stored as f32, bf16 or f16."""
    M = A.shape[1] if transA else A.shape[0]
    K = A.shape[0] if transA else A.shape[1]
    N = B.shape[0] if transB else B.shape[1]
    if (B.shape[1] if transB else B.shape[0]) != K:
        raise RepopsError("repops_gemm_ex: inner dimensions differ")
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype or A.dtype, device=A.device)
    wsb = lib().repops_gemm_ex_workspace_bytes(M, N, K, _LP[A.dtype], _LP[B.dtype], _LP[out.dtype])
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=A.device)
    t0 = _TIMER.begin(stream) if _TIMER else None
    check(lib().repops_gemm_ex(M, N, K, _p(A), _LP[A.dtype], _ld(A), int(bool(transA)), _p(B), _LP[B.dtype], _ld(B),
                               int(bool(transB)), int(epi), _p(bias), float(scale), _p(out), _LP[out.dtype], _ld(out),
                               _p(ws), wsb, _stream(stream)), "repops_gemm_ex")
    if t0 is not None:
        _TIMER.end("gemm", t0, 2 * M * N * K, stream)
    return out


# ------------------------------------------------------------------ reductions
def repops_sum_rows(x, out=None, stream=None):
    _f32(x, "x")
    if out is None:
        out = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    check(lib().repops_sum_rows(_p(x), x.shape[0], x.shape[1], _ld(x), _p(out), _stream(stream)), "repops_sum_rows")
    return out


def repops_sum_cols_seq(x, nseg=1, out=None, ldo=None, stream=None):
    """R-SEQ column folds per segment; out[s*ldo + j] (out may be a flat buffer view)."""
    _f32(x, "x")
    if out is None:
        out = torch.empty((nseg, x.shape[1]), dtype=torch.float32, device=x.device)
    ldo = x.shape[1] if ldo is None else ldo
    check(lib().repops_sum_cols_seq(_p(x), x.shape[0], x.shape[1], _ld(x), nseg, _p(out), ldo, _stream(stream)),
          "repops_sum_cols_seq")
    return out


def repops_tree_sum(parts, out=None, stream=None):
    n = parts[0].numel()
    for q in parts:
        _f32(q, "part")
        if q.numel() != n or not q.is_contiguous():
            raise RepopsError("repops_tree_sum: parts must be contiguous with equal sizes")
    if out is None:
        out = torch.empty_like(parts[0])
    arr = (C.c_void_p * len(parts))(*[q.data_ptr() for q in parts])
    check(lib().repops_tree_sum(arr, len(parts), n, _p(out), _stream(stream)), "repops_tree_sum")
    return out


# ------------------------------------------------------------------ peer memory (multi-GPU DP combine)
class _DevArray:
    """__cuda_array_interface__ view of a raw device allocation (no copy)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


_TYPESTR = {torch.float32: "<f4", torch.int32: "<i4", torch.uint8: "|u1"}


def repops_ipc_alloc(n, dtype=torch.float32, device=None):
    """(tensor, handle bytes): n zero-filled elements in an IPC-shareable cudaMalloc block.
    The caller keeps the tensor alive and frees the block with repops_ipc_free(tensor)."""
    esz = torch.empty(0, dtype=dtype).element_size()
    ptr, h = C.c_void_p(), (C.c_uint8 * 64)()
    check(lib().repops_ipc_alloc(int(n) * esz, C.byref(ptr), h), "repops_ipc_alloc")
    t = torch.as_tensor(_DevArray(ptr.value, n, _TYPESTR[dtype]), device=device or torch.cuda.current_device())
    return t, bytes(h)


def repops_ipc_open(handle, n, dtype=torch.float32, device=None):
    """tensor view of a peer's allocation (repops_ipc_close(tensor) unmaps it)."""
    ptr = C.c_void_p()
    check(lib().repops_ipc_open((C.c_uint8 * 64).from_buffer_copy(handle), C.byref(ptr)), "repops_ipc_open")
    return torch.as_tensor(_DevArray(ptr.value, n, _TYPESTR[dtype]), device=device or torch.cuda.current_device())


def repops_ipc_close(t):
    check(lib().repops_ipc_close(t.data_ptr()), "repops_ipc_close")


def repops_ipc_free(t):
    check(lib().repops_ipc_free(t.data_ptr()), "repops_ipc_free")


def repops_p2p_tree_combine(parts, lo, hi, outs, stream=None, status=None):
    """out[q][i] = R-TREE_S over parts[*][i] for i in [lo, hi), stored into every outs[q].
    status: optional device int32 set by a timed-out repops_p2p_wait -- nothing is stored then."""
    G = len(parts)
    if len(outs) != G:
        raise RepopsError("repops_p2p_tree_combine: need one output per part")
    pa = (C.c_void_p * G)(*[_p(q) for q in parts])
    oa = (C.c_void_p * G)(*[_p(q) for q in outs])
    check(lib().repops_p2p_tree_combine(pa, G, int(lo), int(hi), oa, _p(status), _stream(stream)),
          "repops_p2p_tree_combine")


def repops_p2p_signal(peer_flags, slot, epoch, stream=None):
    fa = (C.c_void_p * len(peer_flags))(*[_p(q) for q in peer_flags])
    check(lib().repops_p2p_signal(fa, len(peer_flags), int(slot), int(epoch) & 0xFFFFFFFF, _stream(stream)),
          "repops_p2p_signal")


def repops_p2p_wait(flags, G, epoch, timeout_ms=60000, status=None, stream=None):
    check(lib().repops_p2p_wait(_p(flags), int(G), int(epoch) & 0xFFFFFFFF, int(timeout_ms), _p(status),
                                _stream(stream)), "repops_p2p_wait")


# ------------------------------------------------------------------ row operators
def repops_softmax(x, causal=False, out=None, stream=None):
    _f32(x, "x")
    if out is None:
        out = torch.empty_like(x)
    check(lib().repops_softmax(_p(x), x.shape[0], x.shape[1], _ld(x), int(bool(causal)), _p(out), _ld(out),
                               _stream(stream)), "repops_softmax")
    return out


def repops_softmax_backward(y, dy, scale=1.0, out=None, stream=None):
    _f32(y, "y"), _f32(dy, "dy")
    if out is None:
        out = torch.empty_like(y)
    check(lib().repops_softmax_backward(_p(y), _ld(y), _p(dy), _ld(dy), y.shape[0], y.shape[1], float(scale),
                                        _p(out), _ld(out), _stream(stream)), "repops_softmax_backward")
    return out


def _contig(t, name):
    _f32(t, name)
    if not t.is_contiguous():
        raise RepopsError(f"{name} must be contiguous")
    return t


def repops_layernorm(x, gamma, beta, eps=1e-5, out=None, mean=None, rstd=None, stream=None):
    _contig(x, "x")
    rows, cols = x.shape
    if out is None:
        out = torch.empty_like(x)
    if mean is None:
        mean = torch.empty(rows, dtype=torch.float32, device=x.device)
    if rstd is None:
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    check(lib().repops_layernorm(_p(x), _p(gamma), _p(beta), rows, cols, float(eps), _p(out), _p(mean), _p(rstd),
                                 _stream(stream)), "repops_layernorm")
    return out, mean, rstd


def repops_layernorm_backward(dy, x, gamma, mean, rstd, dres=None, out=None, stream=None):
    _contig(dy, "dy"), _contig(x, "x")
    rows, cols = x.shape
    if out is None:
        out = torch.empty_like(x)
    check(lib().repops_layernorm_backward(_p(dy), _p(x), _p(gamma), _p(mean), _p(rstd), _p(dres), rows, cols,
                                          _p(out), _stream(stream)), "repops_layernorm_backward")
    return out


def repops_layernorm_backward_params(dy, x, mean, rstd, nseg=1, dgamma=None, dbeta=None, ldo=None, stream=None):
    rows, cols = x.shape
    ldo = cols if ldo is None else ldo
    if dgamma is None:
        dgamma = torch.empty((nseg, cols), dtype=torch.float32, device=x.device)
    if dbeta is None:
        dbeta = torch.empty((nseg, cols), dtype=torch.float32, device=x.device)
    check(lib().repops_layernorm_backward_params(_p(dy), _p(x), _p(mean), _p(rstd), rows, cols, nseg, _p(dgamma),
                                                 _p(dbeta), ldo, _stream(stream)), "repops_layernorm_backward_params")
    return dgamma, dbeta


def repops_cross_entropy(logits, labels, scale=1.0, loss=None, dlogits=None, want_grad=True, V=None, stream=None):
    """logits: (rows, ld) with the first V columns valid (V defaults to all)."""
    _f32(logits, "logits")
    rows = logits.shape[0]
    V = logits.shape[1] if V is None else V
    if labels.dtype != torch.int32:
        raise RepopsError("labels must be int32")
    if loss is None:
        loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
    if want_grad and dlogits is None:
        dlogits = torch.empty_like(logits)
    check(lib().repops_cross_entropy(_p(logits), rows, V, _ld(logits), _p(labels), float(scale), _p(loss),
                                     _p(dlogits) if want_grad else None,
                                     _ld(dlogits) if want_grad else V, _stream(stream)), "repops_cross_entropy")
    return loss, dlogits


# ------------------------------------------------------------------ elementwise
def _unary(name, x, out, stream):
    _contig(x, "x")
    if out is None:
        out = torch.empty_like(x)
    check(getattr(lib(), name)(_p(x), x.numel(), _p(out), _stream(stream)), name)
    return out


def repops_exp(x, out=None, stream=None):
    return _unary("repops_exp", x, out, stream)


def repops_log(x, out=None, stream=None):
    return _unary("repops_log", x, out, stream)


def repops_tanh(x, out=None, stream=None):
    return _unary("repops_tanh", x, out, stream)


def repops_rsqrt(x, out=None, stream=None):
    return _unary("repops_rsqrt", x, out, stream)


def repops_gelu(x, out=None, stream=None):
    return _unary("repops_gelu", x, out, stream)


def repops_sin(x, out=None, stream=None):
    """R26 (Cephes sinf chain)."""
    return _unary("repops_sin", x, out, stream)


def repops_cos(x, out=None, stream=None):
    """R26 (Cephes cosf chain)."""
    return _unary("repops_cos", x, out, stream)


def repops_rand_uniform(seed, stream_id, n, out=None, stream=None):
    """R28: u_i in [0, 1) from Philox4x32-10 (seed, stream_id, i)."""
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device="cuda")
    check(lib().repops_rand_uniform(int(seed), int(stream_id), int(n), _p(out), _stream(stream)),
          "repops_rand_uniform")
    return out


def repops_dropout(x, p, seed, stream_id, out=None, mask=None, stream=None):
    """R28: y = keep ? x * (1 / (1 - p)) : +0, keep = u >= p; returns (y, mask or None)."""
    _contig(x, "x")
    if out is None:
        out = torch.empty_like(x)
    check(lib().repops_dropout(_p(x), x.numel(), float(p), int(seed), int(stream_id), _p(out), _p(mask),
                               _stream(stream)), "repops_dropout")
    return out, mask


def repops_dropout_backward(dy, p, seed, stream_id, out=None, stream=None):
    """R28: dx = keep ? dy * (1 / (1 - p)) : +0 (mask regenerated from the counter)."""
    _contig(dy, "dy")
    if out is None:
        out = torch.empty_like(dy)
    check(lib().repops_dropout_backward(_p(dy), dy.numel(), float(p), int(seed), int(stream_id), _p(out),
                                        _stream(stream)), "repops_dropout_backward")
    return out


def repops_erf(x, out=None, stream=None):
    """R27 (Cephes erff / erfcf chain)."""
    return _unary("repops_erf", x, out, stream)


def repops_gelu_erf(x, out=None, stream=None):
    """R27: exact GELU 0.5 x (1 + erf(x / sqrt 2))."""
    return _unary("repops_gelu_erf", x, out, stream)


def repops_gelu_erf_backward(x, dy, out=None, stream=None):
    """R27: dx = dy (cdf + x pdf)."""
    _contig(x, "x"), _contig(dy, "dy")
    if out is None:
        out = torch.empty_like(x)
    check(lib().repops_gelu_erf_backward(_p(x), _p(dy), x.numel(), _p(out), _stream(stream)),
          "repops_gelu_erf_backward")
    return out


def repops_rope_tables(inv_freq, T, cos=None, sin=None, stream=None):
    """R26: (cos, sin) [T, h] with angle fmul(t, inv_freq[i])."""
    _contig(inv_freq, "inv_freq")
    h = inv_freq.numel()
    cos = torch.empty((T, h), dtype=torch.float32, device=inv_freq.device) if cos is None else cos
    sin = torch.empty((T, h), dtype=torch.float32, device=inv_freq.device) if sin is None else sin
    check(lib().repops_rope_tables(_p(inv_freq), int(T), h, _p(cos), _p(sin), _stream(stream)), "repops_rope_tables")
    return cos, sin


def repops_relu(x, out=None, stream=None):
    """R24: relu(x) = x > 0 ? x : +0."""
    return _unary("repops_relu", x, out, stream)


def repops_relu_backward(x, g, out=None, stream=None):
    """R24: dx = x > 0 ? g : +0 (subgradient 0 at x = 0)."""
    _contig(x, "x"), _contig(g, "g")
    if out is None:
        out = torch.empty_like(x)
    check(lib().repops_relu_backward(_p(x), _p(g), x.numel(), _p(out), _stream(stream)), "repops_relu_backward")
    return out


def repops_gelu_backward(x, dy, out=None, stream=None):
    _contig(x, "x"), _contig(dy, "dy")
    if out is None:
        out = torch.empty_like(x)
    check(lib().repops_gelu_backward(_p(x), _p(dy), x.numel(), _p(out), _stream(stream)), "repops_gelu_backward")
    return out


def repops_add(a, b, out=None, stream=None):
    _contig(a, "a"), _contig(b, "b")
    if out is None:
        out = torch.empty_like(a)
    check(lib().repops_add(_p(a), _p(b), a.numel(), _p(out), _stream(stream)), "repops_add")
    return out


def repops_embedding(tok, wte, wpe, T, out=None, stream=None):
    if tok.dtype != torch.int32:
        raise RepopsError("tok must be int32")
    Cc = wte.shape[1]
    if out is None:
        out = torch.empty((tok.numel(), Cc), dtype=torch.float32, device=wte.device)
    check(lib().repops_embedding(_p(tok), tok.numel(), T, _p(wte), _p(wpe), Cc, _p(out), _stream(stream)),
          "repops_embedding")
    return out


def repops_embedding_backward(tok, dx0, T, dwte, dwpe=None, stream=None):
    """Accumulates the shard's embedding gradient INTO dwte (and dwpe)."""
    check(lib().repops_embedding_backward(_p(tok), tok.numel(), T, _p(dx0), dx0.shape[1], _p(dwte), _p(dwpe),
                                          _stream(stream)), "repops_embedding_backward")
    return dwte, dwpe


def repops_adamw_segments(p, g, m, v, seg_start, decay, step, lr, b1, b2, eps, wd, stream=None):
    """AdamW over back-to-back parameter tensors in one launch; seg_start: nseg+1 element
    offsets (first 0), decay: nseg flags.  In place on p, m, v."""
    for t, nm in ((p, "p"), (g, "g"), (m, "m"), (v, "v")):
        _contig(t, nm)
    nseg = len(decay)
    st = (C.c_int64 * (nseg + 1))(*[int(x) for x in seg_start])
    dc = (C.c_uint8 * nseg)(*[1 if d else 0 for d in decay])
    check(lib().repops_adamw_segments(_p(p), _p(g), _p(m), _p(v), nseg, st, dc, int(step), float(lr), float(b1),
                                      float(b2), float(eps), float(wd), _stream(stream)), "repops_adamw_segments")
    return p, m, v


def repops_adamw(p, g, m, v, step, lr, b1, b2, eps, wd, decay, stream=None):
    """In place on p, m, v."""
    for t, nm in ((p, "p"), (g, "g"), (m, "m"), (v, "v")):
        _contig(t, nm)
    check(lib().repops_adamw(_p(p), _p(g), _p(m), _p(v), p.numel(), int(step), float(lr), float(b1), float(b2),
                             float(eps), float(wd), int(bool(decay)), _stream(stream)), "repops_adamw")
    return p, m, v


def repops_rmsnorm(x, w, eps=1e-5, out=None, rstd=None, stream=None):
    """R-RMSNORM (contiguous rows, cols <= 4096).  Returns (y, rstd)."""
    _contig(x, "x")
    rows, cols = x.shape
    if out is None:
        out = torch.empty_like(x)
    if rstd is None:
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    check(lib().repops_rmsnorm(_p(x), _p(w), rows, cols, float(eps), _p(out), _p(rstd), _stream(stream)),
          "repops_rmsnorm")
    return out, rstd


def repops_swiglu(g, u, out=None, stream=None):
    _contig(g, "g"), _contig(u, "u")
    if out is None:
        out = torch.empty_like(g)
    check(lib().repops_swiglu(_p(g), _p(u), g.numel(), _p(out), _stream(stream)), "repops_swiglu")
    return out


def repops_rope(x, cos_t, sin_t, nhead, hd, out=None, stream=None):
    """R-ROPE on x [ntok, >= nhead*hd] (row stride = ld) with tables [ntok, hd/2]."""
    _f32(x, "x")
    if out is None:
        out = torch.empty_like(x)
    check(lib().repops_rope(_p(x), x.shape[0], nhead, hd, _ld(x), _p(cos_t), _p(sin_t), _p(out), _ld(out),
                            _stream(stream)), "repops_rope")
    return out


def repops_gather_rows(table, idx, out=None, stream=None):
    if idx.dtype != torch.int32:
        raise RepopsError("idx must be int32")
    n, Cc = idx.numel(), table.shape[1]
    if out is None:
        out = torch.empty((n, Cc), dtype=torch.float32, device=table.device)
    check(lib().repops_gather_rows(_p(table), _p(idx), n, Cc, _p(out), _stream(stream)), "repops_gather_rows")
    return out


def repops_fill_uniform(out, seed, scale=1.0, stream=None):
    """Device twin of synth.uniform(seed, shape, scale) (input generation only)."""
    check(lib().repops_fill_uniform(_p(out), out.numel(), int(seed) & 0xFFFFFFFFFFFFFFFF, float(scale),
                                    _stream(stream)), "repops_fill_uniform")
    return out


def repops_copy2d(src, dst, stream=None):
    """dst[:, :] = src (both 2-D views with unit column stride; data movement only)."""
    rows, cols = src.shape
    check(lib().repops_copy2d(_p(src), rows, cols, _ld(src), _p(dst), _ld(dst), _stream(stream)), "repops_copy2d")
    return dst


def repops_copy2d_batched(src, dst, rows, cols, lds, ss, ldd, sd, nb, stream=None):
    """for b < nb: dst[b*sd + r*ldd + c] = src[b*ss + r*lds + c] (element offsets; data movement)."""
    check(lib().repops_copy2d_batched(_p(src), rows, cols, lds, ss, _p(dst), ldd, sd, nb, _stream(stream)),
          "repops_copy2d_batched")
    return dst


def repops_transpose(x, out=None, stream=None):
    """out = x^T (bit-exact data movement)."""
    _f32(x, "x")
    rows, cols = x.shape
    if out is None:
        out = torch.empty((cols, rows), dtype=torch.float32, device=x.device)
    check(lib().repops_transpose(_p(x), rows, cols, _ld(x), _p(out), _ld(out), _stream(stream)), "repops_transpose")
    return out


def repops_flip_bit(t, elem, bit, stream=None):
    check(lib().repops_flip_bit(_p(t), int(elem), int(bit), _stream(stream)), "repops_flip_bit")
    return t


# ------------------------------------------------------------------ Verde commitments
class CommitWorkspace:
    """Caller-owned device workspace for verde_commit_tensors (grown on demand)."""

    def __init__(self, device="cuda"):
        self.device = torch.device(device)
        self.buf = None

    def get(self, nbytes: int):
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=self.device)
        return self.buf


def _desc(t, digest, mode=0, leaves_out=None, base_leaves=None, dirty=None) -> TensorDesc:
    if not t.is_contiguous():
        raise RepopsError("committed tensors must be contiguous")
    nch = (t.numel() * t.element_size() + 4095) // 4096
    for buf, nb, what in ((leaves_out, 32 * nch, "leaves_out"), (base_leaves, 32 * nch, "base_leaves"),
                          (dirty, nch, "dirty")):
        if buf is not None and (buf.dtype != torch.uint8 or buf.numel() < nb or buf.device != t.device):
            raise ValueError(f"{what}: need a uint8 device buffer of >= {nb} bytes")
    if (base_leaves is None) != (dirty is None):
        raise ValueError("base_leaves and dirty go together")
    d = TensorDesc()
    d.leaves_out = leaves_out.data_ptr() if leaves_out is not None else None
    d.base_leaves = base_leaves.data_ptr() if base_leaves is not None else None
    d.dirty = dirty.data_ptr() if dirty is not None else None
    d.data = t.data_ptr() if t.numel() else None
    d.nbytes = t.numel() * t.element_size()
    d.dtype = _DT[t.dtype]
    d.rank = t.dim()
    for i, s in enumerate(t.shape):
        d.dims[i] = s
    d.digest = digest.data_ptr()
    d.mode = mode
    return d


def repops_ffma2_probe_tflops(ctas_per_sm=4, iters=20000):
    """Diagnostic: FP32 FMA rate of register-resident FFMA2 chains over the whole GPU --
    the R-GEMM's practical ceiling, TFLOP/s."""
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    ctas = sms * int(ctas_per_sm)
    out = torch.empty(ctas * 128, dtype=torch.float32, device="cuda")
    run = lambda: check(lib().repops_ffma2_probe(ctas, int(iters), out.data_ptr(), _stream(None)),  # noqa: E731
                        "repops_ffma2_probe")
    run()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    b.synchronize()
    return ctas * 128 * int(iters) * 128 / (a.elapsed_time(b) * 1e-3) / 1e12


def verde_sha256_probe_gbs(ctas_per_sm=9, iters=2000):
    """Diagnostic: the SHA-256 compression rate with register-resident blocks (no memory
    traffic) over the whole GPU -- the commitment kernels' practical ALU ceiling, GB/s."""
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    ctas = sms * int(ctas_per_sm)
    out = torch.empty(ctas * 128, dtype=torch.int32, device="cuda")
    run = lambda: check(lib().verde_sha256_probe(ctas, int(iters), out.data_ptr(), _stream(None)),  # noqa: E731
                        "verde_sha256_probe")
    run()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    b.synchronize()
    return ctas * 128 * int(iters) * 64 / (a.elapsed_time(b) * 1e-3) / 1e9


def verde_dirty_chunks(rows, row_bytes, nbytes, out, all_chunks=False, stream=None):
    """uint8 flags per 4096-byte chunk of a row-major tensor: 1 where one of `rows` (int32
    device tensor) meets the chunk (verde_tensor_desc.dirty of an incremental commit)."""
    nch = (int(nbytes) + 4095) // 4096
    if out.dtype != torch.uint8 or out.numel() < nch:
        raise ValueError(f"out: need >= {nch} uint8 flags")
    if rows is not None and rows.dtype != torch.int32:
        raise ValueError("rows must be int32")
    n = 0 if rows is None else rows.numel()
    check(lib().verde_dirty_chunks(rows.data_ptr() if n else None, n, int(row_bytes), int(nbytes),
                                   int(bool(all_chunks)), out.data_ptr(), _stream(stream)), "verde_dirty_chunks")
    return out


def verde_commit_tensors(tensors, digests=None, ws: CommitWorkspace | None = None, stream=None, mode=0):
    """R-TCOMMIT for a list of tensors in one batched launch sequence.  Returns a
    (n, 32) uint8 CUDA tensor of digests (written asynchronously).  mode=1
    returns data roots (slab subtree roots) instead of digests."""
    n = len(tensors)
    dev = tensors[0].device
    if digests is None:
        digests = torch.empty((n, 32), dtype=torch.uint8, device=dev)
    arr = (TensorDesc * n)(*[_desc(t, digests[i], mode) for i, t in enumerate(tensors)])
    need = lib().verde_commit_workspace_bytes(arr, n)
    ws = ws or CommitWorkspace(dev)
    buf = ws.get(need)
    check(lib().verde_commit_tensors(arr, n, buf.data_ptr(), buf.numel(), _stream(stream)), "verde_commit_tensors")
    return digests


class CommitPlan:
    """verde_commit_plan_*: a prepared commit of a fixed list of tensors into
    fixed digest slots; run() only enqueues kernels."""

    def __init__(self, tensors, digests, modes=None, device=None, incremental=None):
        """incremental: {index: dict(leaves_out=..., base_leaves=..., dirty=...)} per tensor
        (verde_tensor_desc's incremental-commit fields; same digests)."""
        n = len(tensors)
        self.n = n
        modes = modes or [0] * n
        inc = incremental or {}
        self._keep = (list(tensors), digests, inc)
        arr = (TensorDesc * n)(*[_desc(t, digests[i], modes[i], **inc.get(i, {})) for i, t in enumerate(tensors)])
        need = lib().verde_commit_workspace_bytes(arr, n)
        dev = device or tensors[0].device
        self.ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        self.nbytes = sum(t.numel() * t.element_size() for t in tensors)
        h = C.c_void_p()
        check(lib().verde_commit_plan_create(arr, n, self.ws.data_ptr(), self.ws.numel(), C.byref(h)),
              "verde_commit_plan_create")
        self.h = h

    def run(self, stream=None):
        t0 = _TIMER.begin(stream) if _TIMER else None
        check(lib().verde_commit_plan_run(self.h, _stream(stream)), "verde_commit_plan_run")
        if t0 is not None:
            _TIMER.end("commit", t0, self.nbytes, stream)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().verde_commit_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass


class RootPlan:
    """verde_root_plan_*: node digests + RFC 6962 step root on the device.
    blob/offs/slots/soffs: host numpy arrays of the static node serialisation
    (copied to the device once); table: device uint8 [n_slots, 32]."""

    def __init__(self, blob, offs, slots, soffs, table, with_nodes=True):
        dev = table.device
        n = len(offs) - 1
        self.n = n
        self.blob = torch.from_numpy(blob).to(dev)
        self.offs = torch.from_numpy(offs).to(dev)
        self.slots = torch.from_numpy(slots).to(dev)
        self.soffs = torch.from_numpy(soffs).to(dev)
        self.table = table
        self.nodes = torch.zeros((n, 32), dtype=torch.uint8, device=dev) if with_nodes else None
        self.root = torch.zeros(32, dtype=torch.uint8, device=dev)
        self.ws = torch.empty(max(lib().verde_root_plan_workspace_bytes(n), 256), dtype=torch.uint8, device=dev)
        h = C.c_void_p()
        check(lib().verde_root_plan_create(n, self.blob.data_ptr(), self.offs.data_ptr(), self.slots.data_ptr(),
                                           self.soffs.data_ptr(), table.data_ptr(),
                                           self.nodes.data_ptr() if with_nodes else None, self.root.data_ptr(),
                                           self.ws.data_ptr(), self.ws.numel(), C.byref(h)), "verde_root_plan_create")
        self.h = h

    def run(self, stream=None):
        check(lib().verde_root_plan_run(self.h, _stream(stream)), "verde_root_plan_run")

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().verde_root_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass


def verde_commit_tensor(t, ws: CommitWorkspace | None = None, stream=None):
    return verde_commit_tensors([t], ws=ws, stream=stream)[0]


def verde_digest_from_subroots(subroots: bytes, dtype: int, shape, nbytes: int) -> bytes:
    """Digest of a tensor committed as k = len(subroots)/32 aligned slabs (mode=1)."""
    k = len(subroots) // 32
    dims = (C.c_int64 * max(len(shape), 1))(*shape)
    buf = C.create_string_buffer(bytes(subroots), max(len(subroots), 1))
    out = C.create_string_buffer(32)
    check(lib().verde_digest_from_subroots(buf, k, int(dtype), len(shape), dims, int(nbytes), out),
          "verde_digest_from_subroots")
    return out.raw


def gemm_num_cfgs() -> int:
    """Number of R-GEMM tile configurations (test hook: every one gives the same bits)."""
    return lib().repops_gemm_num_cfgs()


def launch_count() -> int:
    """Kernels enqueued by librepops.so in this process so far."""
    return lib().repops_launch_count()


def verde_merkle_root(digests: list[bytes] | bytes) -> bytes:
    blob = b"".join(digests) if isinstance(digests, list) else bytes(digests)
    n = len(blob) // 32
    buf = C.create_string_buffer(blob, max(len(blob), 1))
    out = C.create_string_buffer(32)
    check(lib().verde_merkle_root(buf, n, out), "verde_merkle_root")
    return out.raw


def verde_sha256(data: bytes) -> bytes:
    buf = C.create_string_buffer(bytes(data), max(len(data), 1))
    out = C.create_string_buffer(32)
    check(lib().verde_sha256(buf, len(data), out), "verde_sha256")
    return out.raw


def verde_node_digest(index, op, shard, attrs, inputs, dsts, in_digests, out_digests) -> bytes:
    """attrs: {key(int): value(u64)}; inputs: [(src_node, src_slot)]; dsts: [dst_node];
    in/out_digests: lists of 32-byte strings."""
    keys = sorted(attrs)
    nd = Node()
    nd.index, nd.op, nd.shard = index, op, shard
    ak = (C.c_uint32 * max(len(keys), 1))(*keys)
    av = (C.c_uint64 * max(len(keys), 1))(*[attrs[k] for k in keys])
    nd.n_attr, nd.attr_keys, nd.attr_vals = len(keys), C.cast(ak, C.c_void_p), C.cast(av, C.c_void_p)
    sn = (C.c_uint32 * max(len(inputs), 1))(*[s for s, _ in inputs])
    ss = (C.c_uint32 * max(len(inputs), 1))(*[q for _, q in inputs])
    ind = C.create_string_buffer(b"".join(in_digests), max(32 * len(in_digests), 1))
    nd.n_in, nd.in_src_node, nd.in_src_slot = len(inputs), C.cast(sn, C.c_void_p), C.cast(ss, C.c_void_p)
    nd.in_digests = C.cast(ind, C.c_void_p)
    dn = (C.c_uint32 * max(len(dsts), 1))(*dsts)
    nd.n_dst, nd.dst_nodes = len(dsts), C.cast(dn, C.c_void_p)
    outd = C.create_string_buffer(b"".join(out_digests), max(32 * len(out_digests), 1))
    nd.n_out, nd.out_digests = len(out_digests), C.cast(outd, C.c_void_p)
    out = C.create_string_buffer(32)
    check(lib().verde_node_digest(C.byref(nd), out), "verde_node_digest")
    return out.raw


def verde_first_divergence(seq0: bytes, seq1: bytes, hashed=False) -> tuple[int, int]:
    """(first differing index or -1, number of subtree comparisons); hashed: the
    items are leaf hashes (verde_first_divergence_hashed)."""
    n = len(seq0) // 32
    a = C.create_string_buffer(bytes(seq0), max(len(seq0), 1))
    b = C.create_string_buffer(bytes(seq1), max(len(seq1), 1))
    d = C.c_int64()
    r = C.c_int64()
    fn = lib().verde_first_divergence_hashed if hashed else lib().verde_first_divergence
    check(fn(a, b, n, C.byref(d), C.byref(r)), "verde_first_divergence")
    return d.value, r.value


def verde_merkle_root_hashed(leaf_hashes: bytes) -> bytes:
    """RFC 6962 MTH over leaf hashes (= the R11 data root of a tensor's chunk leaves)."""
    blob = bytes(leaf_hashes)
    buf = C.create_string_buffer(blob, max(len(blob), 1))
    out = C.create_string_buffer(32)
    check(lib().verde_merkle_root_hashed(buf, len(blob) // 32, out), "verde_merkle_root_hashed")
    return out.raw


def verde_merkle_audit_path(items: bytes, m: int, hashed=False) -> list[bytes]:
    """RFC 6962 audit path of item m (membership proof)."""
    blob = bytes(items)
    buf = C.create_string_buffer(blob, max(len(blob), 1))
    path = C.create_string_buffer(64 * 32)
    ln = C.c_int32()
    check(lib().verde_merkle_audit_path(buf, len(blob) // 32, int(m), int(bool(hashed)), path, C.byref(ln)),
          "verde_merkle_audit_path")
    return [path.raw[32 * i:32 * i + 32] for i in range(ln.value)]


def verde_merkle_verify_path(leaf_hash: bytes, m: int, n: int, path: list[bytes], root: bytes) -> bool:
    """RFC 9162 inclusion check of leaf_hash at index m of an n-leaf tree with `root`."""
    p = b"".join(path)
    pb = C.create_string_buffer(p, max(len(p), 1))
    ok = C.c_int()
    check(lib().verde_merkle_verify_path(bytes(leaf_hash), int(m), int(n), pb, len(path), bytes(root), C.byref(ok)),
          "verde_merkle_verify_path")
    return bool(ok.value)


def verde_tensor_digest_from_root(data_root: bytes, dtype: int, dims, nbytes: int) -> bytes:
    dims = list(dims)
    arr = (C.c_int64 * max(len(dims), 1))(*dims)
    out = C.create_string_buffer(32)
    check(lib().verde_tensor_digest_from_root(bytes(data_root), int(dtype), len(dims), arr, int(nbytes), out),
          "verde_tensor_digest_from_root")
    return out.raw


def verde_chunk_leaves(t, stream=None):
    """uint8 [ceil(nbytes/4096), 32] device tensor of the R11 chunk leaf hashes of t."""
    if not t.is_contiguous():
        raise RepopsError("verde_chunk_leaves: tensor must be contiguous")
    nbytes = t.numel() * t.element_size()
    out = torch.empty(((nbytes + 4095) // 4096, 32), dtype=torch.uint8, device=t.device)
    check(lib().verde_chunk_leaves(_p(t), nbytes, _p(out), _stream(stream)), "verde_chunk_leaves")
    return out
