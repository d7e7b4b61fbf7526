"""CPU oracle for the RepOps hot path (arXiv 2502.19405, Sec. 3 "RepOps" and
Sec. 2.2 commitments).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs are the only permitted users.
The product package ``paper_2502_19405_b200`` never imports this module, and
this module never imports the product.  The two share no code; the only
common dependency is ``synth`` (seeded input generation, no method arithmetic).

The arithmetic lives in ``repops_oracle.c`` (plain single-threaded C, built
with ``-O2 -ffp-contract=off -fno-fast-math``).  This file only builds/loads it
and marshals numpy arrays.  Each wrapper names the C function (and through it
the paper passage) it calls.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "repops_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fno-strict-aliasing",
          "-std=c11", "-fPIC", "-shared"]
# REPOPS_ORACLE_SANITIZE=1: an AddressSanitizer + UndefinedBehaviorSanitizer build of the same
# source (tests/test_oracle_sanitizers.py runs the oracle test suite against it; the process
# needs libasan preloaded).  Same arithmetic flags, so the same bits.
if os.environ.get("REPOPS_ORACLE_SANITIZE") == "1":
    _LIB = os.path.join(_HERE, "liboracle_san.so")
    CFLAGS = ["-O1", "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined",
              "-fno-sanitize-recover=all", "-ffp-contract=off", "-fno-fast-math", "-fno-strict-aliasing",
              "-std=c11", "-fPIC", "-shared"]

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/liboracle.so (plain gcc)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            i64, f32, i32, vp = C.c_int64, C.c_float, C.c_int, C.c_void_p
            sig = {
                "orc_fpenv_ok": (i32, []),
                "orc_gemm": (None, [i64, i64, i64, vp, i64, i32, vp, i64, i32, i32, vp, f32, vp, i64]),
                "orc_csum": (f32, [vp, i64, i64]),
                "orc_cdot": (f32, [vp, vp, i64]),
                "orc_sum_rows": (None, [vp, i64, i64, i64, vp]),
                "orc_sum_cols_seq": (None, [vp, i64, i64, i64, i64, vp]),
                "orc_exp": (f32, [f32]),
                "orc_log": (f32, [f32]),
                "orc_tanh": (f32, [f32]),
                "orc_rsqrt": (f32, [f32]),
                "orc_exp_vec": (None, [vp, i64, vp]),
                "orc_log_vec": (None, [vp, i64, vp]),
                "orc_tanh_vec": (None, [vp, i64, vp]),
                "orc_rsqrt_vec": (None, [vp, i64, vp]),
                "orc_add": (None, [vp, vp, i64, vp]),
                "orc_gelu": (None, [vp, i64, vp]),
                "orc_relu": (None, [vp, i64, vp]),
                "orc_sin_vec": (None, [vp, i64, vp]),
                "orc_erf_vec": (None, [vp, i64, vp]),
                "orc_philox4x32_10": (None, [vp, vp, vp]),
                "orc_convert": (None, [vp, i32, i64, i64, i64, vp, i32, i64]),
                "orc_gemm_ex": (None, [i64, i64, i64, vp, i32, i64, i32, vp, i32, i64, i32, i32, vp, f32, vp, i32,
                                       i64]),
                "orc_rand_uniform": (None, [C.c_uint64, C.c_uint64, i64, vp]),
                "orc_dropout": (None, [vp, i64, f32, C.c_uint64, C.c_uint64, vp, vp]),
                "orc_dropout_backward": (None, [vp, i64, f32, C.c_uint64, C.c_uint64, vp]),
                "orc_gelu_erf": (None, [vp, i64, vp]),
                "orc_gelu_erf_backward": (None, [vp, vp, i64, vp]),
                "orc_cos_vec": (None, [vp, i64, vp]),
                "orc_rope_tables": (None, [vp, i64, i64, vp, vp]),
                "orc_relu_backward": (None, [vp, vp, i64, vp]),
                "orc_gelu_backward": (None, [vp, vp, i64, vp]),
                "orc_softmax": (None, [vp, i64, i64, i64, i32, vp, i64]),
                "orc_softmax_backward": (None, [vp, i64, vp, i64, i64, i64, f32, vp, i64]),
                "orc_layernorm": (None, [vp, vp, vp, i64, i64, f32, vp, vp, vp]),
                "orc_layernorm_backward": (None, [vp, vp, vp, vp, vp, vp, i64, i64, vp]),
                "orc_layernorm_backward_params": (None, [vp, vp, vp, vp, i64, i64, i64, vp, vp]),
                "orc_cross_entropy": (None, [vp, i64, i64, i64, vp, f32, vp, vp, i64]),
                "orc_embedding": (None, [vp, i64, i64, vp, vp, i64, vp]),
                "orc_embedding_backward": (None, [vp, i64, i64, vp, i64, vp, vp]),
                "orc_tree_sum": (None, [vp, i32, i64, vp]),
                "orc_adamw": (None, [vp, vp, vp, vp, i64, i64, f32, f32, f32, f32, f32, i32]),
                "orc_sha256": (None, [vp, i64, vp]),
                "orc_merkle_root": (i32, [vp, i64, vp]),
                "orc_commit_tensor": (None, [vp, i64, i32, i32, vp, vp]),
                "orc_data_root": (None, [vp, i64, vp]),
                "orc_mth": (None, [vp, vp, i64, vp]),
                "orc_rmsnorm": (None, [vp, vp, i64, i64, f32, vp, vp]),
                "orc_swiglu": (None, [vp, vp, i64, vp]),
                "orc_rope": (None, [vp, i64, i64, i64, i64, vp, vp, vp, i64]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
            if not L.orc_fpenv_ok():
                raise RuntimeError("oracle: MXCSR has FTZ/DAZ set or non-RN rounding")
    return _lib


# ------------------------------------------------------------------ marshalling
def _f32(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def f2u(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def u2f(a) -> np.ndarray:
    return np.asarray(a, dtype=np.uint32).view(np.float32)


# ------------------------------------------------------------------ R-GEMM
def gemm(A, B, transA=False, transB=False, epi=0, bias=None, scale=1.0, M=None, N=None, K=None):
    """R-GEMM (orc_gemm).  A is (M,K) or, if transA, (K,M);
    B is (K,N) or, if transB, (N,K).  epi 0/1/2 = none/bias/scale."""
    A = _f32(A)
    B = _f32(B)
    if M is None:
        M = A.shape[1] if transA else A.shape[0]
        K = A.shape[0] if transA else A.shape[1]
        N = B.shape[0] if transB else B.shape[1]
    Cm = np.empty((M, N), dtype=np.float32)
    b = _f32(bias) if bias is not None else None
    lib().orc_gemm(M, N, K, _p(A), A.shape[1] if A.ndim == 2 else 1, int(transA),
                   _p(B), B.shape[1] if B.ndim == 2 else 1, int(transB), int(epi),
                   _p(b) if b is not None else None, float(scale), _p(Cm), N)
    return Cm


def gemm_element(A, B, i, j, transA=False, transB=False, epi=0, bias=None, scale=1.0):
    """One output element C[i,j] of R-GEMM (a full K fold), for sampled parity."""
    A = _f32(A)
    B = _f32(B)
    K = A.shape[0] if transA else A.shape[1]
    lda = A.shape[1]
    ldb = B.shape[1]
    i, j = int(i), int(j)
    a_off = i if transA else i * lda
    b_off = j * ldb if transB else j
    out = np.empty((1, 1), dtype=np.float32)
    bb = None if bias is None else _f32(np.asarray(bias)[j:j + 1])
    pa = C.c_void_p(A.ctypes.data + 4 * a_off)
    pb = C.c_void_p(B.ctypes.data + 4 * b_off)
    lib().orc_gemm(1, 1, K, pa, lda, int(transA), pb, ldb, int(transB), int(epi),
                   _p(bb) if bb is not None else None, float(scale), _p(out), 1)
    return out[0, 0]


# ------------------------------------------------------------------ reductions
def csum(x) -> np.float32:
    """R-CSUM (orc_csum; P:588-590 + reading R4)."""
    x = _f32(x).ravel()
    return np.float32(lib().orc_csum(_p(x), x.size, 1))


def cdot(u, v) -> np.float32:
    u = _f32(u).ravel()
    v = _f32(v).ravel()
    assert u.size == v.size
    return np.float32(lib().orc_cdot(_p(u), _p(v), u.size))


def sum_rows(x):
    x = _f32(x)
    out = np.empty(x.shape[0], dtype=np.float32)
    lib().orc_sum_rows(_p(x), x.shape[0], x.shape[1], x.shape[1], _p(out))
    return out


def sum_cols_seq(x, nseg=1):
    """R-SEQ column folds, rows split into nseg contiguous segments."""
    x = _f32(x)
    out = np.empty((nseg, x.shape[1]), dtype=np.float32)
    lib().orc_sum_cols_seq(_p(x), x.shape[0], x.shape[1], x.shape[1], nseg, _p(out))
    return out


# ------------------------------------------------------------------ math
def _vec(name, x):
    x = _f32(x)
    y = np.empty_like(x)
    getattr(lib(), name)(_p(x), x.size, _p(y))
    return y


def exp(x):
    return _vec("orc_exp_vec", x)


def log(x):
    return _vec("orc_log_vec", x)


def tanh(x):
    return _vec("orc_tanh_vec", x)


def rsqrt(x):
    return _vec("orc_rsqrt_vec", x)


def gelu(x):
    return _vec("orc_gelu", x)


def gelu_backward(x, dy):
    x = _f32(x)
    dy = _f32(dy)
    dx = np.empty_like(x)
    lib().orc_gelu_backward(_p(x), _p(dy), x.size, _p(dx))
    return dx


def erf(x):
    """orc_erf (Cephes erff / erfcf chain, reading R27)."""
    return _vec("orc_erf_vec", x)


def gelu_erf(x):
    """orc_gelu_erf: exact GELU 0.5 x (1 + erf(x / sqrt 2)) (reading R27)."""
    return _vec("orc_gelu_erf", x)


def gelu_erf_backward(x, dy):
    """orc_gelu_erf_backward (reading R27)."""
    x = _f32(x)
    dy = _f32(dy)
    dx = np.empty_like(x)
    lib().orc_gelu_erf_backward(_p(x), _p(dy), x.size, _p(dx))
    return dx


_DT_CODE = {"f32": 1, "bf16": 4, "f16": 5}


def convert(x, src, dst):
    """orc_convert (reading R30): x is a 2-D array of the storage type's bit patterns
    (float32 for "f32", uint16 for "bf16" / "f16"); returns dst's bit patterns."""
    x = np.ascontiguousarray(x, dtype=np.float32 if src == "f32" else np.uint16)
    x2 = x.reshape(-1, x.shape[-1]) if x.ndim else x.reshape(1, 1)
    out = np.empty(x2.shape, dtype=np.float32 if dst == "f32" else np.uint16)
    lib().orc_convert(_p(x2), _DT_CODE[src], x2.shape[0], x2.shape[1], x2.shape[1], _p(out), _DT_CODE[dst],
                      x2.shape[1])
    return out.reshape(x.shape)


def gemm_ex(A, adt, B, bdt, cdt, transA=False, transB=False, epi=0, bias=None, scale=1.0):
    """orc_gemm_ex (reading R30): stored-precision operands, binary32 R-GEMM, narrowed C."""
    A = np.ascontiguousarray(A, dtype=np.float32 if adt == "f32" else np.uint16)
    B = np.ascontiguousarray(B, dtype=np.float32 if bdt == "f32" else np.uint16)
    M = A.shape[1] if transA else A.shape[0]
    K = A.shape[0] if transA else A.shape[1]
    N = B.shape[0] if transB else B.shape[1]
    Cm = np.empty((M, N), dtype=np.float32 if cdt == "f32" else np.uint16)
    b = _f32(bias) if bias is not None else None
    lib().orc_gemm_ex(M, N, K, _p(A), _DT_CODE[adt], A.shape[1], int(transA), _p(B), _DT_CODE[bdt], B.shape[1],
                      int(transB), int(epi), _p(b) if b is not None else None, float(scale), _p(Cm), _DT_CODE[cdt], N)
    return Cm


def philox4x32_10(ctr, key):
    """orc_philox4x32_10: one Philox4x32-10 block (reading R28)."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.empty(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def rand_uniform(seed, stream, n):
    """orc_rand_uniform: u_i in [0, 1) on the 2^-24 grid (reading R28)."""
    y = np.empty(n, np.float32)
    lib().orc_rand_uniform(seed, stream, n, _p(y))
    return y


def dropout(x, p, seed, stream):
    """orc_dropout -> (y, mask) (reading R28)."""
    x = _f32(x)
    y = np.empty_like(x)
    m = np.empty(x.size, np.uint8)
    lib().orc_dropout(_p(x), x.size, p, seed, stream, _p(y), _p(m))
    return y, m


def dropout_backward(dy, p, seed, stream):
    """orc_dropout_backward (reading R28)."""
    dy = _f32(dy)
    dx = np.empty_like(dy)
    lib().orc_dropout_backward(_p(dy), dy.size, p, seed, stream, _p(dx))
    return dx


def sin(x):
    """orc_sin (Cephes sinf chain, reading R26)."""
    return _vec("orc_sin_vec", x)


def cos(x):
    """orc_cos (Cephes cosf chain, reading R26)."""
    return _vec("orc_cos_vec", x)


def rope_tables_from_inv_freq(inv_freq, T):
    """orc_rope_tables: (cos, sin) [T, h] of angle fmul(t, inv_freq[i]) (reading R26)."""
    f = _f32(inv_freq)
    h = f.size
    c = np.empty((T, h), np.float32)
    s = np.empty((T, h), np.float32)
    lib().orc_rope_tables(_p(f), T, h, _p(c), _p(s))
    return c, s


def relu(x):
    """orc_relu (reading R24)."""
    return _vec("orc_relu", x)


def relu_backward(x, g):
    """orc_relu_backward (reading R24; subgradient 0 at x = 0)."""
    x = _f32(x)
    g = _f32(g)
    dx = np.empty_like(x)
    lib().orc_relu_backward(_p(x), _p(g), x.size, _p(dx))
    return dx


def add(a, b):
    a = _f32(a)
    b = _f32(b)
    y = np.empty_like(a)
    lib().orc_add(_p(a), _p(b), a.size, _p(y))
    return y


# ------------------------------------------------------------------ row ops
def softmax(x, causal=False):
    x = _f32(x)
    y = np.empty_like(x)
    lib().orc_softmax(_p(x), x.shape[0], x.shape[1], x.shape[1], int(causal), _p(y), x.shape[1])
    return y


def softmax_backward(y, dy, scale=1.0):
    y = _f32(y)
    dy = _f32(dy)
    dx = np.empty_like(y)
    r, c = y.shape
    lib().orc_softmax_backward(_p(y), c, _p(dy), c, r, c, float(scale), _p(dx), c)
    return dx


def layernorm(x, gamma, beta, eps=1e-5):
    x = _f32(x)
    g = _f32(gamma)
    b = _f32(beta)
    r, c = x.shape
    y = np.empty_like(x)
    mean = np.empty(r, np.float32)
    rstd = np.empty(r, np.float32)
    lib().orc_layernorm(_p(x), _p(g), _p(b), r, c, float(eps), _p(y), _p(mean), _p(rstd))
    return y, mean, rstd


def layernorm_backward(dy, x, gamma, mean, rstd, dres=None):
    dy, x, g, mean, rstd = map(_f32, (dy, x, gamma, mean, rstd))
    r, c = x.shape
    dx = np.empty_like(x)
    dr = _f32(dres) if dres is not None else None
    lib().orc_layernorm_backward(_p(dy), _p(x), _p(g), _p(mean), _p(rstd),
                                 _p(dr) if dr is not None else None, r, c, _p(dx))
    return dx


def layernorm_backward_params(dy, x, mean, rstd, nseg=1):
    dy, x, mean, rstd = map(_f32, (dy, x, mean, rstd))
    r, c = x.shape
    dg = np.empty((nseg, c), np.float32)
    db = np.empty((nseg, c), np.float32)
    lib().orc_layernorm_backward_params(_p(dy), _p(x), _p(mean), _p(rstd), r, c, nseg, _p(dg), _p(db))
    return dg, db


def rmsnorm(x, w, eps=1e-5):
    """R-RMSNORM (orc_rmsnorm).  Returns (y, rstd)."""
    x = _f32(x)
    w = _f32(w)
    r, c = x.shape
    y = np.empty_like(x)
    rs = np.empty(r, np.float32)
    lib().orc_rmsnorm(_p(x), _p(w), r, c, float(eps), _p(y), _p(rs))
    return y, rs


def swiglu(g, u):
    """R-SWIGLU: silu(g) * u elementwise (orc_swiglu)."""
    g = _f32(g)
    u = _f32(u)
    h = np.empty_like(g)
    lib().orc_swiglu(_p(g), _p(u), g.size, _p(h))
    return h


def rope(x, cos, sin, nhead, hd):
    """R-ROPE on x [ntok, nhead*hd] (rows = tokens) with tables [ntok, hd/2]."""
    x = _f32(x)
    cos = _f32(cos)
    sin = _f32(sin)
    y = np.empty_like(x)
    lib().orc_rope(_p(x), x.shape[0], nhead, hd, x.shape[1], _p(cos), _p(sin), _p(y), x.shape[1])
    return y


def cross_entropy(logits, labels, scale=1.0, want_grad=True):
    x = _f32(logits)
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    r, V = x.shape
    loss = np.empty(r, np.float32)
    d = np.empty_like(x) if want_grad else None
    lib().orc_cross_entropy(_p(x), r, V, V, _p(lab), float(scale), _p(loss),
                            _p(d) if d is not None else None, V)
    return loss, d


def embedding(tok, wte, wpe, T):
    tok = np.ascontiguousarray(tok, dtype=np.int32)
    wte = _f32(wte)
    wpe = _f32(wpe)
    Cc = wte.shape[1]
    x0 = np.empty((tok.size, Cc), np.float32)
    lib().orc_embedding(_p(tok), tok.size, T, _p(wte), _p(wpe), Cc, _p(x0))
    return x0


def embedding_backward(tok, dx0, T, dwte, dwpe=None):
    """Accumulates into (copies of) dwte / dwpe; returns them."""
    tok = np.ascontiguousarray(tok, dtype=np.int32)
    dx0 = _f32(dx0)
    dwte = _f32(dwte).copy()
    dwpe = _f32(dwpe).copy() if dwpe is not None else None
    lib().orc_embedding_backward(_p(tok), tok.size, T, _p(dx0), dx0.shape[1], _p(dwte),
                                 _p(dwpe) if dwpe is not None else None)
    return dwte, dwpe


def tree_sum(parts):
    """R-TREE_S over a list of equally shaped arrays (len = power of two)."""
    parts = [_f32(p) for p in parts]
    n = parts[0].size
    arr = (C.c_void_p * len(parts))(*[p.ctypes.data for p in parts])
    out = np.empty_like(parts[0])
    lib().orc_tree_sum(arr, len(parts), n, _p(out))
    return out


def adamw(p, g, m, v, step, lr, b1, b2, eps, wd, decay):
    p = _f32(p).copy()
    m = _f32(m).copy()
    v = _f32(v).copy()
    g = _f32(g)
    lib().orc_adamw(_p(p), _p(g), _p(m), _p(v), p.size, int(step), float(lr), float(b1),
                    float(b2), float(eps), float(wd), int(decay))
    return p, m, v


# ------------------------------------------------------------------ hashing
def _bytes(b) -> np.ndarray:
    if isinstance(b, (bytes, bytearray)):
        return np.frombuffer(bytes(b), dtype=np.uint8).copy() if len(b) else np.zeros(1, np.uint8)
    return np.ascontiguousarray(b).view(np.uint8).ravel()


def sha256(b) -> bytes:
    n = len(b) if isinstance(b, (bytes, bytearray)) else np.asarray(b).nbytes
    arr = _bytes(b)
    out = np.empty(32, np.uint8)
    lib().orc_sha256(_p(arr), n, _p(out))
    return out.tobytes()


def merkle_root(digests) -> bytes:
    """R-MERKLE: RFC 6962 MTH over 32-byte entries; raises on n == 0."""
    arr = np.frombuffer(b"".join(digests), dtype=np.uint8).copy() if digests else np.zeros(1, np.uint8)
    out = np.empty(32, np.uint8)
    if lib().orc_merkle_root(_p(arr), len(digests), _p(out)) != 0:
        raise ValueError("merkle_root: empty leaf list")
    return out.tobytes()


def mth(entries) -> bytes:
    """RFC 6962 MTH over variable-length byte-string entries (orc_mth)."""
    blob = b"".join(entries)
    off = np.zeros(len(entries) + 1, np.int64)
    for i, e in enumerate(entries):
        off[i + 1] = off[i] + len(e)
    buf = np.frombuffer(blob, np.uint8).copy() if blob else np.zeros(1, np.uint8)
    out = np.empty(32, np.uint8)
    lib().orc_mth(_p(buf), _p(off), len(entries), _p(out))
    return out.tobytes()


def data_root(t) -> bytes:
    arr = np.asarray(t)
    arr = arr if arr.flags.c_contiguous else arr.copy()  # (ascontiguousarray would make 0-d into 1-d)
    n = arr.nbytes
    buf = arr.reshape(-1).view(np.uint8) if n else np.zeros(1, np.uint8)
    out = np.empty(32, np.uint8)
    lib().orc_data_root(_p(buf), n, _p(out))
    return out.tobytes()


DTYPE_F32 = 1
DTYPE_I32 = 2


def commit_tensor(t, dtype_code=None) -> bytes:
    """R-TCOMMIT digest of an array (shape = its numpy shape)."""
    arr = np.asarray(t)
    arr = arr if arr.flags.c_contiguous else arr.copy()  # (ascontiguousarray would make 0-d into 1-d)
    if dtype_code is None:
        dtype_code = {np.dtype(np.float32): DTYPE_F32, np.dtype(np.int32): DTYPE_I32}[arr.dtype]
    dims = np.asarray(arr.shape, dtype=np.int64) if arr.ndim else np.zeros(1, np.int64)
    n = arr.nbytes
    buf = arr.reshape(-1).view(np.uint8) if n else np.zeros(1, np.uint8)
    out = np.empty(32, np.uint8)
    lib().orc_commit_tensor(_p(buf), n, int(dtype_code), arr.ndim, _p(dims), _p(out))
    return out.tobytes()
