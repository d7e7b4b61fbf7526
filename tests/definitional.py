"""Definitional transcription of the canonical operator readings -- TEST ONLY.

A second, independent statement of the op sequences that SURVEY.md §8(c) and
DESIGN.md §3 fix (R-EXP, R-LOG, R-TANH, R-GELU fwd/bwd, R-CSUM/R-CDOT,
R-SOFTMAX fwd/bwd, R-LN fwd/bwd, R-CE, R-ADAMW), written op by op from that text
in numpy binary32 (every numpy float32 +, -, *, /, sqrt is one IEEE-754
round-to-nearest-even operation; numpy never contracts a*b+c) plus `fma32`, an
exactly rounded binary32 fused multiply-add built below from float64 error-free
transformations.  It shares nothing with oracle/repops_oracle.c (different
language, vectorised across elements, its own constants typed from the text) and
nothing with the CUDA path.  tests/test_oracle_definitional.py compares the two
bit for bit, so a drift in the oracle's op order (a divide instead of a
reciprocal-multiply, an unfused LN affine, a mistyped polynomial coefficient) fails.

Elementwise functions take/return float32 arrays; row operators take one row.
"""
from __future__ import annotations

import numpy as np

f32 = np.float32


def F(bits: int) -> np.float32:
    """a binary32 constant given by its bit pattern"""
    return np.array([bits], np.uint32).view(np.float32)[0]


# ---------------------------------------------------------------------- exact fma
def fma32(a, b, c):
    """Correctly rounded binary32 fma(a, b, c) (one rounding), vectorised.

    a*b of two binary32 values is exact in binary64 (48 significant bits).  The sum
    p + c is formed in binary64 with round-to-ODD (TwoSum gives the exact error e;
    when e != 0 the truncated sum's last bit is forced to 1); a round-to-odd result
    with >= 24 + 2 bits rounds to binary32 exactly as the real sum would (the
    classic round-to-odd double-rounding theorem), gradual underflow included.
    Non-finite operands fall back to binary64 arithmetic (same IEEE special-value
    rules).  Pinned against the exact-rational model tests/ieee_sim.fma."""
    a = np.asarray(a, np.float32).astype(np.float64)
    b = np.asarray(b, np.float32).astype(np.float64)
    c = np.asarray(c, np.float32).astype(np.float64)
    a, b, c = np.broadcast_arrays(a, b, c)
    with np.errstate(all="ignore"):
        p = a * b
        s = p + c
        bb = s - p
        e = (p - (s - bb)) + (c - bb)
        sb = np.ascontiguousarray(s).view(np.uint64).copy()
        finite = np.isfinite(s) & np.isfinite(p) & np.isfinite(c)
        inexact = finite & (e != 0)
        # |exact| < |s| when e has the opposite sign of s: truncation is one step toward 0
        away = inexact & ((e < 0) != (s < 0))
        sb = np.where(away, sb - np.uint64(1), sb)
        sb = np.where(inexact, sb | np.uint64(1), sb)
        r = sb.view(np.float64).astype(np.float32)
    return r


def fmul(a, b):
    with np.errstate(all="ignore"):
        return (np.asarray(a, np.float32) * np.asarray(b, np.float32)).astype(np.float32)


def fadd(a, b):
    with np.errstate(all="ignore"):
        return (np.asarray(a, np.float32) + np.asarray(b, np.float32)).astype(np.float32)


def fsub(a, b):
    with np.errstate(all="ignore"):
        return (np.asarray(a, np.float32) - np.asarray(b, np.float32)).astype(np.float32)


def fdiv(a, b):
    with np.errstate(all="ignore"):
        return (np.asarray(a, np.float32) / np.asarray(b, np.float32)).astype(np.float32)


def fsqrt(a):
    with np.errstate(all="ignore"):
        return np.sqrt(np.asarray(a, np.float32)).astype(np.float32)


CANON_NAN = F(0x7FC00000)


def canon(x):
    x = np.asarray(x, np.float32)
    return np.where(np.isnan(x), CANON_NAN, x).astype(np.float32)


# ---------------------------------------------------------------------- R-EXP
def exp(x):
    """SURVEY §8(c) R-EXP steps 1-6 (Cephes expf constants, P:571-574 / R5)."""
    x = np.asarray(x, np.float32)
    with np.errstate(all="ignore"):
        t = fmul(x, F(0x3FB8AA3B))                                   # log2(e)
        kf = fsub(fadd(t, f32(12582912.0)), f32(12582912.0))          # RN-even integer
        r = fma32(kf, f32(-0.693359375), x)
        r = fma32(kf, f32(2.12194440e-4), r)
        p = np.full_like(x, f32(1.9875691500E-4))
        for c in (1.3981999507E-3, 8.3334519073E-3, 4.1665795894E-2, 1.6666665459E-1, 5.0000001201E-1):
            p = fma32(p, r, f32(c))
        y = fadd(fma32(p, fmul(r, r), r), f32(1.0))
        k = np.where(np.isfinite(kf), kf, 0).astype(np.int64)
        k1 = k >> 1
        k2 = k - k1
        pw = lambda q: np.clip(q + 127, 0, 255).astype(np.uint32) << np.uint32(23)  # noqa: E731  2^q
        y = fmul(fmul(y, pw(k1).view(np.float32)), pw(k2).view(np.float32))
    y = np.where(x > f32(89.0), f32(np.inf), y)
    y = np.where(x < f32(-104.0), f32(0.0), y)
    return canon(np.where(np.isnan(x), CANON_NAN, y))


# ---------------------------------------------------------------------- R-LOG
LOG_C = (-1.1514610310E-1, 1.1676998740E-1, -1.2420140846E-1, 1.4249322787E-1, -1.6668057665E-1,
         2.0000714765E-1, -2.4999993993E-1, 3.3333331174E-1)


def log(x, coeffs=LOG_C):
    """SURVEY §8(c) R-LOG (Cephes logf, R5)."""
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.int64)
    sub = (u & 0x7F800000) == 0
    xs = np.where(sub, fmul(x, f32(2.0 ** 23)), x)
    us = xs.view(np.uint32).astype(np.int64)
    e = ((us >> 23) & 0xFF) - 126 - np.where(sub, 23, 0)
    m = ((us & 0x007FFFFF) | 0x3F000000).astype(np.uint32).view(np.float32)
    lo = m < f32(0.70710678)
    e = np.where(lo, e - 1, e)
    m = np.where(lo, fadd(m, m), m)
    f = fsub(m, f32(1.0))
    z = fmul(f, f)
    p = np.full_like(f, f32(7.0376836292E-2))
    for c in coeffs:
        p = fma32(p, f, f32(c))
    ef = e.astype(np.float32)
    y = fmul(fmul(p, f), z)
    y = fma32(ef, f32(-2.12194440e-4), y)
    y = fma32(z, f32(-0.5), y)
    y = fadd(f, y)
    y = fma32(ef, f32(0.693359375), y)
    y = np.where(x == 0, f32(-np.inf), y)
    y = np.where(x == np.inf, f32(np.inf), y)
    y = np.where((x < 0) | np.isnan(x), CANON_NAN, y)
    return y.astype(np.float32)


# ---------------------------------------------------------------------- R-TANH
def tanh(u):
    """SURVEY §8(c) R-TANH (small branch: Cephes tanhf polynomial; large: 1 - 2/(e^2a + 1))."""
    u = np.asarray(u, np.float32)
    a = np.abs(u)
    z = fmul(u, u)
    p = np.full_like(u, f32(-5.70498872745E-3))
    for c in (2.06390887954E-2, -5.37397155531E-2, 1.33314422036E-1, -3.33332819422E-1):
        p = fma32(p, z, f32(c))
    small = fma32(fmul(p, z), a, a)
    aa = np.minimum(a, f32(44.0))
    e = exp(fadd(aa, aa))
    large = fsub(f32(1.0), fdiv(f32(2.0), fadd(e, f32(1.0))))
    t = np.where(a < f32(0.625), small, large)
    t = np.copysign(t, u).astype(np.float32)
    return np.where(np.isnan(u), CANON_NAN, t).astype(np.float32)


# ---------------------------------------------------------------------- R-GELU (R16)
GELU_A, GELU_S, GELU_3A = F(0x3D372713), F(0x3F4C422A), F(0x3E095D4F)   # 0.044715, sqrt(2/pi), 3*0.044715


def gelu(x):
    x = np.asarray(x, np.float32)
    x2 = fmul(x, x)
    x3 = fmul(x2, x)
    inner = fma32(GELU_A, x3, x)
    u = fmul(GELU_S, inner)
    t = tanh(u)
    return canon(fmul(fmul(f32(0.5), x), fadd(f32(1.0), t)))


def gelu_backward(x, dy):
    x = np.asarray(x, np.float32)
    x2 = fmul(x, x)
    x3 = fmul(x2, x)
    t = tanh(fmul(GELU_S, fma32(GELU_A, x3, x)))
    di = fma32(GELU_3A, x2, f32(1.0))
    s2 = fsub(f32(1.0), fmul(t, t))
    g = fadd(fmul(f32(0.5), fadd(f32(1.0), t)), fmul(fmul(fmul(f32(0.5), x), s2), fmul(GELU_S, di)))
    return canon(fmul(dy, g))


# ---------------------------------------------------------------------- R-CSUM / R-CDOT (R4)
SLOTS, TILE = 128, 4096


def _tree128(p):
    p = p.copy()
    h = 64
    while h >= 1:
        p[:h] = fadd(p[:h], p[h:2 * h])
        h //= 2
    return p[0]


def csum(x):
    x = np.asarray(x, np.float32).ravel()
    n = x.size
    if n > TILE:
        return csum(np.array([csum(x[t:t + TILE]) for t in range(0, n, TILE)], np.float32))
    p = np.zeros(SLOTS, np.float32)
    for i0 in range(0, n, SLOTS):  # slot i % 128 folds x[i] in ascending i (one slot per lane of the chunk)
        blk = x[i0:i0 + SLOTS]
        p[:blk.size] = fadd(p[:blk.size], blk)
    return _tree128(p)


def cdot(u, v):
    u = np.asarray(u, np.float32).ravel()
    v = np.asarray(v, np.float32).ravel()
    n = u.size
    if n > TILE:
        return csum(np.array([cdot(u[t:t + TILE], v[t:t + TILE]) for t in range(0, n, TILE)], np.float32))
    p = np.zeros(SLOTS, np.float32)
    for i0 in range(0, n, SLOTS):
        k = min(SLOTS, n - i0)
        p[:k] = fma32(u[i0:i0 + k], v[i0:i0 + k], p[:k])
    return _tree128(p)


def seq(x):
    """R-SEQ: ascending fold from +0 along axis 0"""
    x = np.asarray(x, np.float32)
    acc = np.zeros(x.shape[1:], np.float32)
    for t in range(x.shape[0]):
        acc = fadd(acc, x[t])
    return acc


# ---------------------------------------------------------------------- R-SOFTMAX (R7)
def softmax_row(x, valid=None):
    x = np.asarray(x, np.float32)
    n = x.size if valid is None else valid
    m = np.max(x[:n])
    e = exp(fsub(x[:n], m))
    s = csum(e)
    r = fdiv(f32(1.0), s)
    y = np.zeros_like(x)
    y[:n] = fmul(e, r)
    return canon(y)


def softmax_backward_row(y, dy, scale=1.0):
    c = cdot(y, dy)
    dx = fmul(y, fsub(dy, c))
    if scale != 1.0:
        dx = fmul(dx, f32(scale))
    return canon(dx)


# ---------------------------------------------------------------------- R-LN (R8)
def layernorm_row(x, g, b, eps=1e-5):
    x = np.asarray(x, np.float32)
    n = f32(x.size)
    mu = fdiv(csum(x), n)
    d = fsub(x, mu)
    var = fdiv(cdot(d, d), n)
    rstd = fdiv(f32(1.0), fsqrt(fadd(var, f32(eps))))
    xh = fmul(d, rstd)
    return canon(fma32(xh, g, b)), mu, rstd


def layernorm_backward_row(dy, x, g, mu, rstd, dres=None):
    n = f32(np.asarray(x).size)
    xh = fmul(fsub(x, mu), rstd)
    gg = fmul(dy, g)
    a = fdiv(csum(gg), n)
    bq = fdiv(cdot(gg, xh), n)
    dx = fmul(fsub(fsub(gg, a), fmul(xh, bq)), rstd)
    if dres is not None:
        dx = fadd(dres, dx)
    return canon(dx)


def layernorm_params(dy, x, mu, rstd):
    """per-shard dgamma = R-SEQ fma(dy, xh), dbeta = R-SEQ(dy) over the rows"""
    dg = np.zeros(x.shape[1], np.float32)
    db = np.zeros(x.shape[1], np.float32)
    for t in range(x.shape[0]):
        xh = fmul(fsub(x[t], mu[t]), rstd[t])
        dg = fma32(dy[t], xh, dg)
        db = fadd(db, dy[t])
    return dg, db


# ---------------------------------------------------------------------- R-CE (R17)
def cross_entropy_row(x, label, scale):
    x = np.asarray(x, np.float32)
    m = np.max(x)
    e = exp(fsub(x, m))
    s = csum(e)
    loss = fsub(fadd(m, log(np.array([s], np.float32))[0]), x[label])
    onehot = np.zeros_like(x)
    onehot[label] = 1
    dl = fmul(fsub(fmul(e, fdiv(f32(1.0), s)), onehot), f32(scale))
    return f32(loss), canon(dl)


# ---------------------------------------------------------------------- R-ADAMW (R15)
def adamw(p, g, m, v, step, lr, b1, b2, eps, wd, decay):
    b1, b2, lr, eps, wd = map(f32, (b1, b2, lr, eps, wd))
    pb1 = f32(1.0)
    pb2 = f32(1.0)
    for _ in range(step):  # beta^t by iterated binary32 multiplies
        pb1 = fmul(pb1, b1)
        pb2 = fmul(pb2, b2)
    bc1 = fsub(f32(1.0), pb1)
    bc2 = fsub(f32(1.0), pb2)
    m2 = fadd(fmul(b1, m), fmul(fsub(f32(1.0), b1), g))
    v2 = fadd(fmul(b2, v), fmul(fsub(f32(1.0), b2), fmul(g, g)))
    upd = fdiv(fdiv(m2, bc1), fadd(fsqrt(fdiv(v2, bc2)), eps))
    if decay:
        upd = fadd(upd, fmul(wd, p))
    p2 = fsub(p, fmul(lr, upd))
    return canon(p2), canon(m2), canon(v2)
