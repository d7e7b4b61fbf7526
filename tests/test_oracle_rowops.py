"""Pins for the oracle's row operators: softmax (reading R7), LayerNorm
(reading R8), cross-entropy, embedding, AdamW (reading R15).
Closed forms, exact special cases and float64 error bounds."""
import math

import numpy as np
import pytest

import oracle
import synth


def bits(x):
    return np.asarray(x, dtype=np.float32).view(np.uint32)


# ---------------------------------------------------------------- softmax
def test_softmax_closed_forms():
    # [c, c] -> [0.5, 0.5] exactly; uniform row of 2^k -> 2^-k exactly
    assert np.array_equal(oracle.softmax(np.float32([[3.25, 3.25]])), np.float32([[0.5, 0.5]]))
    for k in (1, 5, 9, 12):
        y = oracle.softmax(np.full((2, 2 ** k), -1.5, np.float32))
        assert np.all(y == np.float32(2.0 ** -k))
    # [0, ln 2] ~ [1/3, 2/3]
    y = oracle.softmax(np.float32([[0.0, math.log(2)]]))
    assert abs(y[0, 0] - 1 / 3) < 1e-6 and abs(y[0, 1] - 2 / 3) < 1e-6


def test_softmax_shift_invariance_bitwise():
    # x + c exact for every element -> x - max is identical -> identical output bits
    x = synth.small_ints(3, (4, 300), -20, 20) * np.float32(0.25)
    y1 = oracle.softmax(x)
    y2 = oracle.softmax(x + np.float32(64.0))
    assert np.array_equal(bits(y1), bits(y2))


def test_softmax_causal_mask_and_bound():
    T = 64
    x = synth.uniform(5, (3 * T, T), 4.0)
    y = oracle.softmax(x, causal=True)
    for r in range(3 * T):
        L = r % T + 1
        assert np.all(bits(y[r, L:]) == 0)
        xd = x[r, :L].astype(np.float64)
        ref = np.exp(xd - xd.max())
        ref /= ref.sum()
        assert np.max(np.abs(y[r, :L] - ref) / ref) < 8 * 2.0 ** -23
    # the causal row r equals the plain softmax of its first (r mod T)+1 entries
    r = 77
    L = r % T + 1
    assert np.array_equal(bits(y[r, :L]), bits(oracle.softmax(x[r:r + 1, :L])[0]))


def test_softmax_long_rows_multi_tile():
    x = synth.uniform(6, (2, 50257), 8.0)
    y = oracle.softmax(x).astype(np.float64)
    xd = x.astype(np.float64)
    ref = np.exp(xd - xd.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    assert np.max(np.abs(y - ref) / ref) < 16 * 2.0 ** -23


def test_softmax_backward_bound_and_constant_dy():
    y = oracle.softmax(synth.uniform(7, (8, 512), 3.0))
    dy = synth.uniform(8, (8, 512))
    dx = oracle.softmax_backward(y, dy, scale=0.125).astype(np.float64)
    yd, gd = y.astype(np.float64), dy.astype(np.float64)
    ref = yd * (gd - (yd * gd).sum(1, keepdims=True)) * 0.125
    assert np.max(np.abs(dx - ref)) < 1e-8
    # constant dy = c: dx_i = y_i (c - CDOT(y, c)) = y_i c (1 - sum y) ~ 0
    dx0 = oracle.softmax_backward(y, np.full_like(y, 2.0))
    assert np.max(np.abs(dx0)) < 1e-8


# ---------------------------------------------------------------- layernorm
def test_layernorm_constant_row_gives_beta():
    x = np.full((3, 768), 1.75, np.float32)
    gamma = synth.uniform(1, 768)
    beta = synth.uniform(2, 768)
    y, mean, rstd = oracle.layernorm(x, gamma, beta)
    assert np.array_equal(bits(y), bits(np.broadcast_to(beta, y.shape)))
    assert np.all(mean == 1.75)
    assert np.all(rstd == np.float32(1.0) / np.sqrt(np.float32(1e-5)))


def test_layernorm_bound():
    x = synth.uniform(3, (16, 768), 2.0)
    gamma = synth.uniform(4, 768)
    beta = synth.uniform(5, 768)
    y, mean, rstd = oracle.layernorm(x, gamma, beta)
    xd = x.astype(np.float64)
    mu = xd.mean(1, keepdims=True)
    var = ((xd - mu) ** 2).mean(1, keepdims=True)
    ref = (xd - mu) / np.sqrt(var + np.float32(1e-5)) * gamma + beta
    assert np.max(np.abs(y - ref)) < 2e-6
    assert np.max(np.abs(mean - mu[:, 0])) < 1e-7


def test_layernorm_backward_bound():
    x = synth.uniform(9, (16, 768), 2.0)
    gamma = synth.uniform(10, 768)
    beta = synth.uniform(11, 768)
    dy = synth.uniform(12, (16, 768))
    dres = synth.uniform(13, (16, 768))
    y, mean, rstd = oracle.layernorm(x, gamma, beta)
    dx = oracle.layernorm_backward(dy, x, gamma, mean, rstd)
    # float64 analytic LN backward
    xd, gd, gm = x.astype(np.float64), dy.astype(np.float64), gamma.astype(np.float64)
    mu = xd.mean(1, keepdims=True)
    rs = 1 / np.sqrt(((xd - mu) ** 2).mean(1, keepdims=True) + 1e-5)
    xh = (xd - mu) * rs
    g = gd * gm
    ref = (g - g.mean(1, keepdims=True) - xh * (g * xh).mean(1, keepdims=True)) * rs
    assert np.max(np.abs(dx - ref)) < 5e-5
    # residual accumulate is exactly one IEEE add
    dx2 = oracle.layernorm_backward(dy, x, gamma, mean, rstd, dres=dres)
    assert np.array_equal(bits(dx2), bits(dres + dx))
    # parameter gradients: exact-integer data for dbeta; bound for dgamma
    dg, db = oracle.layernorm_backward_params(dy, x, mean, rstd, nseg=4)
    assert np.max(np.abs(db - gd.reshape(4, 4, 768).sum(1))) < 1e-6
    xhf = ((x - mean[:, None]) * rstd[:, None]).astype(np.float64)
    assert np.max(np.abs(dg - (gd * xhf).reshape(4, 4, 768).sum(1))) < 1e-5


# ---------------------------------------------------------------- cross entropy
def test_cross_entropy_uniform_and_bound():
    # uniform logits over C=4 -> ln 4 within 1e-6
    loss, d = oracle.cross_entropy(np.zeros((3, 4), np.float32), np.array([0, 1, 3]))
    assert np.all(np.abs(loss - math.log(4)) < 1e-6)
    # gradient of uniform: (1/4 - onehot) exactly
    assert np.array_equal(d[0], np.float32([-0.75, 0.25, 0.25, 0.25]))
    V = 50257
    x = synth.uniform(4, (4, V), 6.0)
    lab = synth.integers(5, 4, V)
    loss, d = oracle.cross_entropy(x, lab, scale=2.0 ** -12)
    xd = x.astype(np.float64)
    m = xd.max(1, keepdims=True)
    lse = m[:, 0] + np.log(np.exp(xd - m).sum(1))
    ref = lse - xd[np.arange(4), lab]
    assert np.max(np.abs(loss - ref)) < 4e-6
    p = np.exp(xd - lse[:, None])
    p[np.arange(4), lab] -= 1
    assert np.max(np.abs(d - p * 2.0 ** -12)) < 1e-10
    # finite-difference check of the gradient, small row
    x = synth.uniform(6, (1, 9), 2.0).astype(np.float32)
    lab = np.array([4])
    _, d = oracle.cross_entropy(x, lab)
    for i in range(9):
        e = np.zeros_like(x)
        h = 1e-3
        e[0, i] = h
        lp, _ = oracle.cross_entropy(x + e, lab, want_grad=False)
        lm, _ = oracle.cross_entropy(x - e, lab, want_grad=False)
        assert abs((lp[0] - lm[0]) / (2 * h) - d[0, i]) < 2e-3


# ---------------------------------------------------------------- embedding
def test_embedding_forward_is_one_add():
    wte = synth.uniform(1, (50, 16))
    wpe = synth.uniform(2, (8, 16))
    tok = synth.integers(3, 24, 50)
    x0 = oracle.embedding(tok, wte, wpe, T=8)
    ref = wte[tok] + wpe[np.arange(24) % 8]
    assert np.array_equal(bits(x0), bits(ref))


def test_embedding_backward_pins():
    T = 8
    tok = np.array([3, 1, 3, 3, 0, 1, 7, 3] * 2, np.int32)
    dx0 = synth.small_ints(4, (16, 5))
    dwte, dwpe = oracle.embedding_backward(tok, dx0, T, np.zeros((10, 5), np.float32),
                                           np.full((T, 5), 7.0, np.float32))  # dwpe is overwritten
    ref = np.zeros((10, 5), np.int64)
    np.add.at(ref, tok, dx0.astype(np.int64))
    assert np.array_equal(dwte, ref.astype(np.float32))
    assert np.array_equal(dwpe, (dx0[:8] + dx0[8:]).astype(np.float32))
    # ascending-token fold: rows for token 3 hold [2^24, 1, 1]: 2^24 -> 2^24 -> 2^24,
    # then added to the incoming 0 -> 2^24 (a pairwise order would give 2^24 + 2)
    tok = np.array([3, 3, 3], np.int32)
    dx0 = np.array([[2.0 ** 24], [1.0], [1.0]], np.float32)
    dwte, _ = oracle.embedding_backward(tok, dx0, 3, np.zeros((4, 1), np.float32))
    assert dwte[3, 0] == 2.0 ** 24 and np.all(bits(dwte[[0, 1, 2], 0]) == 0)
    # rows never used keep their incoming bits (incl. -0)
    inc = np.full((4, 1), -0.0, np.float32)
    dwte, _ = oracle.embedding_backward(tok, dx0, 3, inc)
    assert bits(dwte[0, 0]) == 0x80000000


# ---------------------------------------------------------------- AdamW
def test_adamw_closed_forms():
    n = 1000
    p = synth.uniform(1, n)
    g = synth.uniform(2, n)
    z = np.zeros(n, np.float32)
    lr, b1, b2, eps, wd = 6e-4, 0.9, 0.95, 1e-8, 0.1
    p1, m1, v1 = oracle.adamw(p, g, z, z, 1, lr, b1, b2, eps, wd, decay=False)
    # step 1: m' = (1-b1) g, v' = (1-b2) g^2 (one rounding each), mhat ~ g, vhat ~ g^2
    assert np.array_equal(m1, (np.float32(1) - np.float32(b1)) * g)
    assert np.array_equal(v1, (np.float32(1) - np.float32(b2)) * (g * g))
    # so p' ~ p - lr * sign(g) for |g| >> eps
    big = np.abs(g) > 1e-3
    assert np.max(np.abs((p.astype(np.float64) - p1)[big] - lr * np.sign(g[big]))) < 1e-7
    # zero gradient + decay: upd = 0 + wd*p  ->  p' = p - lr*(wd*p)
    p2, _, _ = oracle.adamw(p, z, z, z, 1, lr, b1, b2, eps, wd, decay=True)
    ref = p - np.float32(lr) * (np.float32(wd) * p)
    assert np.array_equal(bits(p2), bits(ref.astype(np.float32)))
    # float64 bound at a later step with state
    m = synth.uniform(3, n, 0.01)
    v = np.abs(synth.uniform(4, n, 0.001))
    p3, m3, v3 = oracle.adamw(p, g, m, v, 7, lr, b1, b2, eps, wd, decay=True)
    gd, md, vd, pd = (a.astype(np.float64) for a in (g, m, v, p))
    mr = b1 * md + (1 - b1) * gd
    vr = b2 * vd + (1 - b2) * gd * gd
    upd = (mr / (1 - b1 ** 7)) / (np.sqrt(vr / (1 - b2 ** 7)) + eps) + wd * pd
    assert np.max(np.abs(p3 - (pd - lr * upd))) < 1e-7
