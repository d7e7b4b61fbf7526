"""Pins for the oracle's Llama operators (config 4): RMSNorm, SwiGLU, RoPE
(readings R20-R22).  Exact special cases, float64 bounds, algebraic identities."""
import numpy as np

import oracle
import synth


def bits(x):
    return np.asarray(x, dtype=np.float32).view(np.uint32)


def test_rmsnorm_exact_cases_and_bound():
    # a row of equal |c| entries: ms = c^2 exactly for c = 2 (CDOT of 4s / n exact), rstd = 1/sqrt(4+eps)
    x = np.full((2, 64), 2.0, np.float32)
    x[1] *= -1
    w = synth.uniform(3, 64)
    y, rs = oracle.rmsnorm(x, w, eps=0.0)
    assert np.all(rs == 0.5) and np.array_equal(y[0], w) and np.array_equal(y[1], -w)
    x = synth.uniform(4, (8, 4096), 3.0)
    w = synth.uniform(5, 4096)
    y, rs = oracle.rmsnorm(x, w)
    xd = x.astype(np.float64)
    ref = xd / np.sqrt((xd ** 2).mean(1, keepdims=True) + 1e-5) * w
    assert np.max(np.abs(y - ref)) < 3e-6
    # the normalised row (w = 1) has mean square ~1
    y1, _ = oracle.rmsnorm(x, np.ones(4096, np.float32))
    assert np.all(np.abs((y1.astype(np.float64) ** 2).mean(1) - 1) < 1e-4)


def test_swiglu_values_and_bound():
    g = np.float32([0.0, -0.0, 100.0, -100.0, 1.0])
    u = np.float32([3.0, 3.0, 2.0, 2.0, 1.0])
    h = oracle.swiglu(g, u)
    assert h[0] == 0 and h[2] == 200.0 and abs(h[3]) < 1e-30
    assert abs(h[4] - 1 / (1 + np.exp(-1.0))) < 1e-7
    g = synth.uniform(6, 100000, 20.0)
    u = synth.uniform(7, 100000, 2.0)
    h = oracle.swiglu(g, u).astype(np.float64)
    gd = g.astype(np.float64)
    ref = gd / (1 + np.exp(-gd)) * u
    assert np.max(np.abs(h - ref) / np.maximum(np.abs(ref), 1e-3)) < 4e-7


def test_rope_identities():
    T, H, hd = 16, 4, 32
    x = synth.uniform(8, (T, H * hd))
    ones, zeros = np.ones((T, hd // 2), np.float32), np.zeros((T, hd // 2), np.float32)
    # cos = 1, sin = 0: identity (x*1 - y*0 = x exactly)
    assert np.array_equal(bits(oracle.rope(x, ones, zeros, H, hd)), bits(x))
    # cos = 0, sin = 1: exact rotation by 90 degrees -> (-x2, x1)
    y = oracle.rope(x, zeros, ones, H, hd).reshape(T, H, hd)
    xr = x.reshape(T, H, hd)
    assert np.array_equal(y[..., :hd // 2], -xr[..., hd // 2:])
    assert np.array_equal(y[..., hd // 2:], xr[..., :hd // 2])
    # general angles: norm preserved to rounding, matches float64 rotation
    ang = synth.uniform(9, (T, hd // 2), 3.0).astype(np.float64)
    c, s = np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
    y = oracle.rope(x, c, s, H, hd).reshape(T, H, hd).astype(np.float64)
    a, b = xr[..., :hd // 2].astype(np.float64), xr[..., hd // 2:].astype(np.float64)
    cd, sd = c.astype(np.float64)[:, None, :], s.astype(np.float64)[:, None, :]
    assert np.max(np.abs(y[..., :hd // 2] - (a * cd - b * sd))) < 3e-7
    assert np.max(np.abs(y[..., hd // 2:] - (b * cd + a * sd))) < 3e-7
