"""Pins for the oracle's software math (reading R5/R6):
accuracy against float64 libm over strided sweeps of every binary32 in range
(a dropped or mistyped polynomial coefficient breaks the ulp bound), exact
special values, and the correctly-rounded rsqrt composition."""
import math

import numpy as np
import pytest

import oracle
import synth


def u2f(u):
    return np.asarray(u, dtype=np.uint32).view(np.float32)


def bits(x):
    return np.asarray(x, dtype=np.float32).view(np.uint32)


def ulp_of(ref64: np.ndarray) -> np.ndarray:
    a = np.abs(ref64)
    e = np.floor(np.log2(np.maximum(a, 2.0 ** -149)))
    return np.exp2(np.maximum(e, -126) - 23)


def sweep(lo_bits, hi_bits, stride):
    return u2f(np.arange(lo_bits, hi_bits, stride, dtype=np.uint64).astype(np.uint32))


def ulp_err(fn_oracle, fn64, x):
    y = fn_oracle(x).astype(np.float64)
    ref = fn64(x.astype(np.float64))
    return np.abs(y - ref) / ulp_of(ref)


def test_exp_special_values():
    f = oracle.exp
    assert bits(f(np.float32([0.0])))[0] == 0x3F800000
    assert bits(f(np.float32([-0.0])))[0] == 0x3F800000
    assert bits(f(np.float32([1.0])))[0] == 0x402DF854  # correctly rounded e
    assert np.isfinite(f(np.float32([88.72283172607422])))[0]
    assert np.isinf(f(np.float32([88.72283935546875])))[0]
    assert bits(f(np.float32([np.inf])))[0] == 0x7F800000
    assert bits(f(np.float32([-np.inf])))[0] == 0
    assert bits(f(np.float32([-104.5])))[0] == 0
    assert bits(f(np.float32([np.nan])))[0] == 0x7FC00000
    assert bits(f(u2f([0xFFC00001])))[0] == 0x7FC00000


def test_exp_accuracy_sweep():
    # positive side up to 88.72, negative side down to -87.33 (normal results)
    for lo, hi in ((0x00000000, 0x42B17218), (0x80000000, 0xC2AEAC50)):
        x = sweep(lo, hi, 97)
        err = ulp_err(oracle.exp, np.exp, x)
        assert err.max() <= 1.5, err.max()
    # subnormal results: absolute error <= 1 unit of 2^-149
    x = np.linspace(-103.9, -87.34, 200001).astype(np.float32)
    y = oracle.exp(x).astype(np.float64)
    assert np.max(np.abs(y - np.exp(x.astype(np.float64)))) <= 2.0 ** -149


def test_log_special_values():
    f = oracle.log
    assert bits(f(np.float32([1.0])))[0] == 0
    assert bits(f(np.float32([2.0])))[0] == 0x3F317218  # correctly rounded ln 2
    assert bits(f(np.float32([0.0])))[0] == 0xFF800000
    assert bits(f(np.float32([-0.0])))[0] == 0xFF800000
    assert bits(f(np.float32([-1.0])))[0] == 0x7FC00000
    assert bits(f(np.float32([np.inf])))[0] == 0x7F800000
    assert bits(f(np.float32([np.nan])))[0] == 0x7FC00000


def test_log_accuracy_sweep():
    x = sweep(0x00000001, 0x7F800000, 61)
    err = ulp_err(oracle.log, np.log, x)
    assert err.max() <= 1.0, err.max()


def test_tanh_values_and_sweep():
    f = oracle.tanh
    assert bits(f(np.float32([0.0])))[0] == 0
    assert bits(f(np.float32([-0.0])))[0] == 0x80000000
    assert f(np.float32([np.inf]))[0] == 1.0 and f(np.float32([-np.inf]))[0] == -1.0
    assert f(np.float32([20.0]))[0] == 1.0
    assert bits(f(np.float32([np.nan])))[0] == 0x7FC00000
    x = np.concatenate([np.linspace(-12, 12, 2000001).astype(np.float32),
                        sweep(0x30000000, 0x3F200000, 101)])
    err = ulp_err(oracle.tanh, np.tanh, x)
    assert err.max() <= 1.5, err.max()
    # odd symmetry is exact (copysign of the |u| result)
    assert np.array_equal(bits(f(-x)), bits(f(x)) ^ np.uint32(0x80000000))


def test_rsqrt_correctly_rounded_composition():
    f = oracle.rsqrt
    assert f(np.float32([4.0]))[0] == 0.5 and f(np.float32([0.25]))[0] == 2.0
    assert bits(f(np.float32([0.0])))[0] == 0x7F800000
    assert bits(f(np.float32([-1.0])))[0] == 0x7FC00000
    # IEEE sqrt and divide are correctly rounded, so numpy's float32 ops are the same composition
    x = sweep(0x00000001, 0x7F800000, 7919)
    with np.errstate(all="ignore"):
        ref = np.float32(1.0) / np.sqrt(x)
    assert np.array_equal(bits(f(x)), bits(ref))


def test_gelu_pins():
    x = np.concatenate([np.linspace(-10, 10, 200001), [0.0, -0.0, 30.0, -30.0]]).astype(np.float32)
    y = oracle.gelu(x).astype(np.float64)
    xd = x.astype(np.float64)
    ref = 0.5 * xd * (1 + np.tanh(math.sqrt(2 / math.pi) * (xd + 0.044715 * xd ** 3)))
    # (1 + t) cancels for x << 0, so the bound is conditioned on |x|/2, not on |y|:
    # a few ulp of t (~2^-23 each) scaled by 0.5|x|, plus 2 ulp of the result
    bound = 0.5 * np.abs(xd) * 2.0 ** -21 + 2 * np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 2.0 ** -126))) - 23)
    assert np.all(np.abs(y - ref) <= bound)
    assert y[-4] == 0 and y[-2] == 30.0 and y[-1] == 0.0
    # backward against the analytic derivative in float64
    dy = np.ones_like(x)
    g = oracle.gelu_backward(x, dy).astype(np.float64)
    c = math.sqrt(2 / math.pi)
    u = c * (xd + 0.044715 * xd ** 3)
    t = np.tanh(u)
    gref = 0.5 * (1 + t) + 0.5 * xd * (1 - t * t) * c * (1 + 3 * 0.044715 * xd ** 2)
    assert np.max(np.abs(g - gref)) < 2e-6
    # dy scaling is one IEEE multiply
    dy2 = np.full_like(x, 0.375)
    assert np.array_equal(oracle.gelu_backward(x, dy2), (oracle.gelu_backward(x, dy) * np.float32(0.375)))


# ---------------------------------------------------------------------- sin / cos (reading R26)
def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_sin_cos_accuracy_sweep():
    """Cephes sinf/cosf accuracy: |error| <= 2^-23 over [-3000, 3000] against float64,
    relative error <= 1e-7 on the reduced interval [-pi/4, pi/4] (Cephes: 7.8e-8)."""
    x = np.linspace(-3000, 3000, 600001).astype(np.float32)
    x64 = x.astype(np.float64)
    assert np.max(np.abs(oracle.sin(x) - np.sin(x64))) <= 2.0 ** -23
    assert np.max(np.abs(oracle.cos(x) - np.cos(x64))) <= 2.0 ** -23
    y = np.linspace(-0.785, 0.785, 100001).astype(np.float32)
    y64 = y.astype(np.float64)
    nz = np.abs(y64) > 1e-30
    assert np.max(np.abs(oracle.sin(y)[nz] - np.sin(y64[nz])) / np.abs(np.sin(y64[nz]))) <= 1e-7
    assert np.max(np.abs(oracle.cos(y) - np.cos(y64)) / np.cos(y64)) <= 1e-7


def test_sin_cos_exact_identities_and_special_values():
    x = synth.uniform(3, 100001, 2000.0)
    assert np.array_equal(_bits(oracle.sin(-x)), _bits(-oracle.sin(x)))   # odd, bit for bit
    assert np.array_equal(_bits(oracle.cos(-x)), _bits(oracle.cos(x)))    # even, bit for bit
    z = np.float32([0.0, -0.0])
    # the chain's zero: fmaf(p z, r, r) = (-0)(-0) + (-0) = +0, so sin(-0) = +0 (R26)
    assert _bits(oracle.sin(z)).tolist() == [0, 0]
    assert oracle.cos(z).tolist() == [1.0, 1.0]
    bad = np.float32([np.inf, -np.inf, np.nan])
    assert np.all(_bits(oracle.sin(bad)) == 0x7FC00000) and np.all(_bits(oracle.cos(bad)) == 0x7FC00000)
    assert oracle.sin(np.float32([3e7]))[0] == 0.0 and oracle.cos(np.float32([-3e7]))[0] == 0.0  # Cephes TLOSS
    s, c = oracle.sin(x).astype(np.float64), oracle.cos(x).astype(np.float64)
    assert np.max(np.abs(s * s + c * c - 1.0)) < 4e-7


def test_rope_tables_from_inv_freq():
    hd, T = 128, 2048
    inv = (500000.0 ** (-np.arange(0, hd, 2, dtype=np.float64) / hd)).astype(np.float32)
    c, s = oracle.rope_tables_from_inv_freq(inv, T)
    assert np.all(c[0] == 1.0) and np.all(_bits(s[0]) == 0)                # t = 0: angle +0
    ang = (np.arange(T, dtype=np.float32)[:, None] * inv[None, :]).astype(np.float32)  # the rounded fmul
    assert np.max(np.abs(c - np.cos(ang.astype(np.float64)))) <= 2.0 ** -23
    assert np.max(np.abs(s - np.sin(ang.astype(np.float64)))) <= 2.0 ** -23


# ---------------------------------------------------------------------- erf / exact GELU (reading R27)
def test_erf_accuracy_and_exact_properties():
    x = np.linspace(-6, 6, 240001).astype(np.float32)
    ref = np.array([math.erf(float(v)) for v in x])
    e = oracle.erf(x)
    assert np.max(np.abs(e - ref)) <= 1.5e-7                      # Cephes erff / erfcf accuracy
    small = (np.abs(x) <= 1) & (x != 0)
    assert np.max(np.abs(e[small] - ref[small]) / np.abs(ref[small])) <= 2e-7
    assert np.all(np.diff(e.astype(np.float64)) >= 0)            # monotone on the sweep
    y = synth.uniform(8, 50001, 8.0)
    assert np.array_equal(_bits(oracle.erf(-y)), _bits(-oracle.erf(y)))  # odd, bit for bit
    sp = oracle.erf(np.float32([0.0, 10.0, -10.0, 1e30, np.inf, -np.inf, np.nan]))
    assert sp[:6].tolist() == [0.0, 1.0, -1.0, 1.0, 1.0, -1.0] and _bits(sp)[6] == 0x7FC00000


def test_gelu_erf_against_float64_and_its_derivative():
    x = synth.uniform(9, 100001, 8.0)
    x64 = x.astype(np.float64)
    ref = 0.5 * x64 * (1 + np.array([math.erf(v / math.sqrt(2)) for v in x64]))
    g = oracle.gelu_erf(x)
    assert np.all(np.abs(g - ref) <= 4e-7 * np.abs(x64) + 1e-7)
    assert oracle.gelu_erf(np.float32([20.0]))[0] == 20.0 and oracle.gelu_erf(np.float32([0.0]))[0] == 0.0
    # backward = d/dx of the float64 GELU (central differences away from nothing special)
    xs = synth.uniform(10, 200, 4.0).astype(np.float64)
    h = 1e-4
    f = lambda v: 0.5 * v * (1 + np.array([math.erf(t / math.sqrt(2)) for t in v]))  # noqa: E731
    fd = (f(xs + h) - f(xs - h)) / (2 * h)
    dy = synth.uniform(11, 200, 2.0)
    got = oracle.gelu_erf_backward(xs.astype(np.float32), dy)
    assert np.allclose(got, fd * dy, rtol=1e-5, atol=1e-6)
