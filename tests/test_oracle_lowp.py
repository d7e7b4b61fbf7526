"""Pins of the oracle's lower-precision storage (reading R30): narrowing
binary32 -> binary16 / bfloat16 against numpy's and torch's IEEE round-to-nearest-even
conversions over strided sweeps of all 2^32 bit patterns, exact widening over all 2^16
patterns, and the stored-operand GEMM against exact integer arithmetic."""
import numpy as np
import torch

import oracle


def _sweep(stride):
    return np.arange(0, 2 ** 32, stride, dtype=np.uint64).astype(np.uint32).view(np.float32)


def _ties_and_edges():
    # exact f16 / bf16 ties and range edges, both signs
    v = [1 + 2 ** -11, 1 + 3 * 2 ** -11, 65504, 65519.996, 65520, 2 ** -24, 2 ** -25, 3 * 2 ** -25, 2 ** -14,
         2 ** -14 - 2 ** -25, 1 + 2 ** -8, 1 + 3 * 2 ** -8, 3.3895314e38, 1.17549435e-38, 1e-45, 0.0]
    v = np.float32(v)
    return np.concatenate([v, -v])


def test_f16_narrowing_matches_numpy():
    x = np.concatenate([_sweep(4099), _ties_and_edges()])
    with np.errstate(over="ignore"):
        ref = x.astype(np.float16).view(np.uint16)
    got = oracle.convert(x[None], "f32", "f16").ravel()
    nan = np.isnan(x)
    assert np.array_equal(got[~nan], ref[~nan])
    assert np.all(got[nan] == 0x7E00)


def test_f16_widening_exact_all_patterns():
    h = np.arange(2 ** 16, dtype=np.uint32).astype(np.uint16)
    ref = h.view(np.float16).astype(np.float32)
    got = oracle.convert(h[None], "f16", "f32").ravel()
    nan = np.isnan(ref)
    assert np.array_equal(got[~nan].view(np.uint32), ref[~nan].view(np.uint32))
    assert np.all(got[nan].view(np.uint32) == 0x7FC00000)


def test_bf16_narrowing_matches_torch():
    x = np.concatenate([_sweep(4099), _ties_and_edges()])
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = oracle.convert(x[None], "f32", "bf16").ravel()
    nan = np.isnan(x)
    assert np.array_equal(got[~nan], ref[~nan])
    assert np.all(got[nan] == 0x7FC0)


def test_bf16_widening_exact_all_patterns():
    h = np.arange(2 ** 16, dtype=np.uint32).astype(np.uint16)
    ref = torch.from_numpy(h.view(np.int16)).view(torch.bfloat16).float().numpy()
    got = oracle.convert(h[None], "bf16", "f32").ravel()
    nan = np.isnan(ref)
    assert np.array_equal(got[~nan].view(np.uint32), ref[~nan].view(np.uint32))
    assert np.all(got[nan].view(np.uint32) == 0x7FC00000)


def test_gemm_ex_small_integers_exact():
    # integers |v| <= 8 are exact in bf16 and f16; K = 64 partial sums stay < 2^11 (exact in f16 too)
    rng = np.random.default_rng(5)
    A = rng.integers(-8, 9, (33, 64)).astype(np.float32)
    B = rng.integers(-4, 5, (64, 17)).astype(np.float32)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float32)
    for dt in ("bf16", "f16"):
        a, b = oracle.convert(A, "f32", dt), oracle.convert(B, "f32", dt)
        c = oracle.gemm_ex(a, dt, b, dt, dt)   # the fold is exact in binary32, then one narrowing
        assert np.array_equal(c, oracle.convert(exact, "f32", dt))
        if dt == "f16":                        # |C| <= 2048: exact in binary16 as well
            assert np.array_equal(oracle.convert(c, dt, "f32"), exact)
        assert np.array_equal(oracle.gemm_ex(a, dt, b.T.copy(), dt, "f32", transB=True), exact)
    # mixed: f32 A, bf16 B, f32 C == R-GEMM on the widened operand
    Af = rng.standard_normal((20, 30)).astype(np.float32)
    Bf = rng.standard_normal((30, 12)).astype(np.float32)
    bb = oracle.convert(Bf, "f32", "bf16")
    want = oracle.gemm(Af, oracle.convert(bb, "bf16", "f32"))
    assert np.array_equal(oracle.gemm_ex(Af, "f32", bb, "bf16", "f32").view(np.uint32), want.view(np.uint32))
