"""Pins for the oracle's R-GEMM (Sec. 3.2 listing).

Each pin is independent of the oracle's own code: exact integer arithmetic,
hand-derived values, an exact-rational IEEE model (tests/ieee_sim.py), and an
FP64 error bound.
"""
import numpy as np
import pytest

import oracle
import synth
from tests import ieee_sim as S


def bits(x):
    return np.asarray(x, dtype=np.float32).view(np.uint32)


def test_spec_examples():
    # [[1,2],[3,4]] x I2 and x [[5,6],[7,8]] (exact small-integer arithmetic)
    A = np.array([[1, 2], [3, 4]], np.float32)
    assert np.array_equal(oracle.gemm(A, np.eye(2, dtype=np.float32)), A)
    assert np.array_equal(oracle.gemm(A, np.array([[5, 6], [7, 8]], np.float32)),
                          np.array([[19, 22], [43, 50]], np.float32))


@pytest.mark.parametrize("M,N,K", [(7, 5, 3), (33, 17, 65), (64, 64, 128)])
@pytest.mark.parametrize("tA,tB", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_exact_small_integers_all_transposes(M, N, K, tA, tB):
    # |partial sums| < 2^24, so every order gives the exact integer result
    A = synth.small_ints(synth.seed_for("gi", M, K), (M, K))
    B = synth.small_ints(synth.seed_for("gi", K, N), (K, N))
    ref = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float32)
    Ain = np.ascontiguousarray(A.T) if tA else A
    Bin = np.ascontiguousarray(B.T) if tB else B
    got = oracle.gemm(Ain, Bin, transA=bool(tA), transB=bool(tB))
    assert np.array_equal(got, ref)


def test_order_pin_k_ascending():
    # a=[1,1,1], b=[2^24, 1, -2^24]: ascending k gives 2^24 -> 2^24 (1 lost, tie to even) -> 0;
    # the order (0,2,1) would give 1.  (Fraction-checked below.)
    A = np.array([[1, 1, 1]], np.float32)
    B = np.array([[2.0 ** 24], [1], [-(2.0 ** 24)]], np.float32)
    assert oracle.gemm(A, B)[0, 0] == 0.0
    acc = np.float32(0)
    for k in (0, 2, 1):
        acc = S.fma(A[0, k], B[k, 0], acc)
    assert acc == 1.0


def test_fma_pin_single_rounding():
    # k=0: acc = -1;  k=1: fma(1+2^-12, 1+2^-12, -1) = 2^-11 + 2^-24 exactly
    # (unfused: (1+2^-12)^2 rounds to 1+2^-11, minus 1 = 2^-11)
    a = np.float32(1 + 2.0 ** -12)
    A = np.array([[1, a]], np.float32)
    B = np.array([[-1], [a]], np.float32)
    got = oracle.gemm(A, B)[0, 0]
    assert got == np.float32(2.0 ** -11 + 2.0 ** -24)
    assert float(got) == 4.883408546447754e-4


def test_plus_zero_init_and_k0():
    # acc starts at +0: a single product of -0 gives +0 (fold from +0, not a copy)
    A = np.array([[-0.0]], np.float32)
    B = np.array([[1.0]], np.float32)
    assert bits(oracle.gemm(A, B))[0, 0] == 0x00000000
    # K = 0: C = epi(+0)
    Z = oracle.gemm(np.zeros((2, 0), np.float32), np.zeros((0, 3), np.float32), M=2, N=3, K=0)
    assert np.all(bits(Z) == 0)
    Zb = oracle.gemm(np.zeros((2, 0), np.float32), np.zeros((0, 3), np.float32), epi=1,
                     bias=np.array([1, -2, 3], np.float32), M=2, N=3, K=0)
    assert np.array_equal(Zb, np.array([[1, -2, 3]] * 2, np.float32))


def test_epilogues_applied_after_fold():
    A = synth.uniform(11, (5, 9))
    B = synth.uniform(12, (9, 4))
    bias = synth.uniform(13, (4,))
    base = oracle.gemm(A, B)
    # bias: one IEEE add per element after the fold (numpy float32 add is IEEE RN)
    assert np.array_equal(oracle.gemm(A, B, epi=1, bias=bias), (base + bias).astype(np.float32))
    # scale: one IEEE multiply after the fold
    assert np.array_equal(oracle.gemm(A, B, epi=2, scale=0.125), (base * np.float32(0.125)))
    s = np.float32(0.08838834764831845)
    assert np.array_equal(oracle.gemm(A, B, epi=2, scale=float(s)), (base * s).astype(np.float32))


@pytest.mark.parametrize("M,N,K,seed", [(3, 4, 17, 1), (8, 8, 32, 2), (2, 3, 40, 3)])
def test_bruteforce_exact_rational(M, N, K, seed):
    # every element recomputed in the exact-rational IEEE model, ascending k, fused
    A = synth.uniform(seed, (M, K))
    B = synth.uniform(seed + 100, (K, N))
    B[K // 2, :] *= np.float32(2.0 ** 20)  # large dynamic range so rounding matters
    got = oracle.gemm(A, B)
    for i in range(M):
        for j in range(N):
            acc = np.float32(0.0)
            for k in range(K):
                acc = S.fma(A[i, k], B[k, j], acc)
            assert bits(got[i, j]) == bits(acc), (i, j)


def test_fp64_error_bound():
    # |C - C64| <= gamma_K * sum|a||b| with gamma_K = K u / (1 - K u), u = 2^-24
    M, N, K = 16, 16, 1024
    A = synth.uniform(21, (M, K))
    B = synth.uniform(22, (K, N))
    got = oracle.gemm(A, B).astype(np.float64)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    absum = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
    u = 2.0 ** -24
    gamma = K * u / (1 - K * u)
    assert np.all(np.abs(got - ref) <= gamma * absum)


def test_reordered_sum_differs_canonical_does_not():
    # Negative control (north_star invariant): a split-K / pairwise order differs
    # somewhere on random data, while repeated canonical calls never differ.
    M, N, K = 32, 32, 512
    A = synth.uniform(31, (M, K))
    B = synth.uniform(32, (K, N))
    c1 = oracle.gemm(A, B)
    c2 = oracle.gemm(A, B)
    assert np.array_equal(bits(c1), bits(c2))
    half = K // 2
    split = (oracle.gemm(A[:, :half], B[:half]) + oracle.gemm(A[:, half:], B[half:])).astype(np.float32)
    assert np.any(bits(split) != bits(c1))


def test_gemm_element_matches_full():
    A = synth.uniform(41, (9, 33))
    B = synth.uniform(42, (33, 7))
    full = oracle.gemm(A, B)
    for (i, j) in [(0, 0), (8, 6), (4, 3)]:
        assert bits(oracle.gemm_element(A, B, i, j)) == bits(full[i, j])
    Bt = np.ascontiguousarray(B.T)
    At = np.ascontiguousarray(A.T)
    for (i, j) in [(0, 0), (8, 6), (4, 3)]:
        assert bits(oracle.gemm_element(At, Bt, i, j, transA=True, transB=True)) == bits(full[i, j])


def test_nan_canonical_output():
    A = np.array([[np.inf, 1.0]], np.float32)
    B = np.array([[0.0], [1.0]], np.float32)  # inf*0 = NaN
    assert bits(oracle.gemm(A, B))[0, 0] == 0x7FC00000
