"""Pins for the oracle's canonical reductions: R-CSUM / R-CDOT (PAPER.md
P:588-590, reading R4), R-SEQ column folds, R-TREE_S (reading R14).

Expected values are derived by hand in the comments (exact arithmetic with
ties-to-even at 2^24, where the binary32 spacing is 2), or are exact integer
sums that hold for ANY order -- so a dropped/duplicated element, a wrong slot
index, a wrong tree pairing or a wrong tile rule fails one of them.
"""
import numpy as np
import pytest

import oracle
import synth

T24 = 2.0 ** 24


def b(x):
    return int(np.float32(x).view(np.uint32))


def test_csum_hand_values():
    assert oracle.csum([1, 2, 3, 4]) == 10
    assert oracle.csum([]) == 0 and b(oracle.csum([])) == 0
    # slots start at +0: (+0) + (-0) = +0
    assert b(oracle.csum([-0.0] * 5)) == 0x00000000
    assert oracle.csum([1.0] * 4097) == 4097


def test_csum_slot_and_tree_pins():
    # [1, 1, 2^24]: slots p0=1, p1=1, p2=2^24; TREE: h=2: p0 = 1 + 2^24 -> 2^24 (tie, even);
    # h=1: p0 = 2^24 + 1 -> 2^24.  A serial fold would give 1+1=2, 2+2^24 = 2^24+2.
    assert b(oracle.csum([1, 1, T24])) == 0x4B800000
    # x[0]=2^24, x[1]=1, x[65]=1: the h=64 level pairs slot 1 with slot 65 first (1+1=2),
    # then h=1 gives 2^24 + 2 = 16777218 exactly.  Serial-slot or adjacent-pair trees
    # would add the ones to 2^24 one at a time and lose both (16777216).
    x = np.zeros(66, np.float32)
    x[0], x[1], x[65] = T24, 1, 1
    assert oracle.csum(x) == 16777218.0
    # slot assignment i % 128: x[0]=2^24 and x[128]=1 share slot 0 (2^24+1 -> 2^24);
    # x[1]=1 sits in slot 1; final h=1: 2^24 + 1 -> 2^24.
    x = np.zeros(129, np.float32)
    x[0], x[128], x[1] = T24, 1, 1
    assert oracle.csum(x) == T24
    # ... whereas with x[1] replaced by x[129] (slot 1 too) the two ones meet in slot 1
    x = np.zeros(130, np.float32)
    x[0], x[1], x[129] = T24, 1, 1
    assert oracle.csum(x) == T24 + 2


def test_csum_tile_rule():
    # [2^24, 1 x 4097] (4098 elements):
    # tile 0 = [2^24, 1 x 4095]: slot 0 = 2^24 (31 ones lost), slots 1..127 = 32 each;
    # TREE: p0 = 2^24+32+64+128+256+512+1024+2048 = 16781280.  tile 1 = [1, 1] -> 2.
    # CSUM([16781280, 2]) = 16781282.  (exact: 16781313; serial fold: 16777216)
    x = np.ones(4098, np.float32)
    x[0] = T24
    assert oracle.csum(x) == 16781282.0


def test_csum_exact_integers_any_length():
    for n in (1, 127, 128, 129, 4095, 4096, 4097, 50257, 3 * 4096 * 4096 // 1024):
        x = synth.small_ints(synth.seed_for("cs", n), n, 0, 4)
        assert oracle.csum(x) == float(x.astype(np.int64).sum())


def test_csum_error_bound_random():
    x = synth.uniform(5, 50257)
    ref = float(np.sum(x.astype(np.float64)))
    # tile sums + tree: depth <= 32 + 7 + 13 + 7 additions per element
    bound = 60 * 2.0 ** -24 * float(np.sum(np.abs(x.astype(np.float64))))
    assert abs(float(oracle.csum(x)) - ref) <= bound


def test_cdot_pins():
    u = synth.small_ints(1, 777, -5, 5)
    v = synth.small_ints(2, 777, -5, 5)
    assert oracle.cdot(u, v) == float((u.astype(np.int64) * v.astype(np.int64)).sum())
    # slot update is ONE fused fma: elements 0 and 128 share slot 0:
    # p0 = fma(1,-1,0) = -1;  p0 = fma(1+2^-12, 1+2^-12, -1) = 2^-11 + 2^-24 (exact)
    a = np.float32(1 + 2.0 ** -12)
    uu = np.zeros(129, np.float32)
    vv = np.zeros(129, np.float32)
    uu[0], vv[0], uu[128], vv[128] = 1, -1, a, a
    assert oracle.cdot(uu, vv) == np.float32(2.0 ** -11 + 2.0 ** -24)
    # multi-tile: tile results are combined with CSUM (tile dots 3*4096 and 3*1)
    n = 4097
    assert oracle.cdot(np.full(n, 3, np.float32), np.ones(n, np.float32)) == 3 * n


def test_sum_rows_matches_csum():
    x = synth.uniform(7, (5, 300))
    rows = oracle.sum_rows(x)
    for r in range(5):
        assert b(rows[r]) == b(oracle.csum(x[r]))


def test_seq_column_fold():
    # exact integers: any order
    x = synth.small_ints(9, (64, 33))
    out = oracle.sum_cols_seq(x, nseg=4)
    ref = x.astype(np.int64).reshape(4, 16, 33).sum(axis=1).astype(np.float32)
    assert np.array_equal(out, ref)
    # ascending order pin: column [2^24, 1, 1, 2^24 ... ] folds 2^24 -> 2^24 -> 2^24
    # while the reverse order [.., 1, 1] would first make 2 then 2^24+2
    y = np.array([[T24], [1], [1]], np.float32)
    assert oracle.sum_cols_seq(y)[0, 0] == T24
    assert oracle.sum_cols_seq(y[::-1].copy())[0, 0] == T24 + 2
    # fold from +0: a single -0 row gives +0
    assert b(oracle.sum_cols_seq(np.array([[-0.0]], np.float32))[0, 0]) == 0


def test_tree_sum_pins():
    # g = [2^24, 0, 1, 1]: ((g0+g1)+(g2+g3)) = 2^24 + 2; serial ((g0+g1)+g2)+g3 = 2^24
    parts = [np.array([v], np.float32) for v in (T24, 0, 1, 1)]
    assert oracle.tree_sum(parts)[0] == T24 + 2
    # 8 parts: (((0,1),(2,3)),((4,5),(6,7))): put 2^24 in part 0 and ones in parts 4,5
    vals = [T24, 0, 0, 0, 1, 1, 0, 0]
    parts = [np.array([v], np.float32) for v in vals]
    assert oracle.tree_sum(parts)[0] == T24 + 2
    # single part = identity (leaf), even for -0
    assert b(oracle.tree_sum([np.array([-0.0], np.float32)])[0]) == 0x80000000
    # exact integers
    ps = [synth.small_ints(100 + i, 1000) for i in range(8)]
    assert np.array_equal(oracle.tree_sum(ps), np.sum([p.astype(np.int64) for p in ps], 0).astype(np.float32))


@pytest.mark.parametrize("G", [1, 2, 4])
def test_tree_is_aligned_subtrees(G):
    # R-TREE_S over 8 parts == top tree over G aligned local subtrees (multi-GPU identity)
    ps = [synth.uniform(200 + i, 4096) for i in range(8)]
    full = oracle.tree_sum(ps)
    per = 8 // G
    locals_ = [oracle.tree_sum(ps[r * per:(r + 1) * per]) for r in range(G)]
    top = oracle.tree_sum(locals_)
    assert np.array_equal(full.view(np.uint32), top.view(np.uint32))
