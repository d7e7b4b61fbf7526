"""Pins of the oracle's deterministic pseudorandomness (reading R28):
Philox4x32-10 against the Random123 known-answer vectors, the element -> (block, word)
mapping, the [0, 1) 2^-24 grid, statistics, and dropout's closed-form properties."""
import os

import numpy as np

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kat():
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(t, 16) for t in line.split()]
        yield w[:4], w[4:6], w[6:10]


def test_philox_known_answer_vectors():
    n = 0
    for ctr, key, want in _kat():
        assert list(oracle.philox4x32_10(ctr, key)) == want
        n += 1
    assert n == 3


def test_uniform_element_mapping_matches_blocks():
    # element i = word i % 4 of the block with counter (i / 4, 0, stream lo, stream hi), key = seed
    seed, stream = 0x0123456789ABCDEF, 0x0000000500000007
    u = oracle.rand_uniform(seed, stream, 4 * 5 + 3)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for b in range(6):
        w = oracle.philox4x32_10([b, 0, stream & 0xFFFFFFFF, stream >> 32], key)
        for j in range(4):
            i = 4 * b + j
            if i < u.size:
                assert u[i] == np.float32((int(w[j]) >> 8) * 2.0 ** -24)


def test_uniform_grid_range_and_statistics():
    u = oracle.rand_uniform(1, 0, 1_000_000)
    assert u.min() >= 0.0 and u.max() < 1.0
    assert np.all(u * np.float32(2 ** 24) == np.floor(u * np.float32(2 ** 24)))  # on the 2^-24 grid
    assert 0.499 <= u.mean() <= 0.501
    assert abs(np.var(u.astype(np.float64)) - 1 / 12) < 1e-3
    # different streams / seeds give different sequences
    assert not np.array_equal(u[:1000], oracle.rand_uniform(1, 1, 1000))
    assert not np.array_equal(u[:1000], oracle.rand_uniform(2, 0, 1000))
    # purity: a prefix is the same draw
    assert np.array_equal(u[:4097], oracle.rand_uniform(1, 0, 4097))


def test_dropout_closed_forms():
    x = np.linspace(-3, 3, 100_003, dtype=np.float32)
    # p = 0: every u >= 0, scale 1 -> identity (bitwise)
    y, m = oracle.dropout(x, 0.0, 9, 4)
    assert np.array_equal(y.view(np.uint32), x.view(np.uint32)) and m.all()
    # p = 1: no u >= 1 -> all +0
    y, m = oracle.dropout(x, 1.0, 9, 4)
    assert not m.any() and np.all(y.view(np.uint32) == 0)
    # p = 0.5: scale exactly 2, kept = 2x exactly, dropped = +0, keep rate ~ 1/2 (6 sigma)
    y, m = oracle.dropout(x, 0.5, 9, 4)
    k = m.astype(bool)
    assert np.array_equal(y[k], x[k] * np.float32(2))
    assert np.all(y[~k].view(np.uint32) == 0)
    assert abs(k.mean() - 0.5) < 6 * 0.5 / np.sqrt(x.size)
    # the mask is u >= p on the same draws
    u = oracle.rand_uniform(9, 4, x.size)
    assert np.array_equal(k, u >= np.float32(0.5))
    # p = 0.1: scale = fl(1 / fl(0.9))
    y, m = oracle.dropout(x, 0.1, 9, 4)
    sc = np.float32(1) / (np.float32(1) - np.float32(0.1))
    k = m.astype(bool)
    assert np.array_equal(y[k], x[k] * sc)
    assert abs(k.mean() - 0.9) < 6 * 0.3 / np.sqrt(x.size)
    # backward regenerates the same mask and scale
    dy = np.cos(x)
    dx = oracle.dropout_backward(dy, 0.1, 9, 4)
    assert np.array_equal(dx[k], dy[k] * sc) and np.all(dx[~k].view(np.uint32) == 0)
