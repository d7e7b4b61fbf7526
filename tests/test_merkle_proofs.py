"""Merkle membership proofs and leaf-hash trees of the library's host code (no GPU):
RFC 6962 audit paths (PATH(m, D[n]), §2.1.1) checked against an independent
hashlib implementation and the oracle's MTH, RFC 9162 verification accepting every
true proof and rejecting tampered ones, and the data-root / tensor-digest helpers
against the oracle's R-TCOMMIT (reading R11)."""
import hashlib
import os

import numpy as np
import pytest

import oracle
import synth
from paper_2502_19405_b200 import (verde_first_divergence, verde_merkle_audit_path, verde_merkle_root,
                                   verde_merkle_root_hashed, verde_merkle_verify_path,
                                   verde_tensor_digest_from_root)


def H(b):
    return hashlib.sha256(b).digest()


def mth(leaf_hashes):
    n = len(leaf_hashes)
    if n == 1:
        return leaf_hashes[0]
    k = 1
    while 2 * k < n:
        k *= 2
    return H(b"\x01" + mth(leaf_hashes[:k]) + mth(leaf_hashes[k:]))


def path(m, leaf_hashes):  # RFC 6962 §2.1.1, written out
    n = len(leaf_hashes)
    if n == 1:
        return []
    k = 1
    while 2 * k < n:
        k *= 2
    if m < k:
        return path(m, leaf_hashes[:k]) + [mth(leaf_hashes[k:])]
    return path(m - k, leaf_hashes[k:]) + [mth(leaf_hashes[:k])]


def entries(n, seed=1):
    return [H(seed.to_bytes(4, "little") + i.to_bytes(4, "little")) for i in range(n)]


@pytest.mark.parametrize("n", list(range(1, 34)) + [100, 257])
def test_audit_paths_verify_and_match_rfc(n):
    e = entries(n)
    leaves = [H(b"\x00" + x) for x in e]
    root = verde_merkle_root(e)
    assert root == oracle.merkle_root(e) == mth(leaves)
    blob = b"".join(e)
    for m in range(n) if n <= 40 else [0, 1, n // 2, n - 2, n - 1]:
        p = verde_merkle_audit_path(blob, m)
        assert p == path(m, leaves)
        assert verde_merkle_verify_path(leaves[m], m, n, p, root)
        # a different leaf, a different index or a different tree size must fail
        assert not verde_merkle_verify_path(H(b"\x00" + H(b"forged")), m, n, p, root)
        if n > 1:
            assert not verde_merkle_verify_path(leaves[m], (m + 1) % n, n, p, root)
            assert not verde_merkle_verify_path(leaves[m], m, n, p[:-1], root)
        # hashed mode: the same proofs over given leaf hashes
        assert verde_merkle_audit_path(b"".join(leaves), m, hashed=True) == p


def test_hashed_root_and_divergence():
    leaves = [H(b"\x00" + os.urandom(8)) for _ in range(77)]
    assert verde_merkle_root_hashed(b"".join(leaves)) == mth(leaves)
    other = list(leaves)
    other[41] = H(b"x")
    assert verde_first_divergence(b"".join(leaves), b"".join(other), hashed=True)[0] == 41
    assert verde_first_divergence(b"".join(leaves), b"".join(leaves), hashed=True)[0] == -1


@pytest.mark.parametrize("shape", [(3,), (1024,), (1025,), (5, 3001), (0,)])
def test_tensor_digest_from_chunk_leaves_equals_oracle_commit(shape):
    a = synth.uniform(9, shape) if int(np.prod(shape)) else np.zeros(shape, np.float32)
    raw = a.tobytes()
    if raw:
        leaves = [H(b"\x00" + raw[i:i + 4096]) for i in range(0, len(raw), 4096)]
        root = verde_merkle_root_hashed(b"".join(leaves))
    else:
        root = b"\x00" * 32
    assert verde_tensor_digest_from_root(root, 1, a.shape, len(raw)) == oracle.commit_tensor(a)
