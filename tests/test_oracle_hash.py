"""Pins for the oracle's SHA-256 (FIPS 180-4), RFC 6962 MTH (reading R12) and
tensor commitment R-TCOMMIT (reading R11) -- against the published vectors in
tests/golden/ and against Python's hashlib (an independent SHA-256)."""
import hashlib
import os
import struct

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _fips():
    for line in open(os.path.join(GOLD, "sha256_fips180.txt")):
        if line.startswith("#") or not line.strip():
            continue
        spec, hexd = line.split()
        if spec == "empty":
            msg = b""
        elif spec.startswith("rep:"):
            _, n, ch = spec.split(":")
            msg = ch.encode() * int(n)
        else:
            msg = spec.encode()
        yield msg, hexd


def _rfc():
    leaves, roots = None, {}
    for line in open(os.path.join(GOLD, "rfc6962_mth.txt")):
        if line.startswith("#") or not line.strip():
            continue
        if line.startswith("leaves:"):
            leaves = [b"" if h == "-" else bytes.fromhex(h) for h in line.split()[1:]]
        else:
            n, h = line.split()
            roots[int(n)] = h
    return leaves, roots


def H(b):
    return hashlib.sha256(b).digest()


def mth_levelwise(entries):
    """RFC 6962 MTH computed level by level with odd-node promotion (a different
    formulation from the recursive definition the oracle writes out)."""
    if not entries:
        return H(b"")
    level = [H(b"\x00" + e) for e in entries]
    while len(level) > 1:
        nxt = [H(b"\x01" + level[i] + level[i + 1]) for i in range(0, len(level) - 1, 2)]
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    return level[0]


def test_fips_vectors():
    for msg, hexd in _fips():
        assert oracle.sha256(msg).hex() == hexd


def test_sha256_vs_hashlib_all_padding_lengths():
    blob = synth.integers(1, 300, 256).astype(np.uint8).tobytes()
    for n in range(0, 300):
        assert oracle.sha256(blob[:n]) == H(blob[:n]), n


def test_rfc6962_reference_roots():
    leaves, roots = _rfc()
    for n, h in roots.items():
        assert oracle.mth(leaves[:n]).hex() == h
    assert oracle.mth([]) == H(b"")


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13, 64, 100, 257, 299])
def test_merkle_root_equals_levelwise_promotion(n):
    digs = [H(struct.pack("<I", i)) for i in range(n)]
    assert oracle.merkle_root(digs) == mth_levelwise(digs)


def test_merkle_root_empty_is_error():
    with pytest.raises(ValueError):
        oracle.merkle_root([])


def _commit_ref(arr: np.ndarray, dtype_code: int) -> bytes:
    raw = arr.tobytes()  # little-endian binary32 image on x86
    chunks = [raw[i:i + 4096] for i in range(0, len(raw), 4096)]
    root = mth_levelwise(chunks) if chunks else H(b"")
    hdr = b"\x54" + bytes([dtype_code]) + struct.pack("<Q", arr.ndim)
    hdr += b"".join(struct.pack("<Q", d) for d in arr.shape)
    hdr += struct.pack("<Q", len(raw)) + struct.pack("<I", 4096)
    return H(hdr + root)


@pytest.mark.parametrize("shape", [(0,), (1,), (1023,), (1024,), (1025,), (3, 4096), (7, 1000, 3), ()])
def test_commit_tensor_vs_hashlib(shape):
    a = synth.uniform(synth.seed_for("commit", shape), shape if shape else (1,)).reshape(shape)
    assert oracle.commit_tensor(a) == _commit_ref(a, 1)


def test_commit_distinguishes_shape_and_single_bit():
    a = synth.uniform(3, 4096)
    d0 = oracle.commit_tensor(a)
    # scalar vs [1]-shape differ; reshape differs; 1-bit flip differs
    assert oracle.commit_tensor(np.float32(1.0).reshape(())) != oracle.commit_tensor(np.float32([1.0]))
    assert oracle.commit_tensor(a.reshape(64, 64)) != d0
    b = a.copy()
    b.view(np.uint32)[1234] ^= 1
    assert oracle.commit_tensor(b) != d0
    assert oracle.commit_tensor(a.copy()) == d0
