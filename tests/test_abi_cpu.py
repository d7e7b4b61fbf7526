"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every
symbol include/repops.h declares, validates arguments without touching the
device, and its host-side Verde functions (SHA-256, RFC 6962 root, node
digest, divergence search) agree with hashlib / an independent Python
serialisation."""
import ctypes as C
import hashlib
import struct

import pytest

import paper_2502_19405_b200 as R
from paper_2502_19405_b200 import _lib


def H(b):
    return hashlib.sha256(b).digest()


def mth(entries):
    if len(entries) == 1:
        return H(b"\x00" + entries[0])
    k = 1
    while 2 * k < len(entries):
        k *= 2
    return H(b"\x01" + mth(entries[:k]) + mth(entries[k:]))


def test_library_exports_every_header_symbol():
    syms = R.header_symbols()
    assert len(syms) >= 30
    L = R.lib()
    for s in syms:
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, s
    assert L.repops_abi_version() == 1


def test_invalid_arguments_fail_without_device():
    L = R.lib()
    assert L.repops_gemm(-1, 2, 2, None, 2, 0, None, 2, 0, 0, None, 1.0, None, 2, None) == 1
    assert b"negative" in L.repops_last_error()
    assert L.repops_gemm(2, 2, 2, None, 2, 0, None, 2, 0, 7, None, 1.0, None, 2, None) == 1
    assert L.repops_softmax(C.c_void_p(16), 3, 2, 2, 1, C.c_void_p(16), 2, None) == 2  # ESHAPE
    assert L.repops_tree_sum(None, 3, 10, None, None) == 1
    assert L.repops_layernorm(None, None, None, 4, 5000, 1e-5, None, None, None, None) == 1
    # zero-extent calls are no-ops that succeed
    assert L.repops_gemm(0, 5, 5, None, 5, 0, None, 5, 0, 0, None, 1.0, None, 5, None) == 0
    out = C.create_string_buffer(32)
    assert L.verde_merkle_root(None, 0, out) == 1  # empty leaf list


def test_host_sha256_vs_hashlib():
    blob = bytes(range(256)) * 3
    for n in list(range(0, 130)) + [700, 768]:
        assert R.verde_sha256(blob[:n]) == H(blob[:n])


@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 9, 100, 2673])
def test_host_merkle_root_vs_python(n):
    digs = [H(struct.pack("<Q", i)) for i in range(n)]
    assert R.verde_merkle_root(digs) == mth(digs)


def test_node_digest_serialisation():
    ind = [H(b"in0"), H(b"in1")]
    outd = [H(b"out0")]
    attrs = {3: 0x3E000000, 1: 7}
    got = R.verde_node_digest(index=12, op=5, shard=3, attrs=attrs, inputs=[(4, 0), (9, 1)], dsts=[13, 20],
                              in_digests=ind, out_digests=outd)
    ser = b"\x4e" + struct.pack("<IHI", 12, 5, 3) + struct.pack("<I", 2)
    ser += struct.pack("<IQ", 1, 7) + struct.pack("<IQ", 3, 0x3E000000)
    ser += struct.pack("<I", 2) + struct.pack("<II", 4, 0) + struct.pack("<II", 9, 1)
    ser += struct.pack("<I", 2) + struct.pack("<II", 13, 20) + struct.pack("<I", 1)
    ser += b"".join(ind) + b"".join(outd)
    assert got == H(ser)


@pytest.mark.parametrize("n,d", [(1, 0), (2, 1), (5, 4), (2673, 0), (2673, 1234), (2673, 2672), (64, 33)])
def test_first_divergence(n, d):
    a = [H(struct.pack("<I", i)) for i in range(n)]
    b = list(a)
    b[d] = H(b"tampered")
    for j in range(d + 1, n):  # everything after d may differ too
        if j % 3 == 0:
            b[j] = H(b"x" + struct.pack("<I", j))
    got, rounds = R.verde_first_divergence(b"".join(a), b"".join(b))
    assert got == d
    assert rounds <= 2 + (n - 1).bit_length()
    same, _ = R.verde_first_divergence(b"".join(a), b"".join(a))
    assert same == -1


@pytest.mark.parametrize("n,k", [(1024, 1), (1024, 2), (1024, 4), (1024, 8), (2048, 8), (64, 2)])
def test_digest_from_subroots_equals_oracle_whole_tensor_commit(n, k):
    """Config-2 M-split: rank r commits only the data root of
    its (n/k) x n slab; verde_digest_from_subroots joins the k slab roots into the digest
    of the whole n x n output.  It must equal the oracle's R-TCOMMIT of the full tensor
    (the slabs are aligned power-of-two chunk groups, so the RFC 6962 tree splits there)."""
    import numpy as np

    import oracle
    import synth
    C_ = synth.uniform(synth.seed_for("msplit", n, k), (n, n))
    rows = n // k
    sub = b"".join(oracle.data_root(C_[r * rows:(r + 1) * rows]) for r in range(k))
    got = R.verde_digest_from_subroots(sub, R.F32, (n, n), n * n * 4)
    assert got == oracle.commit_tensor(C_)
    # a slab root out of order, or a flipped bit in one slab, changes the digest
    if k > 1:
        swapped = sub[32:64] + sub[:32] + sub[64:]
        assert R.verde_digest_from_subroots(swapped, R.F32, (n, n), n * n * 4) != got
    D = C_.copy()
    D.reshape(-1).view(np.uint32)[n * n - 1] ^= 1
    sub2 = b"".join(oracle.data_root(D[r * rows:(r + 1) * rows]) for r in range(k))
    assert R.verde_digest_from_subroots(sub2, R.F32, (n, n), n * n * 4) != got


def test_digest_from_subroots_rejects_unaligned_slabs():
    with pytest.raises(RuntimeError):
        R.verde_digest_from_subroots(b"\0" * 96, R.F32, (96, 1024), 96 * 1024 * 4)   # k = 3
    with pytest.raises(RuntimeError):
        R.verde_digest_from_subroots(b"\0" * 64, R.F32, (3, 1024), 3 * 1024 * 4)     # 1.5 chunks per slab
