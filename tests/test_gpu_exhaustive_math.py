"""Exhaustive GPU-vs-oracle parity of the software math functions (SURVEY.md §8(c)
pin table: "Exhaustive 2^32 GPU-vs-oracle 0-ULP"; "re-implements ...
mathematical functions"): every one of the 2^32 binary32 bit patterns (all
exponents, both signs, subnormals, infinities, every NaN payload) through the
CUDA kernel and through the oracle, compared chunk by chunk as SHA-256 digests of
the raw output bytes.

The oracle side runs in a pool of host processes (one 2^24-element chunk per job,
inputs generated from the chunk index, no data from the GPU); the GPU side
generates the same bit patterns on the device, runs the product's kernel and
hashes the copied-back chunk on a thread pool.  A differing chunk is then
compared element by element to report the first differing inputs."""
import concurrent.futures as cf
import hashlib
import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CHUNK = 1 << 24
NCHUNK = (1 << 32) // CHUNK
FUNCS = ["exp", "log", "tanh", "rsqrt", "erf", "sin", "cos"]


def _oracle_chunk(args):
    fn, c = args
    import oracle
    x = (np.arange(CHUNK, dtype=np.uint64) + np.uint64(c * CHUNK)).astype(np.uint32).view(np.float32)
    y = getattr(oracle, fn)(x)
    return c, hashlib.sha256(np.ascontiguousarray(y).view(np.uint8)).digest()


@pytest.fixture(scope="module")
def pool():
    import oracle
    oracle.lib()  # build / load once before forking
    n = max(2, (os.cpu_count() or 2) - 2)
    with mp.get_context("fork").Pool(n) as p:
        yield p


@pytest.mark.parametrize("fn", FUNCS)
def test_all_2_32_inputs_bit_identical(fn, pool):
    import oracle
    import paper_2502_19405_b200 as R
    torch.cuda.set_device(0)
    kern = getattr(R, "repops_" + fn)
    ref_async = pool.map_async(_oracle_chunk, [(fn, c) for c in range(NCHUNK)], chunksize=4)
    base = torch.arange(CHUNK, dtype=torch.int64, device="cuda")
    y = torch.empty(CHUNK, dtype=torch.float32, device="cuda")
    hosts = [torch.empty(CHUNK, dtype=torch.float32).pin_memory() for _ in range(4)]
    futs = {}
    with cf.ThreadPoolExecutor(4) as ex:
        for c in range(NCHUNK):
            v = base + c * CHUNK                                  # bit patterns c*2^24 ... c*2^24 + 2^24 - 1
            x = torch.where(v >= 2 ** 31, v - 2 ** 32, v).to(torch.int32).view(torch.float32)
            kern(x, out=y)
            h = hosts[c % 4]
            if c >= 4:
                futs[c - 4].result()  # the host buffer is free again
            h.copy_(y)
            futs[c] = ex.submit(lambda a: hashlib.sha256(a.numpy().view(np.uint8)).digest(), h)
        gpu = {c: f.result() for c, f in futs.items()}
    ref = dict(ref_async.get(timeout=3000))
    bad = [c for c in range(NCHUNK) if gpu[c] != ref[c]]
    if bad:
        c = bad[0]
        x = (np.arange(CHUNK, dtype=np.uint64) + np.uint64(c * CHUNK)).astype(np.uint32).view(np.float32)
        g = kern(torch.from_numpy(x.copy()).cuda()).cpu().numpy().view(np.uint32)
        r = getattr(oracle, fn)(x).view(np.uint32)
        idx = np.flatnonzero(g != r)[:5]
        pytest.fail(f"{fn}: {len(bad)} of {NCHUNK} chunks differ; first inputs "
                    f"{[hex(int(v)) for v in x.view(np.uint32)[idx]]} gpu {[hex(int(v)) for v in g[idx]]} "
                    f"oracle {[hex(int(v)) for v in r[idx]]}")
