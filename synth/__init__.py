"""Seeded synthetic input generators shared by the oracle side and the GPU side.

This module holds NO arithmetic of the method (no GEMM, reduction, math
function or hash): it only turns (seed, index) into bits.  Both sides of every
parity test receive the SAME arrays from here, so nothing either side computes
can leak into the other's inputs.

Generator: SplitMix64, counter based -- element i of stream `seed` is
splitmix64(seed + (i+1) * 0x9E3779B97F4A7C15).  Floats are drawn on a 24-bit
grid, u = (x >> 40) * 2^-23 - 1 in [-1, 1), so every draw is exact in binary32.
Integers in [0, n) use Lemire's multiply-shift on the top 32 bits.

Workload recipes are stated next to each helper.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """n consecutive SplitMix64 outputs of stream `seed`, starting at counter `offset`."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed: int, shape, scale: float = 1.0) -> np.ndarray:
    """float32 U[-1, 1) on a 24-bit grid (exact), optionally times `scale`
    (the product is rounded to binary32 once, here, before either side sees it)."""
    shape = (shape,) if isinstance(shape, int) else tuple(shape)
    n = int(np.prod(shape)) if shape else 1
    k = (splitmix64(seed, n) >> np.uint64(40)).astype(np.float64)
    x = (k * (2.0 ** -23) - 1.0).astype(np.float32)
    if scale != 1.0:
        x = (x.astype(np.float64) * scale).astype(np.float32)
    return x.reshape(shape)


def integers(seed: int, n: int, hi: int) -> np.ndarray:
    """int32 uniform in [0, hi) by Lemire multiply-shift of the top 32 bits."""
    top = (splitmix64(seed, n) >> np.uint64(32)).astype(np.uint64)
    return ((top * np.uint64(hi)) >> np.uint64(32)).astype(np.int32)


def small_ints(seed: int, shape, lo: int = -8, hi: int = 8) -> np.ndarray:
    """float32 integers in [lo, hi) -- for GEMMs whose every partial sum is exact."""
    shape = (shape,) if isinstance(shape, int) else tuple(shape)
    n = int(np.prod(shape))
    return (integers(seed, n, hi - lo).astype(np.int64) + lo).astype(np.float32).reshape(shape)


def seed_for(*labels) -> int:
    """Stable 64-bit stream id from labels (FNV-1a over their text)."""
    h = 0xCBF29CE484222325
    for ch in "/".join(str(x) for x in labels).encode():
        h ^= ch
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


# ----------------------------------------------------------------- recipes
def gemm_inputs(n_or_mnk, tag: str = "gemm"):
    """Config 1/2: A, B ~ U[-1,1) (24-bit grid).  Returns (A[M,K], B[K,N])."""
    if isinstance(n_or_mnk, int):
        M = N = K = n_or_mnk
    else:
        M, N, K = n_or_mnk
    A = uniform(seed_for(tag, "A", M, N, K), (M, K))
    B = uniform(seed_for(tag, "B", M, N, K), (K, N))
    return A, B


# ----------------------------------------------------------------- GPT-2 (BASELINE config 3)
def gpt2_param_specs(n_layer, d, ffn, vocab, n_pos):
    """(name, shape, kind) in the canonical GPT-2 order.  kind: 'w' (2-D weight,
    U[-a, a) with a = 0.02*sqrt(3), i.e. std 0.02), 'g' (LN gain = 1), 'b' (zeros)."""
    specs = [("wte", (vocab, d), "w"), ("wpe", (n_pos, d), "w")]
    for l in range(n_layer):
        p = f"h{l}."
        specs += [(p + "ln1.g", (d,), "g"), (p + "ln1.b", (d,), "b"),
                  (p + "attn.w", (d, 3 * d), "w"), (p + "attn.b", (3 * d,), "b"),
                  (p + "proj.w", (d, d), "w"), (p + "proj.b", (d,), "b"),
                  (p + "ln2.g", (d,), "g"), (p + "ln2.b", (d,), "b"),
                  (p + "fc.w", (d, ffn), "w"), (p + "fc.b", (ffn,), "b"),
                  (p + "fc2.w", (ffn, d), "w"), (p + "fc2.b", (d,), "b")]
    specs += [("lnf.g", (d,), "g"), ("lnf.b", (d,), "b")]
    return specs


def gpt2_param(name, shape, kind, seed=0):
    if kind == "w":
        return uniform(seed_for("gpt2", seed, name), shape, 0.034641016151377546)
    if kind == "g":
        return np.ones(shape, np.float32)
    return np.zeros(shape, np.float32)


def gpt2_tokens(vocab, seq, shard, step=0, seed=0):
    """seq+1 tokens of one shard (one sequence); input = [:-1], target = [1:]."""
    return integers(seed_for("gpt2-tokens", seed, step, shard), seq + 1, vocab)


# ----------------------------------------------------------------- Llama-3-8B-shaped prefill (config 4)
def mlp_inputs(batch=32, width=256, classes=256, seed=0):
    """Config-1 MLP: x[batch x width] U[-1,1); W1 [width x width],
    W2 [width x classes], b1, b2 U[-1/16, 1/16); labels U{0..classes-1}."""
    u = lambda name, shape, scale=1.0: uniform(seed_for("mlp", seed, name), shape, scale)  # noqa: E731
    return {"x": u("x", (batch, width)), "W1": u("W1", (width, width), 1 / 16), "b1": u("b1", width, 1 / 16),
            "W2": u("W2", (width, classes), 1 / 16), "b2": u("b2", classes, 1 / 16),
            "labels": integers(seed_for("mlp", seed, "labels"), batch, classes)}


def llama_param_specs(n_layer, d, n_head, n_kv, hd, ffn, vocab):
    """(name, shape, kind) in canonical order; weights stored [in, out] (y = x W)."""
    specs = [("tok_emb", (vocab, d), "w")]
    for l in range(n_layer):
        p = f"l{l}."
        specs += [(p + "attn_norm", (d,), "g"), (p + "wq", (d, n_head * hd), "w"), (p + "wk", (d, n_kv * hd), "w"),
                  (p + "wv", (d, n_kv * hd), "w"), (p + "wo", (n_head * hd, d), "w"), (p + "mlp_norm", (d,), "g"),
                  (p + "w_gate", (d, ffn), "w"), (p + "w_up", (d, ffn), "w"), (p + "w_down", (ffn, d), "w")]
    specs += [("norm", (d,), "g"), ("lm_head", (d, vocab), "w")]
    return specs


def llama_param_seed(name, seed=0):
    return seed_for("llama", seed, name)


LLAMA_WSCALE = 0.034641016151377546  # U[-a, a), std 0.02


def llama_param(name, shape, kind, seed=0):
    if kind == "w":
        return uniform(llama_param_seed(name, seed), shape, LLAMA_WSCALE)
    return np.ones(shape, np.float32)


def llama_tokens(vocab, seq, seed=0):
    return integers(seed_for("llama-tokens", seed), seq, vocab)


def rope_inv_freq(hd, theta=500000.0):
    """RoPE inverse frequencies theta^(-2i/hd), i < hd/2 (float64, rounded once): input data
    of config 4; the cos/sin tables are computed from them by R26."""
    return (theta ** (-np.arange(0, hd, 2, dtype=np.float64) / hd)).astype(np.float32)


def rope_tables(seq, hd, theta=500000.0):
    """cos/sin tables [seq, hd/2] (float64 angles rounded once to binary32): input data."""
    inv = theta ** (-np.arange(0, hd, 2, dtype=np.float64) / hd)
    ang = np.arange(seq, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
