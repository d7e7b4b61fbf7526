"""Oracle config-1 MLP training step -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

BASELINE.json configs[0] / SURVEY.md §8(d) row 1: Linear-ReLU-Linear-CE (SPEC
S:218's fixture grown to width 256, batch 32), data parallel over S = 8 shards of
4 rows, canonical gradient combine R-TREE_S, AdamW.  A plain composition of the
oracle's canonical operators, shard by shard:

  h = x W1 + b1 (R-GEMM, bias epilogue)   a = relu(h) (R24)   z = a W2 + b2
  (loss, dz) = CE(z, labels, scale = 1/batch)
  da = dz W2^T          dh = relu_backward(h, da)
  per shard s: gW2_s = a_s^T dz_s, gb2_s = SEQ(dz_s), gW1_s = x_s^T dh_s, gb1_s = SEQ(dh_s)
  g = R-TREE_S(g_0..g_7);  (p, m, v) = AdamW(p, g, 0, 0, step 1), decay on W1, W2 only.
"""
from __future__ import annotations

import numpy as np

import synth

from . import adamw, cross_entropy, gemm, relu, relu_backward, sum_cols_seq, tree_sum

PARAMS = ("W1", "b1", "W2", "b2")


def run_step(cfg):
    """cfg: batch, width, classes, shards, lr, beta1, beta2, adam_eps, wd, seed.
    Returns (tensors: dict name -> array, inputs dict)."""
    inp = synth.mlp_inputs(cfg.batch, cfg.width, cfg.classes, cfg.seed)
    x, y = inp["x"], inp["labels"]
    S, R = cfg.shards, cfg.batch // cfg.shards
    out = {}
    grads = {n: [] for n in PARAMS}
    for s in range(S):
        xs, ys = x[s * R:(s + 1) * R], y[s * R:(s + 1) * R]
        h = gemm(xs, inp["W1"], epi=1, bias=inp["b1"])
        a = relu(h)
        z = gemm(a, inp["W2"], epi=1, bias=inp["b2"])
        loss, dz = cross_entropy(z, ys, scale=1.0 / cfg.batch)
        da = gemm(dz, inp["W2"], transB=True)
        dh = relu_backward(h, da)
        grads["W2"].append(gemm(a, dz, transA=True))
        grads["b2"].append(sum_cols_seq(dz)[0])
        grads["W1"].append(gemm(xs, dh, transA=True))
        grads["b1"].append(sum_cols_seq(dh)[0])
        for n, v in (("h", h), ("a", a), ("z", z), ("loss", loss), ("dz", dz), ("da", da), ("dh", dh)):
            out[f"s{s}/{n}"] = v
        for n in PARAMS:
            out[f"s{s}/grad/{n}"] = grads[n][-1]
    for n in PARAMS:
        g = tree_sum(grads[n])
        out[f"grad/{n}"] = g
        z0 = np.zeros_like(inp[n])
        p, m, v = adamw(inp[n], g, z0, z0, 1, cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps, cfg.wd, inp[n].ndim == 2)
        out[f"param'/{n}"], out[f"m'/{n}"], out[f"v'/{n}"] = p, m, v
    return out, inp
