"""Oracle Llama prefill forward -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain composition of the oracle's canonical operators for the config-4 model
(RMSNorm, GQA attention with RoPE, SwiGLU MLP, untied LM head), written per
tensor-parallel column block so that every tensor has the product's name:
block b = query heads [b*qh, (b+1)*qh), KV head b, columns [b*w, (b+1)*w) of
every other weight.  The math of a column block is just the corresponding
output columns of the full operator (an N split never changes an output
element's K order), so this is the model written out block by block.
"""
from __future__ import annotations

import numpy as np

import synth

from . import add, gemm, rmsnorm, rope, rope_tables_from_inv_freq, softmax, swiglu


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def run_prefill(cfg, tokens=None):
    L, d, H, KV, hd, F, V, T, nb = cfg.n_layer, cfg.d, cfg.n_head, cfg.n_kv, cfg.hd, cfg.ffn, cfg.vocab, cfg.seq, cfg.nb
    qh = H // nb
    Db, Fb, Vb = d // nb, F // nb, V // nb
    specs = synth.llama_param_specs(L, d, H, KV, hd, F, V)
    W = {n: synth.llama_param(n, s, k, cfg.seed) for n, s, k in specs}
    tok = synth.llama_tokens(V, T, cfg.seed) if tokens is None else tokens
    inv = synth.rope_inv_freq(hd, cfg.theta)
    cos, sin = rope_tables_from_inv_freq(inv, T)   # R26
    scale = float(np.float32(1.0 / np.sqrt(hd)))
    out = {"tokens": tok.astype(np.int32), "rope/inv_freq": inv, "rope/cos": cos, "rope/sin": sin}
    x = _c(W["tok_emb"][tok])  # exact gather
    out["x0"] = x
    for l in range(L):
        p, q0 = f"l{l}.", f"l{l}/"
        xn, rs1 = rmsnorm(x, W[p + "attn_norm"], cfg.eps)
        out[q0 + "xn"], out[q0 + "rs1"] = xn, rs1
        o_all = np.empty((T, H * hd), np.float32)
        for b in range(nb):
            q = f"l{l}/b{b}/"
            wqkv = np.concatenate([W[p + "wq"][:, b * qh * hd:(b + 1) * qh * hd], W[p + "wk"][:, b * hd:(b + 1) * hd],
                                   W[p + "wv"][:, b * hd:(b + 1) * hd]], axis=1)
            qkv = gemm(xn, _c(wqkv))
            qk = rope(_c(qkv[:, :(qh + 1) * hd]), cos, sin, qh + 1, hd)
            S = np.empty((qh * T, T), np.float32)
            P = np.empty((qh * T, T), np.float32)
            ob = np.empty((T, qh * hd), np.float32)
            k = _c(qk[:, qh * hd:(qh + 1) * hd])
            v = _c(qkv[:, (qh + 1) * hd:])
            for j in range(qh):
                S[j * T:(j + 1) * T] = gemm(_c(qk[:, j * hd:(j + 1) * hd]), k, transB=True, epi=2, scale=scale)
                P[j * T:(j + 1) * T] = softmax(S[j * T:(j + 1) * T], causal=True)
                ob[:, j * hd:(j + 1) * hd] = gemm(_c(P[j * T:(j + 1) * T]), v)
            # R29: attention is one operator; S and P are internal (not committed tensors)
            out.update({q + "qkv": qkv, q + "qk_rope": qk, q + "attn_out": ob})
            o_all[:, b * qh * hd:(b + 1) * qh * hd] = ob
        attn = np.empty((T, d), np.float32)
        for b in range(nb):
            ob = gemm(o_all, _c(W[p + "wo"][:, b * Db:(b + 1) * Db]))
            out[f"l{l}/b{b}/oproj"] = ob
            attn[:, b * Db:(b + 1) * Db] = ob
        h = add(x, attn)
        hn, rs2 = rmsnorm(h, W[p + "mlp_norm"], cfg.eps)
        out.update({q0 + "h": h, q0 + "hn": hn, q0 + "rs2": rs2})
        a_all = np.empty((T, F), np.float32)
        for b in range(nb):
            q = f"l{l}/b{b}/"
            g = gemm(hn, _c(W[p + "w_gate"][:, b * Fb:(b + 1) * Fb]))
            u = gemm(hn, _c(W[p + "w_up"][:, b * Fb:(b + 1) * Fb]))
            a = swiglu(g, u)
            out.update({q + "gate": g, q + "up": u, q + "swiglu": a})
            a_all[:, b * Fb:(b + 1) * Fb] = a
        mlp = np.empty((T, d), np.float32)
        for b in range(nb):
            dn = gemm(a_all, _c(W[p + "w_down"][:, b * Db:(b + 1) * Db]))
            out[f"l{l}/b{b}/down"] = dn
            mlp[:, b * Db:(b + 1) * Db] = dn
        x = add(h, mlp)
        out[f"x{l + 1}"] = x
    xf, rsf = rmsnorm(x, W["norm"], cfg.eps)
    out["xf"], out["rsf"] = xf, rsf
    for b in range(nb):
        out[f"b{b}/logits"] = gemm(xf, _c(W["lm_head"][:, b * Vb:(b + 1) * Vb]))
    return out, W
