"""Oracle GPT-2 training step -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

A plain, per-shard, per-head composition of the oracle's canonical operators
(repops_oracle.c) for one training step of the paper's program (PAPER.md
P:199-205: "a training step comprises a forward pass, backward pass, parameter
updates and an optimizer state update"), written out in the order the math
defines it:

  forward  (per shard s, per layer l):
      ln1 = LN(x);  qkv = ln1 W_attn + b;  S_h = (Q_h K_h^T) * 1/sqrt(hd);
      P_h = causal softmax(S_h);  att_h = P_h V_h;  proj = att W_proj + b;
      xmid = x + proj;  ln2 = LN(xmid);  fc = ln2 W_fc + b;  g = GELU(fc);
      fc2 = g W_fc2 + b;  x' = xmid + fc2
  head:    lnf = LN(x_L); logits = lnf wte^T; (loss, dlogits) = CE(logits, targets, 1/(S T))
  backward: the chain rule of each op (R-GEMM for every product, R-SEQ for the
      token-axis folds of bias / LN-parameter / embedding gradients)
  combine: grad = R-TREE_S over the 8 shards' gradients (per parameter)
  update:  AdamW (R-ADAMW), step 1

Every tensor is returned by the same name the product uses, so tests can
compare the two element by element.  Nothing here imports the product.
"""
from __future__ import annotations

import numpy as np

import synth

from . import (add, adamw, cross_entropy, embedding, embedding_backward, gelu, gelu_backward, gemm,
               layernorm, layernorm_backward, layernorm_backward_params, softmax, softmax_backward,
               sum_cols_seq, tree_sum)


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def layer_forward(W, l, x, cfg):
    """Forward of transformer block l for one shard: x [T, d] -> dict of every
    tensor the block commits (names without the "s{s}/h{l}/" prefix) plus "x_next"."""
    d, H, T = cfg.d, cfg.n_head, cfg.seq
    hd = d // H
    scale = float(np.float32(1.0 / np.sqrt(hd)))
    p = f"h{l}."
    ln1, mu1, rs1 = layernorm(x, W[p + "ln1.g"], W[p + "ln1.b"], cfg.ln_eps)
    qkv = gemm(ln1, W[p + "attn.w"], epi=1, bias=W[p + "attn.b"])
    Sc = np.empty((H * T, T), np.float32)
    Pr = np.empty((H * T, T), np.float32)
    att = np.empty((T, d), np.float32)
    for h in range(H):
        Q = _c(qkv[:, h * hd:(h + 1) * hd])
        K = _c(qkv[:, d + h * hd:d + (h + 1) * hd])
        Vh = _c(qkv[:, 2 * d + h * hd:2 * d + (h + 1) * hd])
        Sc[h * T:(h + 1) * T] = gemm(Q, K, transB=True, epi=2, scale=scale)
        Pr[h * T:(h + 1) * T] = softmax(Sc[h * T:(h + 1) * T], causal=True)
        att[:, h * hd:(h + 1) * hd] = gemm(_c(Pr[h * T:(h + 1) * T]), Vh)
    proj = gemm(att, W[p + "proj.w"], epi=1, bias=W[p + "proj.b"])
    xmid = add(x, proj)
    ln2, mu2, rs2 = layernorm(xmid, W[p + "ln2.g"], W[p + "ln2.b"], cfg.ln_eps)
    fc = gemm(ln2, W[p + "fc.w"], epi=1, bias=W[p + "fc.b"])
    g = gelu(fc)
    fc2 = gemm(g, W[p + "fc2.w"], epi=1, bias=W[p + "fc2.b"])
    xn = add(xmid, fc2)
    return {"ln1": ln1, "mu1": mu1, "rs1": rs1, "qkv": qkv, "scores": Sc, "probs": Pr, "att": att, "proj": proj,
            "xmid": xmid, "ln2": ln2, "mu2": mu2, "rs2": rs2, "fc": fc, "gelu": g, "fc2": fc2, "x_next": xn}


def layer_backward(W, l, x, a, dout, cfg):
    """Backward of block l for one shard from its input x, its saved forward tensors a
    (layer_forward's dict) and the output gradient dout [T, d].  Returns (tensors,
    grads): tensors by their committed names (without prefix) plus "dx" (gradient
    w.r.t. x), grads = this shard's parameter gradients of the block."""
    d, H, T = cfg.d, cfg.n_head, cfg.seq
    hd = d // H
    scale = float(np.float32(1.0 / np.sqrt(hd)))
    p = f"h{l}."
    gr = {}
    dgelu = gemm(dout, W[p + "fc2.w"], transB=True)
    gr[p + "fc2.w"] = gemm(a["gelu"], dout, transA=True)
    gr[p + "fc2.b"] = sum_cols_seq(dout)[0]
    dfc = gelu_backward(a["fc"], dgelu)
    dln2 = gemm(dfc, W[p + "fc.w"], transB=True)
    gr[p + "fc.w"] = gemm(a["ln2"], dfc, transA=True)
    gr[p + "fc.b"] = sum_cols_seq(dfc)[0]
    dxmid = layernorm_backward(dln2, a["xmid"], W[p + "ln2.g"], a["mu2"], a["rs2"], dres=dout)
    dg, db = layernorm_backward_params(dln2, a["xmid"], a["mu2"], a["rs2"])
    gr[p + "ln2.g"], gr[p + "ln2.b"] = dg[0], db[0]
    datt = gemm(dxmid, W[p + "proj.w"], transB=True)
    gr[p + "proj.w"] = gemm(a["att"], dxmid, transA=True)
    gr[p + "proj.b"] = sum_cols_seq(dxmid)[0]
    dP = np.empty((H * T, T), np.float32)
    dS = np.empty((H * T, T), np.float32)
    dqkv = np.empty((T, 3 * d), np.float32)
    for h in range(H):
        dO = _c(datt[:, h * hd:(h + 1) * hd])
        Q = _c(a["qkv"][:, h * hd:(h + 1) * hd])
        K = _c(a["qkv"][:, d + h * hd:d + (h + 1) * hd])
        Vh = _c(a["qkv"][:, 2 * d + h * hd:2 * d + (h + 1) * hd])
        Ph = _c(a["probs"][h * T:(h + 1) * T])
        dP[h * T:(h + 1) * T] = gemm(dO, Vh, transB=True)
        dS[h * T:(h + 1) * T] = softmax_backward(Ph, dP[h * T:(h + 1) * T], scale=scale)
        dSh = _c(dS[h * T:(h + 1) * T])
        dqkv[:, 2 * d + h * hd:2 * d + (h + 1) * hd] = gemm(Ph, dO, transA=True)
        dqkv[:, h * hd:(h + 1) * hd] = gemm(dSh, K)
        dqkv[:, d + h * hd:d + (h + 1) * hd] = gemm(dSh, Q, transA=True)
    dln1 = gemm(dqkv, W[p + "attn.w"], transB=True)
    gr[p + "attn.w"] = gemm(a["ln1"], dqkv, transA=True)
    gr[p + "attn.b"] = sum_cols_seq(dqkv)[0]
    dxn = layernorm_backward(dln1, x, W[p + "ln1.g"], a["mu1"], a["rs1"], dres=dxmid)
    dg, db = layernorm_backward_params(dln1, x, a["mu1"], a["rs1"])
    gr[p + "ln1.g"], gr[p + "ln1.b"] = dg[0], db[0]
    t = {"dgelu": dgelu, "dfc": dfc, "dln2": dln2, "dxmid": dxmid, "datt": datt, "dP": dP, "dS": dS, "dqkv": dqkv,
         "dln1": dln1, "dx": dxn}
    return t, gr


def run_step(cfg, tokens=None, step=1):
    """cfg: object with n_layer, d, n_head, ffn, vocab, n_pos, seq, shards, ln_eps, lr,
    beta1, beta2, adam_eps, wd, seed, vocab_ld.  Returns (tensors: dict name -> array,
    params: dict, new_params/m/v dicts)."""
    L, d, V, T, S = cfg.n_layer, cfg.d, cfg.vocab, cfg.seq, cfg.shards
    ce_scale = 1.0 / (S * T)
    specs = synth.gpt2_param_specs(L, d, cfg.ffn, V, cfg.n_pos)
    W = {name: synth.gpt2_param(name, shape, kind, cfg.seed) for name, shape, kind in specs}
    out = {}
    grads = {name: [None] * S for name, _, _ in specs}
    for s in range(S):
        tok = synth.gpt2_tokens(V, T, s, 0, cfg.seed) if tokens is None else tokens[s]
        tin, tgt = tok[:T], tok[1:]
        pre = f"s{s}/"
        out[pre + "tokens"] = tok.astype(np.int32)
        x = embedding(tin, W["wte"], W["wpe"], T)
        out[pre + "x0"] = x
        saved = []
        for l in range(L):
            q = f"s{s}/h{l}/"
            a = layer_forward(W, l, x, cfg)
            out.update({q + k: v for k, v in a.items() if k != "x_next"})
            out[f"s{s}/x{l + 1}"] = a["x_next"]
            saved.append((x, a))
            x = a["x_next"]
        q = f"s{s}/head/"
        lnf, muf, rsf = layernorm(x, W["lnf.g"], W["lnf.b"], cfg.ln_eps)
        logits = gemm(lnf, W["wte"], transB=True)
        loss, dlog = cross_entropy(logits, tgt, scale=ce_scale)
        pad = lambda a: np.concatenate([a, np.zeros((T, cfg.vocab_ld - V), np.float32)], 1)  # noqa: E731
        out.update({q + "lnf": lnf, q + "muf": muf, q + "rsf": rsf, q + "logits": pad(logits), q + "loss": loss,
                    q + "dlogits": pad(dlog)})
        # ---- backward: head
        dlnf = gemm(dlog, W["wte"])
        gwte_lm = gemm(dlog, lnf, transA=True)
        dx = layernorm_backward(dlnf, x, W["lnf.g"], muf, rsf)
        dg, db = layernorm_backward_params(dlnf, x, muf, rsf)
        out.update({q + "dlnf": dlnf, f"s{s}/grad/wte_lm": gwte_lm, f"s{s}/dx{L}": dx})
        grads["lnf.g"][s], grads["lnf.b"][s] = dg[0], db[0]
        # ---- backward: layers
        for l in reversed(range(L)):
            q = f"s{s}/h{l}/"
            xl, a = saved[l]
            t, gr = layer_backward(W, l, xl, a, dx, cfg)
            for name, g in gr.items():
                grads[name][s] = g
            out.update({q + k: v for k, v in t.items() if k != "dx"})
            out[f"s{s}/dx{l}"] = t["dx"]
            dx = t["dx"]
        gwte, gwpe = embedding_backward(tin, dx, T, gwte_lm, np.zeros((cfg.n_pos, d), np.float32))
        grads["wte"][s], grads["wpe"][s] = gwte, gwpe
        for name, _, _ in specs:
            out[f"s{s}/grad/{name}"] = grads[name][s].reshape(W[name].shape)
    # ---- canonical combine + update
    new_p, new_m, new_v = {}, {}, {}
    for name, shape, kind in specs:
        gsum = tree_sum([grads[name][s].reshape(shape) for s in range(S)])
        out[f"grad/{name}"] = gsum
        z = np.zeros(shape, np.float32)
        pp, mm, vv = adamw(W[name], gsum, z, z, step, cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps, cfg.wd,
                           len(shape) == 2)
        new_p[name], new_m[name], new_v[name] = pp, mm, vv
        out[f"param'/{name}"], out[f"m'/{name}"], out[f"v'/{name}"] = pp, mm, vv
    return out, W, (new_p, new_m, new_v)
