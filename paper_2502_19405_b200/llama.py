"""Llama-3-8B-shaped FP32 prefill forward, tensor-parallel N-split (BASELINE config 4).

RepOps forward of a Llama-3 decoder (RMSNorm, GQA attention with RoPE, SwiGLU
MLP, untied LM head) over T prompt tokens, with every operator output
committed and the pass's node graph hashed into a Merkle root (Verde, Fig. 2).

Tensor parallelism without reordering any reduction (PAPER.md P:585-587 and
the future-work note on model parallelism): every weight matrix is
split along its OUTPUT (N) dimension into NB = 8 column blocks; block b is
computed by rank b // (NB/G) with the full K.  Activations that a block's GEMM
needs in full (attention output, SwiGLU output, the O / down projections'
results) are all-gathered (data movement only) and placed by repops_copy2d.
Megatron's row-parallel K split + all-reduce is never used: it would change
the K order.  Nodes are defined per column block (G-independent), so the
pass's root is bit-identical for G in {1, 2, 4, 8}.

Node order (R13 analogue): params | tokens, RoPE tables, embedding | per layer:
attn RMSNorm, for each block (QKV, RoPE, attention), for each block
O-proj, residual, MLP RMSNorm, for each block (gate, up, SwiGLU), for each block
down, residual | final RMSNorm, for each block LM head.

Attention is ONE operator (reading R29, like PyTorch's scaled_dot_product_attention
node): scores R-GEMM with the 1/sqrt(hd) epilogue, causal R-SOFTMAX, then the PV
R-GEMM; its output (the per-block attention output) is committed, the scores and
probabilities are scratch shared by all layers (a referee recomputes them from the
committed Q/K/V, Verde Case 3).
"""
from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

import synth

from . import (repops_causal_suffix_flags, repops_copy2d_batched, EPI_SCALE, CommitPlan, RootPlan, repops_add, repops_copy2d, repops_fill_uniform, repops_gather_rows,
               repops_attention_probs, repops_attention_probs_supported,
               repops_gemm_strided_batched, repops_rmsnorm, repops_rope, repops_softmax, repops_swiglu,
               repops_rope_tables, repops_transpose, verde_commit_tensors)
from ._lib import check, lib
from .dist import all_gather_rows, gather_shard_digests, shard_block

OP = dict(PARAM_IN=1, TOKENS_IN=2, TABLES_IN=3, EMBED=4, RMSNORM=5, QKV=6, ROPE=7, OPROJ=11, RESIDUAL=12, GATE=13,
          UP=14, SWIGLU=15, DOWN=16, LMHEAD=17, ROPE_TABLES=18, ATTENTION=19)
REPLICATED = 0xFFFFFFFF


@dataclass
class LlamaConfig:
    n_layer: int = 32
    d: int = 4096
    n_head: int = 32
    n_kv: int = 8
    hd: int = 128
    ffn: int = 14336
    vocab: int = 128256
    seq: int = 2048
    eps: float = 1e-5
    theta: float = 500000.0
    nb: int = 8          # tensor-parallel column blocks (one KV head each)
    seed: int = 0

    @staticmethod
    def tiny():
        return LlamaConfig(n_layer=2, d=128, n_head=16, n_kv=8, hd=8, ffn=256, vocab=512, seq=64)

    @property
    def qh(self):  # query heads per block
        return self.n_head // self.nb

    def check(self):
        assert self.n_kv == self.nb and self.n_head % self.nb == 0
        assert self.d % self.nb == 0 and self.ffn % self.nb == 0 and self.vocab % self.nb == 0


@dataclass
class TRef:
    name: str
    view: torch.Tensor
    slot: int = -1
    producer: int = -1
    pslot: int = 0


@dataclass
class NRec:
    index: int
    op: int
    block: int
    attrs: dict
    inputs: list
    outputs: list
    name: str = ""
    dsts: list = field(default_factory=list)


class LlamaPrefill:
    def __init__(self, cfg: LlamaConfig, rank=0, world=1, device="cuda", pg=None, structure_only=False):
        cfg.check()
        self.cfg, self.rank, self.world, self.pg = cfg, rank, world, pg
        self.structure_only = structure_only
        self.dev = torch.device("meta" if structure_only else device)
        self.b0, self.nbl = shard_block(rank, world, cfg.nb)
        c = cfg
        self.Wb = (c.qh + 2) * c.hd        # fused per-block QKV width (qh q heads, 1 k, 1 v)
        self.Fb, self.Db, self.Vb = c.ffn // c.nb, c.d // c.nb, c.vocab // c.nb
        self.specs = synth.llama_param_specs(c.n_layer, c.d, c.n_head, c.n_kv, c.hd, c.ffn, c.vocab)
        self._alloc()
        self._build()

    # ------------------------------------------------------------------ weights
    def _alloc(self):
        c, dev, nbl, T = self.cfg, self.dev, self.nbl, self.cfg.seq
        E = lambda *s: torch.empty(*s, dtype=torch.float32, device=dev)  # noqa: E731
        L, d, hd, qh = c.n_layer, c.d, c.hd, c.qh
        self.tok = torch.empty(T, dtype=torch.int32, device=dev)
        inv = synth.rope_inv_freq(hd, c.theta)
        self.inv_freq = torch.from_numpy(inv).to(dev) if not self.structure_only else E(hd // 2)
        self.cos, self.sin = E(T, hd // 2), E(T, hd // 2)  # R26 tables, computed by the pass
        # local weights in block layout
        self.w = []
        for _ in range(L):
            self.w.append(dict(attn_norm=E(d), wqkv=E(nbl, d, self.Wb), wo=E(nbl, c.n_head * hd, self.Db),
                               mlp_norm=E(d), wg=E(nbl, d, self.Fb), wu=E(nbl, d, self.Fb),
                               wd=E(nbl, c.ffn, self.Db)))
        self.tok_emb = E(c.vocab, d)
        self.norm = E(d)
        self.wlm = E(nbl, d, self.Vb)
        # activations
        self.x = [E(T, d) for _ in range(L + 1)]
        self.act = []
        # R29: attention scores / probabilities are operator-internal scratch shared by all layers
        self.S_scr, self.P_scr = E(nbl, qh * T, T), E(nbl, qh * T, T)
        self.causal_skip = True   # f4: exact causal tile skipping in the attention GEMMs
        # f4: the fused scores + softmax kernel (hd 64 / 128), same P bits.  Off by default: at
        # the Llama shape its 16-row blocks (the widest whose 2048-column score rows fit in
        # shared memory) re-stream K per block at one CTA per SM -- 1165 us vs 767 us for the
        # causal-skip scores R-GEMM + softmax per layer (tools/llama_attn_tune.py)
        self.attn_probs = (os.environ.get("REPOPS_ATTN_PROBS_LLAMA", "0") == "1"
                           and repops_attention_probs_supported(self.cfg.seq, self.cfg.hd))
        self.vflags = torch.empty((nbl, T + 1, hd), dtype=torch.uint8, device=self.dev)
        for _ in range(L):
            self.act.append(dict(xn=E(T, d), rs1=E(T), qkv=E(nbl, T, self.Wb), qk=E(nbl, T, (qh + 1) * hd),
                                 S=self.S_scr, P=self.P_scr, o=E(nbl, T, qh * hd),
                                 o_all=E(T, c.n_head * hd), op=E(nbl, T, self.Db), attn=E(T, d), h=E(T, d),
                                 hn=E(T, d), rs2=E(T), g=E(nbl, T, self.Fb), u=E(nbl, T, self.Fb),
                                 a=E(nbl, T, self.Fb), a_all=E(T, c.ffn), dn=E(nbl, T, self.Db), mlp=E(T, d)))
        self.xf, self.rsf = E(T, d), E(T)
        # X^T scratch: the shared activation operand of every projection is transposed
        # once so the GEMMs run TN; data movement only
        self.xT = E(max(c.ffn, c.n_head * hd, d) * T)
        self.logits = E(nbl, T, self.Vb)

    def load_weights(self):
        """Generate every parameter on the device (SplitMix64, identical to synth.llama_param),
        commit the full tensors (the model checkpoint), keep this rank's column blocks."""
        c = self.cfg
        self.param_digest = {}
        d, hd, qh = c.d, c.hd, c.qh
        for name, shape, kind in self.specs:
            full = torch.empty(shape, dtype=torch.float32, device=self.dev)
            if kind == "w":
                repops_fill_uniform(full, synth.llama_param_seed(name, c.seed), synth.LLAMA_WSCALE)
            else:
                full.fill_(1.0)
            slot = self.tensors[self._pin[name]].slot
            verde_commit_tensors([full], digests=self.digests[slot:slot + 1])  # into the digest table, once
            self._place(name, full)
            del full
        torch.cuda.synchronize()

    def _place(self, name, full):
        c, hd, qh = self.cfg, self.cfg.hd, self.cfg.qh
        if name == "tok_emb":
            self.tok_emb.copy_(full)
            return
        if name == "norm":
            self.norm.copy_(full)
            return
        if name == "lm_head":
            for j in range(self.nbl):
                b = self.b0 + j
                repops_copy2d(full[:, b * self.Vb:(b + 1) * self.Vb], self.wlm[j])
            return
        l, kind = name[1:].split(".", 1)
        w = self.w[int(l)]
        if kind in ("attn_norm", "mlp_norm"):
            w[kind].copy_(full)
            return
        for j in range(self.nbl):
            b = self.b0 + j
            if kind == "wq":
                repops_copy2d(full[:, b * qh * hd:(b + 1) * qh * hd], w["wqkv"][j][:, :qh * hd])
            elif kind == "wk":
                repops_copy2d(full[:, b * hd:(b + 1) * hd], w["wqkv"][j][:, qh * hd:(qh + 1) * hd])
            elif kind == "wv":
                repops_copy2d(full[:, b * hd:(b + 1) * hd], w["wqkv"][j][:, (qh + 1) * hd:])
            elif kind == "wo":
                repops_copy2d(full[:, b * self.Db:(b + 1) * self.Db], w["wo"][j])
            elif kind == "w_gate":
                repops_copy2d(full[:, b * self.Fb:(b + 1) * self.Fb], w["wg"][j])
            elif kind == "w_up":
                repops_copy2d(full[:, b * self.Fb:(b + 1) * self.Fb], w["wu"][j])
            elif kind == "w_down":
                repops_copy2d(full[:, b * self.Db:(b + 1) * self.Db], w["wd"][j])

    # ------------------------------------------------------------------ program
    def _T(self, name, view, block):
        tid = len(self.tensors)
        self.tensors.append(TRef(name, view))
        (self._rep if block == REPLICATED else self._blk[block]).append(tid)
        return tid

    def _node(self, op, block, attrs, inputs, outputs, name):
        idx = len(self.nodes)
        self.nodes.append(NRec(idx, op, block, attrs, inputs, outputs, name))
        for q, t in enumerate(outputs):
            self.tensors[t].producer, self.tensors[t].pslot = idx, q
            if block == REPLICATED or self._local(block):
                self._cur[2].append(t)
        return idx

    def _local(self, b):
        return self.b0 <= b < self.b0 + self.nbl

    def _phase(self, name):
        self._cur = (name, [], [])
        self.phases.append(self._cur)

    def _build(self):
        c = self.cfg
        L, T, d, hd, qh, nb, nbl = c.n_layer, c.seq, c.d, c.hd, c.qh, c.nb, self.nbl
        self.tensors, self.nodes, self.phases = [], [], []
        self._rep, self._blk = [], {b: [] for b in range(nb)}
        dummy = torch.empty(0, device=self.dev)
        T_, N_ = self._T, self._node
        bv = lambda buf, b: buf[b - self.b0] if self._local(b) else dummy  # noqa: E731
        self._phase("inputs")
        pin = {}
        for name, shape, kind in self.specs:
            pin[name] = T_("param/" + name, dummy, REPLICATED)   # digest computed at load time
            N_(OP["PARAM_IN"], REPLICATED, {}, [], [pin[name]], "in/" + name)
        t_tok = T_("tokens", self.tok, REPLICATED)
        N_(OP["TOKENS_IN"], REPLICATED, {}, [], [t_tok], "tokens")
        t_inv = T_("rope/inv_freq", self.inv_freq, REPLICATED)
        N_(OP["TABLES_IN"], REPLICATED, {1: struct.unpack("<Q", struct.pack("<d", c.theta))[0]}, [],
           [t_inv], "rope_inv_freq")
        self._launch(lambda: repops_rope_tables(self.inv_freq, T, cos=self.cos, sin=self.sin))
        t_cos, t_sin = T_("rope/cos", self.cos, REPLICATED), T_("rope/sin", self.sin, REPLICATED)
        N_(OP["ROPE_TABLES"], REPLICATED, {}, [t_inv], [t_cos, t_sin], "rope_tables")
        self._launch(lambda: repops_gather_rows(self.tok_emb, self.tok, out=self.x[0]))
        t_x = T_("x0", self.x[0], REPLICATED)
        N_(OP["EMBED"], REPLICATED, {}, [t_tok, pin["tok_emb"]], [t_x], "embed")
        scale = float(np.float32(1.0 / np.sqrt(hd)))
        for l in range(L):
            a, w, p = self.act[l], self.w[l], f"l{l}."
            self._phase(f"layer{l}")
            self._launch(lambda l=l, a=a, w=w: self._attn(l, a, w, scale))
            t_xn = T_(f"l{l}/xn", a["xn"], REPLICATED)
            t_rs1 = T_(f"l{l}/rs1", a["rs1"], REPLICATED)
            N_(OP["RMSNORM"], REPLICATED, {1: l, 2: 1}, [t_x, pin[p + "attn_norm"]], [t_xn, t_rs1], f"l{l}/attn_norm")
            t_o = []
            for b in range(nb):
                q = f"l{l}/b{b}/"
                wins = [pin[p + "wq"], pin[p + "wk"], pin[p + "wv"]]
                t_qkv = T_(q + "qkv", bv(a["qkv"], b), b)
                N_(OP["QKV"], b, {1: l}, [t_xn] + wins, [t_qkv], q + "qkv")
                t_qk = T_(q + "qk_rope", bv(a["qk"], b), b)
                N_(OP["ROPE"], b, {1: l}, [t_qkv, t_cos, t_sin], [t_qk], q + "rope")
                t_ob = T_(q + "attn_out", bv(a["o"], b), b)
                N_(OP["ATTENTION"], b, {1: l, 3: int(np.float32(scale).view(np.uint32)), 4: 1}, [t_qk, t_qkv],
                   [t_ob], q + "attention")
                t_o.append(t_ob)
            t_op = []
            for b in range(nb):
                q = f"l{l}/b{b}/"
                t = T_(q + "oproj", bv(a["op"], b), b)
                N_(OP["OPROJ"], b, {1: l}, t_o + [pin[p + "wo"]], [t], q + "oproj")
                t_op.append(t)
            t_h = T_(f"l{l}/h", a["h"], REPLICATED)
            N_(OP["RESIDUAL"], REPLICATED, {1: l, 2: 1}, [t_x] + t_op, [t_h], f"l{l}/res1")
            self._phase(f"layer{l}/mlp")
            self._launch(lambda l=l, a=a, w=w: self._mlp(l, a, w))
            t_hn = T_(f"l{l}/hn", a["hn"], REPLICATED)
            t_rs2 = T_(f"l{l}/rs2", a["rs2"], REPLICATED)
            N_(OP["RMSNORM"], REPLICATED, {1: l, 2: 2}, [t_h, pin[p + "mlp_norm"]], [t_hn, t_rs2], f"l{l}/mlp_norm")
            t_a = []
            for b in range(nb):
                q = f"l{l}/b{b}/"
                t_g = T_(q + "gate", bv(a["g"], b), b)
                N_(OP["GATE"], b, {1: l}, [t_hn, pin[p + "w_gate"]], [t_g], q + "gate")
                t_u = T_(q + "up", bv(a["u"], b), b)
                N_(OP["UP"], b, {1: l}, [t_hn, pin[p + "w_up"]], [t_u], q + "up")
                t_s = T_(q + "swiglu", bv(a["a"], b), b)
                N_(OP["SWIGLU"], b, {1: l}, [t_g, t_u], [t_s], q + "swiglu")
                t_a.append(t_s)
            t_dn = []
            for b in range(nb):
                q = f"l{l}/b{b}/"
                t = T_(q + "down", bv(a["dn"], b), b)
                N_(OP["DOWN"], b, {1: l}, t_a + [pin[p + "w_down"]], [t], q + "down")
                t_dn.append(t)
            t_x = T_(f"x{l + 1}", self.x[l + 1], REPLICATED)
            N_(OP["RESIDUAL"], REPLICATED, {1: l, 2: 2}, [t_h] + t_dn, [t_x], f"l{l}/res2")
        self._phase("head")
        self._launch(self._head)
        t_xf = T_("xf", self.xf, REPLICATED)
        t_rsf = T_("rsf", self.rsf, REPLICATED)
        N_(OP["RMSNORM"], REPLICATED, {1: L, 2: 3}, [t_x, pin["norm"]], [t_xf, t_rsf], "final_norm")
        for b in range(nb):
            t = T_(f"b{b}/logits", bv(self.logits, b), b)
            N_(OP["LMHEAD"], b, {}, [t_xf, pin["lm_head"]], [t], f"b{b}/lm_head")
        self._pin = pin
        self._finalize()

    def _launch(self, fn):
        self._cur[1].append(fn)

    # ---- launches (this rank's blocks, batched)
    def _gather_blocks(self, local, full, width):
        """all-gather [nbl, T, width] block results and place block b at full[:, b*width:(b+1)*width]."""
        allb = all_gather_rows(local, self.world, self.pg).reshape(self.cfg.nb, self.cfg.seq, width)
        # one launch for all nb blocks: block b -> columns [b*width, (b+1)*width)
        repops_copy2d_batched(allb, full, self.cfg.seq, width, width, self.cfg.seq * width, full.stride(0), width,
                              self.cfg.nb)

    def _xT(self, x):
        rows, cols = x.shape
        t = self.xT[:rows * cols].view(cols, rows)
        repops_transpose(x, out=t)
        return t

    def _attn(self, l, a, w, scale):
        c = self.cfg
        T, d, hd, qh, nbl, Wb = c.seq, c.d, c.hd, c.qh, self.nbl, self.Wb
        repops_rmsnorm(self.x[l], w["attn_norm"], c.eps, out=a["xn"], rstd=a["rs1"])
        repops_gemm_strided_batched(self._xT(a["xn"]), w["wqkv"], a["qkv"], M=T, N=Wb, K=d, lda=T, ldb=Wb, ldc=Wb,
                                    sA=(0, 0), sB=(d * Wb, 0), sC=(T * Wb, 0), batch=(nbl, 1), transA=True)
        for j in range(nbl):
            repops_rope(a["qkv"][j][:, :(qh + 1) * hd], self.cos, self.sin, qh + 1, hd, out=a["qk"][j])
        W2 = (qh + 1) * hd
        # f4 (exact causal structure, R29 scratch): score tiles entirely above the diagonal
        # are never read by the causal softmax, so they are not computed; the PV folds stop
        # at each tile's last query row and the skipped +0-probability terms are applied in
        # closed form from V's suffix flags -- the attention output bits are those of the
        # full R-GEMM -> R-SOFTMAX -> R-GEMM composition for every input
        if self.attn_probs and self.causal_skip:
            # scores + causal softmax in one kernel: the scores never leave shared memory (R29),
            # key blocks above a row block are not computed (R31); same P bits
            repops_attention_probs(a["qk"], T, hd, W2, (T * W2, hd), 0, qh * hd, (nbl, qh), a["P"],
                                   (qh * T * T, T * T), scale=scale, causal=True, sk=(T * W2, 0))
        else:
            repops_gemm_strided_batched(a["qk"], a["qk"], a["S"], M=T, N=T, K=hd, lda=W2, ldb=W2, ldc=T,
                                        sA=(T * W2, hd), sB=(T * W2, 0), sC=(qh * T * T, T * T), batch=(nbl, qh),
                                        transB=True, epi=EPI_SCALE, scale=scale, offB=qh * hd,
                                        causal=1 if self.causal_skip else 0)
            repops_softmax(a["S"].view(-1, T), causal=True, out=a["P"].view(-1, T))
        if self.causal_skip:
            repops_causal_suffix_flags(a["qkv"], T, hd, Wb, (T * Wb, 0), (nbl, 1), out=self.vflags,
                                       ldf=hd, sF=((T + 1) * hd, 0), offB=(qh + 1) * hd)
        repops_gemm_strided_batched(a["P"], a["qkv"], a["o"], M=T, N=hd, K=T, lda=T, ldb=Wb, ldc=qh * hd,
                                    sA=(qh * T * T, T * T), sB=(T * Wb, 0), sC=(T * qh * hd, hd), batch=(nbl, qh),
                                    offB=(qh + 1) * hd, causal=2 if self.causal_skip else 0, kflags=self.vflags,
                                    ldf=hd, sF=((T + 1) * hd, 0))
        self._gather_blocks(a["o"], a["o_all"], qh * hd)
        HD = c.n_head * hd
        repops_gemm_strided_batched(self._xT(a["o_all"]), w["wo"], a["op"], M=T, N=self.Db, K=HD, lda=T,
                                    ldb=self.Db, ldc=self.Db, sA=(0, 0), sB=(HD * self.Db, 0), sC=(T * self.Db, 0),
                                    batch=(nbl, 1), transA=True)
        self._gather_blocks(a["op"], a["attn"], self.Db)
        repops_add(self.x[l], a["attn"], out=a["h"])

    def _mlp(self, l, a, w):
        c = self.cfg
        T, d, nbl, Fb = c.seq, c.d, self.nbl, self.Fb
        repops_rmsnorm(a["h"], w["mlp_norm"], c.eps, out=a["hn"], rstd=a["rs2"])
        hnT = self._xT(a["hn"])
        for wk, out in (("wg", "g"), ("wu", "u")):
            repops_gemm_strided_batched(hnT, w[wk], a[out], M=T, N=Fb, K=d, lda=T, ldb=Fb, ldc=Fb, sA=(0, 0),
                                        sB=(d * Fb, 0), sC=(T * Fb, 0), batch=(nbl, 1), transA=True)
        repops_swiglu(a["g"], a["u"], out=a["a"])
        self._gather_blocks(a["a"], a["a_all"], Fb)
        repops_gemm_strided_batched(self._xT(a["a_all"]), w["wd"], a["dn"], M=T, N=self.Db, K=c.ffn, lda=T,
                                    ldb=self.Db, ldc=self.Db, sA=(0, 0), sB=(c.ffn * self.Db, 0),
                                    sC=(T * self.Db, 0), batch=(nbl, 1), transA=True)
        self._gather_blocks(a["dn"], a["mlp"], self.Db)
        repops_add(a["h"], a["mlp"], out=self.x[l + 1])

    def _head(self):
        c = self.cfg
        T, d = c.seq, c.d
        repops_rmsnorm(self.x[c.n_layer], self.norm, c.eps, out=self.xf, rstd=self.rsf)
        repops_gemm_strided_batched(self._xT(self.xf), self.wlm, self.logits, M=T, N=self.Vb, K=d, lda=T,
                                    ldb=self.Vb, ldc=self.Vb, sA=(0, 0), sB=(d * self.Vb, 0),
                                    sC=(T * self.Vb, 0), batch=(self.nbl, 1), transA=True)

    # ------------------------------------------------------------------ finalisation / running
    def _finalize(self):
        c = self.cfg
        for i, t in enumerate(self._rep):
            self.tensors[t].slot = i
        per = len(self._blk[0])
        assert all(len(v) == per for v in self._blk.values())
        self.rep_slots, self.blk_slots = len(self._rep), per
        for b in range(c.nb):
            for i, t in enumerate(self._blk[b]):
                self.tensors[t].slot = self.rep_slots + b * per + i
        self.n_slots = self.rep_slots + c.nb * per
        for nd in self.nodes:
            for t in nd.inputs:
                src = self.tensors[t].producer
                if nd.index not in self.nodes[src].dsts:
                    self.nodes[src].dsts.append(nd.index)
        blob, offs, slots, soffs = bytearray(), [0], [], [0]
        for nd in self.nodes:
            keys = sorted(nd.attrs)
            b = bytearray(b"\x4e") + struct.pack("<IHI", nd.index, nd.op, nd.block) + struct.pack("<I", len(keys))
            for k in keys:
                b += struct.pack("<IQ", k, nd.attrs[k])
            b += struct.pack("<I", len(nd.inputs))
            for t in nd.inputs:
                b += struct.pack("<II", self.tensors[t].producer, self.tensors[t].pslot)
            b += struct.pack("<I", len(nd.dsts)) + b"".join(struct.pack("<I", q) for q in nd.dsts)
            b += struct.pack("<I", len(nd.outputs))
            blob += b
            offs.append(len(blob))
            slots += [self.tensors[t].slot for t in nd.inputs + nd.outputs]
            soffs.append(len(slots))
        self.node_blob = np.frombuffer(bytes(blob), np.uint8).copy()
        self.node_offs = np.asarray(offs, np.int64)
        self.node_slots = np.asarray(slots, np.int64)
        self.node_soffs = np.asarray(soffs, np.int64)
        if self.structure_only:
            return
        self.digests = torch.zeros((self.n_slots, 32), dtype=torch.uint8, device=self.dev)
        self.plans = []
        for name, fns, tids in self.phases:
            tids = [t for t in tids if self.tensors[t].view.numel() > 0 or t == -1]
            tids = [t for t in tids if not self.tensors[t].name.startswith("param/")]
            self.plans.append(CommitPlan([self.tensors[t].view for t in tids],
                                         [self.digests[self.tensors[t].slot] for t in tids]) if tids else None)
        self.root_plan = RootPlan(self.node_blob, self.node_offs, self.node_slots, self.node_soffs, self.digests)
        self.root_host = torch.zeros(32, dtype=torch.uint8).pin_memory()
        self.side = torch.cuda.Stream(device=self.dev)
        self.commit_mode = os.environ.get("REPOPS_LLAMA_COMMIT", "side")
        self.commit_bytes = sum(p.nbytes for p in self.plans if p is not None)

    def set_tokens(self, host_tokens=None):
        c = self.cfg
        if host_tokens is None:
            host_tokens = synth.llama_tokens(c.vocab, c.seq, c.seed)
        self.tok.copy_(torch.as_tensor(np.ascontiguousarray(host_tokens, dtype=np.int32)))

    def run(self, commit=True, commit_mode=None):
        """One prefill pass.  commit_mode "side": each phase's commit plan runs on a side
        stream beside the next phases; "inline": on the pass stream right after its phase;
        "end": every plan after the last phase (same digests in every mode)."""
        commit_mode = commit_mode or self.commit_mode
        main = torch.cuda.current_stream()
        side = self.side   # parameter digests were written into the table at load time
        side.wait_stream(main)
        for (name, fns, _), plan in zip(self.phases, self.plans):
            for fn in fns:
                fn()
            if commit and plan is not None:
                if commit_mode == "side":
                    side.wait_stream(main)
                    plan.run(stream=side)
                elif commit_mode == "inline":
                    plan.run(stream=main)
        if commit and commit_mode == "end":
            for plan in self.plans:
                if plan is not None:
                    plan.run(stream=main)
        main.wait_stream(side)

    def device_root(self):
        gather_shard_digests(self.digests, self.rep_slots, self.blk_slots, self.b0, self.nbl, self.world, self.pg)
        self.root_plan.run()
        self.root_host.copy_(self.root_plan.root, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return bytes(self.root_host.numpy())

    def flops(self):
        c = self.cfg
        T, d, hd = c.seq, c.d, c.hd
        lin = 2 * T * d * (c.n_head * hd + 2 * c.n_kv * hd) + 2 * T * c.n_head * hd * d + 3 * 2 * T * d * c.ffn
        attn = 2 * 2 * c.n_head * T * T * hd
        return c.n_layer * (lin + attn) + 2 * T * d * c.vocab
