"""GPT-2 (124M) training step on RepOps with Verde commitments (BASELINE config 3 + 5).

One step = forward + backward + canonical data-parallel gradient combine +
AdamW ("forward pass, backward pass, parameter updates and
an optimizer state update"), every operator a RepOps kernel of librepops.so,
every operator output committed (R-TCOMMIT) and every graph node hashed into
the step's Merkle root (the checkpoint commitment, Fig. 2).

Data parallelism (reading R14): the global batch is S = 8 fixed shards of one
sequence each.  Rank r of G owns shards [r*S/G, (r+1)*S/G).  Per-shard weight
gradients are R-GEMMs with K = the shard's tokens; the shards' gradients are
combined by the balanced tree R-TREE_S (aligned local subtree, NCCL all-gather
of the G partials -- data movement only --, then the top levels on every
rank).  The result is bit-identical for G in {1, 2, 4, 8}.

Node graph (reading R13): the extended computational graph of Fig. 1
(P:367-391), topologically ordered as
  [PARAM_IN x n_params] [for s in 0..S-1: TOKENS_IN, forward nodes, backward nodes]
  [TREE_SUM x n_params] [ADAMW x n_params]
Per-shard nodes are G-independent even though the kernels batch all local
shards into one launch: M-batching of a GEMM and row-batching of a row op are
bits-neutral.  Every node's inputs / outputs are tensors whose digests live
in a device digest table; the host builds the node digests and the step root
with one native call (verde_node_digests_root) after one D2H copy of the table.

Python here only sequences C-ABI calls and owns buffers (torch memory).
"""
from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

import synth

from . import (EPI_BIAS, EPI_SCALE, POST_GELU, POST_GELU_BACKWARD, CommitPlan, repops_add, repops_attention_fwd,
               repops_attention_fwd_supported, repops_attention_dscores, repops_attention_probs,
               repops_attention_probs_supported,
               repops_cross_entropy, repops_embedding,
               repops_embedding_backward, repops_gelu, repops_gelu_backward, repops_gemm,
               repops_gemm_strided_batched, repops_layernorm, repops_layernorm_backward,
               repops_layernorm_backward_params, repops_softmax, repops_softmax_backward, repops_sum_cols_seq,
               repops_adamw, repops_adamw_segments, repops_tree_sum, verde_dirty_chunks)
from ._lib import check, lib
from .dist import P2PTreeCombine, P2PUnavailable, all_gather_rows, dp_tree_combine, dp_tree_combine_sliced, gather_shard_digests, shard_block

# node operator codes (u16)
OP = dict(PARAM_IN=1, TOKENS_IN=2, EMBED=3, LAYERNORM=4, LINEAR=5, ATTN_SCORES=6, SOFTMAX=7, ATTN_PV=8,
          RESIDUAL=9, GELU=10, LM_HEAD=11, CROSS_ENTROPY=12,
          LM_DGRAD=20, LM_WGRAD=21, LN_BWD=22, LN_PARAM_GRAD=23, LINEAR_DGRAD=24, LINEAR_WGRAD=25,
          BIAS_GRAD=26, GELU_BWD=27, ATTN_DP=28, SOFTMAX_BWD=29, ATTN_DQKV=30, EMBED_BWD=31,
          TREE_SUM=40, ADAMW=41, ATTENTION=13, ATTENTION_BWD=32)
# attribute keys
AK = dict(layer=1, eps=2, scale=3, causal=4, lr=5, beta1=6, beta2=7, adam_eps=8, wd=9, step=10, decay=11,
          which=12)


def f32bits(x: float) -> int:
    return int(np.float32(x).view(np.uint32))


@dataclass
class GPT2Config:
    n_layer: int = 12
    d: int = 768
    n_head: int = 12
    ffn: int = 3072
    vocab: int = 50257
    n_pos: int = 1024
    seq: int = 512
    shards: int = 8
    ln_eps: float = 1e-5
    lr: float = 6e-4
    beta1: float = 0.9
    beta2: float = 0.95
    adam_eps: float = 1e-8
    wd: float = 0.1
    seed: int = 0

    @property
    def hd(self):
        return self.d // self.n_head

    @property
    def vocab_ld(self):
        return (self.vocab + 63) // 64 * 64

    @staticmethod
    def tiny():
        return GPT2Config(n_layer=2, d=64, n_head=4, ffn=256, vocab=512, n_pos=64, seq=32, shards=8)


@dataclass
class TensorRef:
    name: str
    view: torch.Tensor
    slot: int               # digest-table slot
    producer: int = -1      # node index
    pslot: int = 0          # output position within the producer


@dataclass
class NodeRec:
    index: int
    op: int
    shard: int              # 0xFFFFFFFF for replicated nodes
    attrs: dict
    inputs: list            # TensorRef indices
    outputs: list
    name: str = ""
    label: str | None = None  # launch label of the op that produces the outputs
    dsts: list = field(default_factory=list)


REPLICATED = 0xFFFFFFFF


class GPT2Step:
    """Static program of one training step for the shards owned by this rank."""

    def __init__(self, cfg: GPT2Config, rank: int = 0, world: int = 1, device="cuda", pg=None,
                 structure_only=False, combine: str = "sliced", p2p_sync: str = "device", attn_nodes: str = "operator",
                 zero1: bool = False):
        """structure_only: build the node graph / slot layout on the 'meta' device
        (no memory, no kernels) -- used by the CPU tests of the host logic."""
        assert cfg.shards % world == 0
        self.cfg, self.rank, self.world, self.pg = cfg, rank, world, pg
        # graph granularity of attention (reading R29): "operator" = one ATTENTION node
        # (qkv -> att) and one ATTENTION_BWD node (qkv, datt -> dqkv), as PyTorch's
        # scaled_dot_product_attention and its backward are single graph nodes; the scores,
        # probabilities and their gradients are operator-internal (recomputable from qkv)
        # and not committed.  "primitive" = round 1's per-primitive nodes (scores, softmax,
        # PV, dP, softmax backward, dQKV), each output committed.
        if attn_nodes not in ("operator", "primitive"):
            raise ValueError(f"unknown attn_nodes {attn_nodes!r}")
        self.attn_op = attn_nodes == "operator"
        self.causal_skip = True   # f4 / R31: exact causal tile skipping where the scores are scratch
        # ZeRO-1 (f1): the optimizer state is partitioned by whole parameter tensors -- rank
        # owner(name) alone keeps m / v of `name`, runs its AdamW, commits its PARAM_IN /
        # TREE_SUM / ADAMW outputs and broadcasts the updated parameter; the digests of the
        # replicated nodes are exchanged by owner, so the step root equals the replicated
        # run's.  Gradients stay fully combined on every rank (stage 1, not 2).
        self.zero1 = zero1
        self.structure_only = structure_only
        self.dev = torch.device("meta" if structure_only else device)
        self.s0, self.S_loc = shard_block(rank, world, cfg.shards)
        self._fault = None
        self.keep_committed = False  # stash tensors an in-place writer overwrites (for disputes)
        # R-TREE_S transport at G > 1 (same bits for all): "sliced" = NCCL all-to-all +
        # all-gather; "gather" = all-gather of partials; "p2p" = one fused kernel per rank
        # over NVLink peer memory (dist.P2PTreeCombine)
        if combine not in ("sliced", "gather", "p2p"):
            raise ValueError(f"unknown combine {combine!r}")
        self.combine, self.p2p_sync, self.p2p = combine, p2p_sync, None
        # f1: with the peer-memory combine each layer's gradient bucket is combined on a
        # comm stream right after that layer's backward (overlapping the next layers'
        # backward); the embedding / final-LN buckets and the "done" barrier follow the
        # embedding backward.  Same bits as one whole-gradient combine (elementwise).
        self.bucketed = True
        self.sliced_combine = combine == "sliced"
        # f4: scores + causal softmax + PV as one kernel (same bits).  Off by default: at the
        # GPT-2 shape the fused kernel (1 CTA / SM, 213 KB of shared memory) measured 307 us
        # per layer vs 253 us for the three tuned launches (tools/attn_fused_bench.py)
        self.fused_attention = False
        # f4 (round 2): scores + causal softmax as one kernel (repops_attention_probs: the scores
        # never leave shared memory, P is written for the PV R-GEMM and the backward), then the
        # PV R-GEMM; same bits as the three launches.  Needs the scores to be operator scratch
        # (R29); fault-injection runs keep the per-op launches
        self.attn_probs = os.environ.get("REPOPS_ATTN_PROBS", "1") == "1"   # (A/B switch for tools)
        # incremental commit of the tied embedding gradient (see the plan construction)
        self.delta_commit = os.environ.get("REPOPS_DELTA_COMMIT", "1") == "1"
        self._inject_active = False
        # its backward twin (repops_attention_dscores: dP in shared memory + softmax backward,
        # same dS bits) measured slower than the dP R-GEMM + softmax_bwd launches (181 vs
        # 161 us per layer, tools/attn_fused_bench.py): off by default
        self.attn_dscores = os.environ.get("REPOPS_ATTN_DSCORES", "0") == "1"
        # GELU / GELU-backward fused into the FC / FC2-dgrad GEMM epilogues (repops_gemm_post):
        # same bits, but measured slower in the step (80.05 -> 80.43 ms; the tanh chain in the
        # epilogue of a 2-3 CTA/SM GEMM hides latency worse than the standalone HBM-bound
        # kernels), so off by default
        self.fuse_gelu = False
        # backward: weight / bias / LN-parameter gradients on an aux stream beside the dgrads
        self.aux_wgrad = not structure_only
        # the aux stream carries critical-path work (joined every layer): high priority, so
        # the block scheduler prefers it over the commit side stream's SHA-256 CTAs
        self.aux = None if structure_only else torch.cuda.Stream(device=device, priority=-1)
        self.attn_probs_ok = (not structure_only) and repops_attention_probs_supported(cfg.seq, cfg.hd)
        self.fused_attention_ok = (not structure_only) and repops_attention_fwd_supported(cfg.seq,
                                                                                            cfg.d // cfg.n_head)
        self.stash = {}
        self.step_no = 0
        # PARAM_IN digest reuse: the step's PARAM_IN tensors (param, m, v) are the previous
        # step's AdamW outputs, byte for byte, when nothing else wrote them in between; their
        # committed digests are then copied instead of re-hashed (1.5 GB of SHA-256 per
        # GPT-2 step).  Anything that writes params / m / v from outside the step must call
        # state_changed() (TrainingRun checkpoint loads, tampering in the dispute tests).
        self.reuse_state_digests = True
        self._state_digests_valid = False
        c = cfg
        self.M = self.S_loc * c.seq
        self._init_params()
        self._alloc()
        self._build_program()

    # ------------------------------------------------------------------ parameters
    def _init_params(self):
        c = self.cfg
        self.specs = synth.gpt2_param_specs(c.n_layer, c.d, c.ffn, c.vocab, c.n_pos)
        self.off, off = {}, 0
        for name, shape, kind in self.specs:
            n = int(np.prod(shape))
            self.off[name] = (off, shape, kind)
            off += n
        self.P = off
        # ZeRO-1 ownership: largest tensors first, each to the least-loaded rank (ties -> lower
        # rank); deterministic, the same on every rank
        self.owner = {name: 0 for name, _, _ in self.specs}
        if self.zero1 and self.world > 1:
            load = [0] * self.world
            for name, shape, _ in sorted(self.specs, key=lambda t: (-int(np.prod(t[1])), t[0])):
                r = min(range(self.world), key=lambda q: (load[q], q))
                self.owner[name] = r
                load[r] += int(np.prod(shape))
        self.owned = [name for name, _, _ in self.specs if self.owner[name] == self.rank or not self.zero1]
        self.moff, mo = {}, 0  # offsets of the owned tensors in the (compact) m / v buffers
        for name in self.owned:
            self.moff[name] = mo
            mo += int(np.prod(self.off[name][1]))
        self.P_own = mo
        if self.structure_only:
            self.params = torch.empty(self.P, device=self.dev)
            self.m = torch.empty(self.P, device=self.dev)
            self.v = torch.empty(self.P, device=self.dev)
            return
        host = np.empty(self.P, np.float32)
        for name, shape, kind in self.specs:
            o, _, _ = self.off[name]
            host[o:o + int(np.prod(shape))] = synth.gpt2_param(name, shape, kind, c.seed).ravel()
        self.params = torch.from_numpy(host).to(self.dev)
        self.m = torch.zeros(self.P_own if self.zero1 else self.P, device=self.dev)
        self.v = torch.zeros(self.P_own if self.zero1 else self.P, device=self.dev)

    def pview(self, buf, name):
        o, shape, _ = self.off[name]
        return buf[o:o + int(np.prod(shape))].view(*shape)

    def mview(self, buf, name):
        """view of `name` in the optimizer-state buffer m / v (ZeRO-1: compact, owned tensors
        only; an empty placeholder for the others)"""
        if not self.zero1:
            return self.pview(buf, name)
        if name not in self.moff:
            return torch.empty(0, device=self.dev)
        o, shape = self.moff[name], self.off[name][1]
        return buf[o:o + int(np.prod(shape))].view(*shape)

    # ------------------------------------------------------------------ buffers
    def _alloc(self):
        c, M, dev = self.cfg, self.M, self.dev
        E = lambda *s: torch.empty(*s, dtype=torch.float32, device=dev)  # noqa: E731
        L, d, T, H = c.n_layer, c.d, c.seq, c.n_head
        self.tok = torch.empty((self.S_loc, T + 1), dtype=torch.int32, device=dev)
        self.x = [E(M, d) for _ in range(L + 1)]
        a = self.act = []
        for _ in range(L):
            a.append(dict(ln1=E(M, d), mu1=E(M), rs1=E(M), qkv=E(M, 3 * d), S=E(self.S_loc * H * T, T),
                          P=E(self.S_loc * H * T, T), att=E(M, d), proj=E(M, d), xmid=E(M, d), ln2=E(M, d),
                          mu2=E(M), rs2=E(M), fc=E(M, c.ffn), gelu=E(M, c.ffn), fc2=E(M, d)))
        self.lnf, self.muf, self.rsf = E(M, d), E(M), E(M)
        self.logits = torch.zeros(M, c.vocab_ld, device=dev)   # padding columns stay 0 (committed bytes)
        self.dlogits = torch.zeros(M, c.vocab_ld, device=dev)
        self.loss_tok = E(M)
        self.dlnf = E(M, d)
        g = self.grad_act = []
        for _ in range(L):
            g.append(dict(dgelu=E(M, c.ffn), dfc=E(M, c.ffn), dln2=E(M, d), dxmid=E(M, d), datt=E(M, d),
                          dP=E(self.S_loc * H * T, T), dS=E(self.S_loc * H * T, T), dqkv=E(M, 3 * d),
                          dln1=E(M, d)))
        self.dx = [E(M, d) for _ in range(L + 1)]  # dx[l] = gradient w.r.t. x[l]
        self.glocal = torch.zeros(self.S_loc, self.P, device=dev)  # per-shard gradients (rows)
        self.combine_fallback = None
        if self.combine == "p2p" and self.world > 1 and not self.structure_only:
            try:
                self.p2p = P2PTreeCombine(self.P, self.rank, self.world, self.pg, sync=self.p2p_sync)
            except P2PUnavailable as e:
                # CUDA IPC peer mapping failed on some rank (all ranks agreed): the NCCL
                # transport of the same R-TREE_S (data movement only, same bits)
                self.p2p, self.combine, self.sliced_combine, self.combine_fallback = None, "sliced", True, str(e)
        if self.p2p is not None:
            self.grad = self.p2p.grad   # IPC buffer every rank's combine kernel writes its slice into
        else:
            self.grad = E(self.P)
        self.shard_loss = E(self.S_loc)
        # transposed copies of the 2-D weights (refreshed every step, data movement
        # only): every dgrad GEMM and the LM head then read an n-contiguous B
        self.wT = {name: E(*shape[::-1]) for name, shape, kind in self.specs
                   if len(shape) == 2 and name != "wpe"}
        # wte^T with vocab_ld columns; the padding columns stay +0, so the LM head
        # can run over all vocab_ld columns with full tiles and write exactly the
        # +0 padding the committed logits already hold (acc = +0 + sum of +-0 = +0)
        self.wteT_pad = torch.zeros(c.d, c.vocab_ld, device=dev)
        self.wT["wte"] = self.wteT_pad[:, :c.vocab]
        # scratch for X^T: every activation-side GEMM operand is transposed first so
        # the GEMM runs TN (A^T tiles are 10-40% faster than row-major A on sm_100a,
        # DESIGN.md §5); data movement only, consumed by the very next GEMM
        self.xT = E(max(c.vocab, c.ffn, 3 * d) * M)

    def _gemm_tn_post(self, X, B, post, out2, Xpost=None, **kw):
        """_gemm_tn with the elementwise consumer fused into the GEMM epilogue
        (repops_gemm_post: C2 = GELU(C) or GELU-backward at Xpost with dy = C)."""
        from . import repops_gemm_post, repops_transpose
        rows, cols = X.shape
        xt = self.xT[:rows * cols].view(cols, rows)
        repops_transpose(X, out=xt)
        return repops_gemm_post(xt, B, post, out2, X=Xpost, transA=True, **kw)

    def _gemm_tn(self, X, B, **kw):
        """repops_gemm(X, B, **kw) computed as (X^T)^T B: X^T is written to the
        scratch first (bit-exact copy), then the GEMM reads it as A^T.  The K
        order of every output element is unchanged (R2)."""
        from . import repops_transpose
        rows, cols = X.shape
        xt = self.xT[:rows * cols].view(cols, rows)
        repops_transpose(X, out=xt)
        return repops_gemm(xt, B, transA=True, **kw)

    # ------------------------------------------------------------------ program construction
    def _build_program(self):
        c = self.cfg
        self.tensors: list[TensorRef] = []
        self.nodes: list[NodeRec] = []
        self.phases = []          # list of (name, [launch closures], [tensor ids to commit])
        self._cur = None
        # digest slots: replicated region first, then S shard regions of equal size
        self.rep_slots = 0
        self.shard_slots = 0

        # pass 1 (count shard slots) uses a dry build of one shard's tensor list;
        # simpler: assign slots lazily per region, then fix the shard stride afterwards.
        self._rep_ids, self._shard_ids = [], {s: [] for s in range(c.shards)}

        def T_(name, view, shard):
            tid = len(self.tensors)
            self.tensors.append(TensorRef(name, view, -1))
            (self._rep_ids if shard == REPLICATED else self._shard_ids[shard]).append(tid)
            return tid

        self._T = T_
        self._deferred = []
        self._label_phase, self._tensor_phase = {}, {}
        # ---- replicated input nodes: parameters with their optimizer state
        self.phase("inputs")
        if not self.structure_only:
            def transposes():
                from . import repops_transpose
                for name, t in self.wT.items():
                    repops_transpose(self.pview(self.params, name), out=t)
            self.launch(transposes)
        self.param_in = {}
        self.param_in_node, self.adamw_node = {}, {}
        for name, shape, kind in self.specs:
            ids = [T_(f"param/{name}", self.pview(self.params, name), REPLICATED),
                   T_(f"m/{name}", self.mview(self.m, name), REPLICATED),
                   T_(f"v/{name}", self.mview(self.v, name), REPLICATED)]
            self.node(OP["PARAM_IN"], REPLICATED, {}, [], ids, f"in/{name}")
            self.param_in[name] = ids
            self.param_in_node[name] = len(self.nodes) - 1
        # ---- per shard (global ids); only local shards get launches, but every
        # shard's structure is recorded so the node list is the global one
        self.shard_nodes = {}
        for s in range(c.shards):
            self._build_shard(s)
        # ---- tree + AdamW (replicated)
        self._build_tree_and_adam()
        self._finalize()

    def phase(self, name):
        self._cur = (name, [], [])
        self.phases.append(self._cur)

    def launch(self, fn):
        self._cur[1].append(fn)

    def _aux(self, fn):
        """Run fn's launches on the aux stream, ordered after everything enqueued so far on
        the current stream (its inputs); inline when disabled or under fault injection
        (so an injected fault lands exactly where the per-op order puts it)."""
        if not self.aux_wgrad or self._fault is not None:
            fn()
            return
        main = torch.cuda.current_stream()
        self.aux.wait_stream(main)
        with torch.cuda.stream(self.aux):
            fn()
        self._aux_pending = True

    def _aux_join(self):
        if getattr(self, "_aux_pending", False):
            torch.cuda.current_stream().wait_stream(self.aux)
            self._aux_pending = False

    def _hook(self, label):
        """Fault-injection point after the launch of op `label` (config 5 dispute demo)."""
        if self._fault is not None and self._fault[0] == label:
            self._fault[1]()

    def node(self, op, shard, attrs, inputs, outputs, name="", defer=False, label=None):
        idx = len(self.nodes)
        if label is None and shard != REPLICATED:
            label = name.split("/", 1)[1]  # "s3/h1/qkv" -> "h1/qkv" (the batched launch's hook label)
        self.nodes.append(NodeRec(idx, op, shard, attrs, inputs, outputs, name, label=label))
        # phase in which the producing launch is enqueued: the first local shard's
        # phase for batched per-shard launches, else the current phase
        ph = len(self.phases) - 1
        if shard != REPLICATED and self._is_local(shard):
            if shard == self.s0:
                self._label_phase[label] = ph
            else:
                ph = self._label_phase.get(label, ph)
        self._tensor_phase.update({t: ph for t in outputs})
        if defer:
            self._tensor_phase.update({t: None for t in outputs})
        for q, t in enumerate(outputs):
            self.tensors[t].producer = idx
            self.tensors[t].pslot = q
            if shard == REPLICATED or self._is_local(shard):
                (self._deferred if defer else self._cur[2]).append(t)
        return idx

    def _is_local(self, s):
        return self.s0 <= s < self.s0 + self.S_loc

    # per-shard slab helpers (views only exist for local shards)
    def _slab(self, buf, s, rows_per_shard):
        sl = s - self.s0
        return buf[sl * rows_per_shard:(sl + 1) * rows_per_shard]

    def _build_shard(self, s):
        c = self.cfg
        L, d, T, H, hd = c.n_layer, c.d, c.seq, c.n_head, c.hd
        local = self._is_local(s)
        first_local = local and s == self.s0
        T_ = self._T
        P_ = self.param_in
        dummy = torch.empty(0, device=self.dev)

        def V(buf, rows):  # view of this shard's slab (or an empty placeholder for remote shards)
            return self._slab(buf, s, rows) if local else dummy

        def attrs(**kw):
            out = {}
            for k, v in kw.items():
                out[AK[k]] = f32bits(v) if isinstance(v, float) else int(v)
            return out

        Mloc, S_loc = self.M, self.S_loc
        sl = s - self.s0
        # ---------------- forward
        self.phase(f"s{s}/tokens")
        t_tok = T_(f"s{s}/tokens", self.tok[sl] if local else dummy, s)
        self.node(OP["TOKENS_IN"], s, {}, [], [t_tok], f"s{s}/tokens")

        if first_local:
            self.launch(lambda: repops_embedding(self.tok_in_flat, self.pview(self.params, "wte"),
                                                 self.pview(self.params, "wpe"), c.seq, out=self.x[0]))
        t_x = T_(f"s{s}/x0", V(self.x[0], T), s)
        self.node(OP["EMBED"], s, {}, [t_tok, P_["wte"][0], P_["wpe"][0]], [t_x], f"s{s}/embed")

        for l in range(L):
            a = self.act[l]
            p = f"h{l}."
            W = lambda n, p=p: self.pview(self.params, p + n)  # noqa: E731  (bind this layer's prefix)
            if first_local:
                def fwd(l=l, a=a, W=W):
                    repops_layernorm(self.x[l], W("ln1.g"), W("ln1.b"), c.ln_eps, out=a["ln1"], mean=a["mu1"],
                                     rstd=a["rs1"])
                    self._hook(f"h{l}/ln1")
                    self._gemm_tn(a["ln1"], W("attn.w"), epi=EPI_BIAS, bias=W("attn.b"), out=a["qkv"])
                    self._hook(f"h{l}/qkv")
                    if self.fused_attention and self.fused_attention_ok and self._fault is None:
                        # one fused kernel writes the same S, P and att bits (f4; no HBM round
                        # trip of S / P between launches); fault-injection runs keep the
                        # per-op launches so a flipped S bit propagates as in the graph
                        # with attention as one operator (R29) the scores are scratch and never
                        # leave shared memory: the kernel computes the key chunks its rows read
                        # and closes the PV fold from V's suffix flags (R31); P stays for the backward
                        repops_attention_fwd(a["qkv"], T, hd, 3 * d, (T * 3 * d, hd), 0, d, 2 * d, (S_loc, H),
                                             a["att"], d, (T * d, hd), S=None if self.attn_op else a["S"],
                                             P=a["P"], sp=(H * T * T, T * T),
                                             scale=1.0 / np.sqrt(hd), causal=True)
                    elif self.attn_op and self.attn_probs and self.attn_probs_ok and self._fault is None:
                        repops_attention_probs(a["qkv"], T, hd, 3 * d, (T * 3 * d, hd), 0, d, (S_loc, H), a["P"],
                                               (H * T * T, T * T), scale=1.0 / np.sqrt(hd), causal=True)
                        repops_gemm_strided_batched(a["P"], a["qkv"], a["att"], M=T, N=hd, K=T, lda=T, ldb=3 * d,
                                                    ldc=d, sA=(H * T * T, T * T), sB=(T * 3 * d, hd),
                                                    sC=(T * d, hd), batch=(S_loc, H), offB=2 * d)
                    else:
                        # scores S = (Q K^T) * 1/sqrt(hd), batched over (local shard, head)
                        # with attention as one operator (R29) the scores are internal scratch: the
                        # tiles above the diagonal, which the causal softmax never reads, are not
                        # computed (R31; tools/causal_bench.py: 106 -> 72 us per layer)
                        skip = self.attn_op and self.causal_skip
                        repops_gemm_strided_batched(a["qkv"], a["qkv"], a["S"], M=T, N=T, K=hd, lda=3 * d,
                                                    ldb=3 * d, ldc=T, sA=(T * 3 * d, hd), sB=(T * 3 * d, hd),
                                                    sC=(H * T * T, T * T), batch=(S_loc, H), transB=True,
                                                    epi=EPI_SCALE, scale=1.0 / np.sqrt(hd), offB=d,
                                                    causal=1 if skip else 0)
                        self._hook(f"h{l}/scores")
                        repops_softmax(a["S"], causal=True, out=a["P"])
                        self._hook(f"h{l}/softmax")
                        # the causal PV (mode 2) does not pay at T = 512: its 384 CTAs are one wave,
                        # so the full-K row tiles set the time (tools/causal_bench.py: 83.5 vs 82.8
                        # us, plus 13 us of suffix flags) -- the full PV runs here
                        repops_gemm_strided_batched(a["P"], a["qkv"], a["att"], M=T, N=hd, K=T, lda=T, ldb=3 * d,
                                                    ldc=d, sA=(H * T * T, T * T), sB=(T * 3 * d, hd),
                                                    sC=(T * d, hd), batch=(S_loc, H), offB=2 * d)
                        self._hook(f"h{l}/pv")
                    self._gemm_tn(a["att"], W("proj.w"), epi=EPI_BIAS, bias=W("proj.b"), out=a["proj"])
                    self._hook(f"h{l}/proj")
                    repops_add(self.x[l], a["proj"], out=a["xmid"])
                    self._hook(f"h{l}/res1")
                    repops_layernorm(a["xmid"], W("ln2.g"), W("ln2.b"), c.ln_eps, out=a["ln2"], mean=a["mu2"],
                                     rstd=a["rs2"])
                    self._hook(f"h{l}/ln2")
                    if self._fault is None and self.fuse_gelu:  # GELU fused into the FC GEMM's epilogue
                        self._gemm_tn_post(a["ln2"], W("fc.w"), POST_GELU, a["gelu"], epi=EPI_BIAS, bias=W("fc.b"),
                                           out=a["fc"])
                    else:                    # fault injection: per-op launches and hooks
                        self._gemm_tn(a["ln2"], W("fc.w"), epi=EPI_BIAS, bias=W("fc.b"), out=a["fc"])
                        self._hook(f"h{l}/fc")
                        repops_gelu(a["fc"], out=a["gelu"])
                        self._hook(f"h{l}/gelu")
                    self._gemm_tn(a["gelu"], W("fc2.w"), epi=EPI_BIAS, bias=W("fc2.b"), out=a["fc2"])
                    self._hook(f"h{l}/fc2")
                    repops_add(a["xmid"], a["fc2"], out=self.x[l + 1])
                    self._hook(f"h{l}/res2")
                self.launch(fwd)
            pre = f"s{s}/h{l}/"
            t_ln1 = T_(pre + "ln1", V(a["ln1"], T), s)
            t_mu1 = T_(pre + "mu1", V(a["mu1"], T), s)
            t_rs1 = T_(pre + "rs1", V(a["rs1"], T), s)
            self.node(OP["LAYERNORM"], s, attrs(layer=l, eps=c.ln_eps, which=1),
                      [t_x, P_[p + "ln1.g"][0], P_[p + "ln1.b"][0]], [t_ln1, t_mu1, t_rs1], pre + "ln1")
            t_qkv = T_(pre + "qkv", V(a["qkv"], T), s)
            self.node(OP["LINEAR"], s, attrs(layer=l, which=1), [t_ln1, P_[p + "attn.w"][0], P_[p + "attn.b"][0]],
                      [t_qkv], pre + "qkv")
            if self.attn_op:
                t_P = None
                t_att = T_(pre + "att", V(a["att"], T), s)
                self.node(OP["ATTENTION"], s, attrs(layer=l, scale=float(1.0 / np.sqrt(hd)), causal=1), [t_qkv],
                          [t_att], pre + "attention", label=f"h{l}/pv")
            else:
                t_S = T_(pre + "scores", V(a["S"], H * T), s)
                self.node(OP["ATTN_SCORES"], s, attrs(layer=l, scale=float(1.0 / np.sqrt(hd))), [t_qkv], [t_S],
                          pre + "scores")
                t_P = T_(pre + "probs", V(a["P"], H * T), s)
                self.node(OP["SOFTMAX"], s, attrs(layer=l, causal=1), [t_S], [t_P], pre + "softmax")
                t_att = T_(pre + "att", V(a["att"], T), s)
                self.node(OP["ATTN_PV"], s, attrs(layer=l), [t_P, t_qkv], [t_att], pre + "pv")
            t_proj = T_(pre + "proj", V(a["proj"], T), s)
            self.node(OP["LINEAR"], s, attrs(layer=l, which=2), [t_att, P_[p + "proj.w"][0], P_[p + "proj.b"][0]],
                      [t_proj], pre + "proj")
            t_xmid = T_(pre + "xmid", V(a["xmid"], T), s)
            self.node(OP["RESIDUAL"], s, attrs(layer=l, which=1), [t_x, t_proj], [t_xmid], pre + "res1")
            t_ln2 = T_(pre + "ln2", V(a["ln2"], T), s)
            t_mu2 = T_(pre + "mu2", V(a["mu2"], T), s)
            t_rs2 = T_(pre + "rs2", V(a["rs2"], T), s)
            self.node(OP["LAYERNORM"], s, attrs(layer=l, eps=c.ln_eps, which=2),
                      [t_xmid, P_[p + "ln2.g"][0], P_[p + "ln2.b"][0]], [t_ln2, t_mu2, t_rs2], pre + "ln2")
            t_fc = T_(pre + "fc", V(a["fc"], T), s)
            self.node(OP["LINEAR"], s, attrs(layer=l, which=3), [t_ln2, P_[p + "fc.w"][0], P_[p + "fc.b"][0]],
                      [t_fc], pre + "fc")
            t_gelu = T_(pre + "gelu", V(a["gelu"], T), s)
            self.node(OP["GELU"], s, attrs(layer=l), [t_fc], [t_gelu], pre + "gelu")
            t_fc2 = T_(pre + "fc2", V(a["fc2"], T), s)
            self.node(OP["LINEAR"], s, attrs(layer=l, which=4), [t_gelu, P_[p + "fc2.w"][0], P_[p + "fc2.b"][0]],
                      [t_fc2], pre + "fc2")
            t_xn = T_(f"s{s}/x{l + 1}", V(self.x[l + 1], T), s)
            self.node(OP["RESIDUAL"], s, attrs(layer=l, which=2), [t_xmid, t_fc2], [t_xn], pre + "res2")
            a["_ids"] = a.get("_ids", {})
            a["_ids"][s] = dict(ln1=t_ln1, mu1=t_mu1, rs1=t_rs1, qkv=t_qkv, P=t_P, att=t_att, xmid=t_xmid,
                                ln2=t_ln2, mu2=t_mu2, rs2=t_rs2, fc=t_fc, gelu=t_gelu, x=t_x)
            t_x = t_xn
            self.phase(f"s{s}/fwd{l + 1}")
        # ---------------- head
        if first_local:
            def head():
                repops_layernorm(self.x[L], self.pview(self.params, "lnf.g"), self.pview(self.params, "lnf.b"),
                                 c.ln_eps, out=self.lnf, mean=self.muf, rstd=self.rsf)
                self._hook("head/lnf")
                wte = self.pview(self.params, "wte")
                self._gemm_tn(self.lnf, self.wteT_pad, out=self.logits)
                self._hook("head/lm_head")
                repops_cross_entropy(self.logits, self.targets_flat, scale=1.0 / (c.shards * c.seq),
                                     loss=self.loss_tok, dlogits=self.dlogits, V=c.vocab)
                self._hook("head/ce")
            self.launch(head)
        pre = f"s{s}/head/"
        t_lnf = T_(pre + "lnf", V(self.lnf, T), s)
        t_muf = T_(pre + "muf", V(self.muf, T), s)
        t_rsf = T_(pre + "rsf", V(self.rsf, T), s)
        self.node(OP["LAYERNORM"], s, attrs(layer=L, eps=c.ln_eps, which=3),
                  [t_x, P_["lnf.g"][0], P_["lnf.b"][0]], [t_lnf, t_muf, t_rsf], pre + "lnf")
        t_logits = T_(pre + "logits", V(self.logits, T), s)
        self.node(OP["LM_HEAD"], s, {}, [t_lnf, P_["wte"][0]], [t_logits], pre + "lm_head")
        t_loss = T_(pre + "loss", V(self.loss_tok, T), s)
        t_dlog = T_(pre + "dlogits", V(self.dlogits, T), s)
        self.node(OP["CROSS_ENTROPY"], s, attrs(scale=float(1.0 / (c.shards * c.seq))), [t_logits, t_tok],
                  [t_loss, t_dlog], pre + "ce")
        # ---------------- backward: head
        self.phase(f"s{s}/bwd_head")
        gl = self.glocal
        G_ = lambda n: self._gslice(s, n)  # noqa: E731  this shard's gradient slice of parameter n
        if first_local:
            def head_bwd():
                wte = self.pview(self.params, "wte")
                o = self.off["wte"][0]

                def w_lm():  # aux stream, beside the LM dgrad (N = 768: wave-quantised)
                    repops_gemm_strided_batched(self.dlogits, self.lnf, gl, M=c.vocab, N=d, K=T, lda=c.vocab_ld,
                                                ldb=d, ldc=d, sA=(T * c.vocab_ld, 0), sB=(T * d, 0),
                                                sC=(self.P, 0), batch=(S_loc, 1), transA=True, offC=o)
                    self._hook("head/lm_wgrad")
                self._aux(w_lm)
                self._gemm_tn(self.dlogits[:, :c.vocab], wte, out=self.dlnf)
                self._hook("head/lm_dgrad")
                repops_layernorm_backward(self.dlnf, self.x[L], self.pview(self.params, "lnf.g"), self.muf, self.rsf,
                                          out=self.dx[L])
                self._hook("head/lnf_bwd")
                repops_layernorm_backward_params(self.dlnf, self.x[L], self.muf, self.rsf, nseg=S_loc,
                                                 dgamma=gl[:, self.off["lnf.g"][0]:],
                                                 dbeta=gl[:, self.off["lnf.b"][0]:], ldo=self.P)
                self._hook("head/lnf_params")
                self._aux_join()
            self.launch(head_bwd)
        t_dlnf = T_(pre + "dlnf", V(self.dlnf, T), s)
        self.node(OP["LM_DGRAD"], s, {}, [t_dlog, P_["wte"][0]], [t_dlnf], pre + "lm_dgrad")
        t_gwte_lm = T_(f"s{s}/grad/wte_lm", G_("wte"), s)
        self.node(OP["LM_WGRAD"], s, {}, [t_dlog, t_lnf], [t_gwte_lm], pre + "lm_wgrad")
        t_dx = T_(f"s{s}/dx{L}", V(self.dx[L], T), s)
        self.node(OP["LN_BWD"], s, attrs(layer=L, which=3), [t_dlnf, t_x, P_["lnf.g"][0], t_muf, t_rsf], [t_dx],
                  pre + "lnf_bwd")
        self.final_grad = getattr(self, "final_grad", {})
        fg = self.final_grad.setdefault(s, {})
        fg["lnf.g"] = T_(f"s{s}/grad/lnf.g", G_("lnf.g"), s)
        fg["lnf.b"] = T_(f"s{s}/grad/lnf.b", G_("lnf.b"), s)
        self.node(OP["LN_PARAM_GRAD"], s, attrs(layer=L, which=3), [t_dlnf, t_x, t_muf, t_rsf],
                  [fg["lnf.g"], fg["lnf.b"]], pre + "lnf_params")
        # ---------------- backward: layers
        for l in reversed(range(L)):
            a, g = self.act[l], self.grad_act[l]
            ids = a["_ids"][s]
            p = f"h{l}."
            W = lambda n, p=p: self.pview(self.params, p + n)  # noqa: E731
            self.phase(f"s{s}/bwd{l}")
            if first_local:
                def bwd(l=l, a=a, g=g, W=W, p=p):
                    dout = self.dx[l + 1]
                    o = lambda n: self.off[p + n][0]  # noqa: E731
                    # weight / bias / LN-parameter gradients depend only on this layer's
                    # activations and output gradients: they run on the aux stream beside
                    # the dgrad chain (filling its wave-quantised GEMMs' idle SM slots)

                    def w_fc2():
                        repops_gemm_strided_batched(a["gelu"], dout, gl, M=c.ffn, N=d, K=T, lda=c.ffn, ldb=d,
                                                    ldc=d, sA=(T * c.ffn, 0), sB=(T * d, 0), sC=(self.P, 0),
                                                    batch=(S_loc, 1), transA=True, offC=o("fc2.w"))
                        self._hook(f"h{l}/fc2_wgrad")
                        repops_sum_cols_seq(dout, nseg=S_loc, out=gl[:, o("fc2.b"):], ldo=self.P)
                        self._hook(f"h{l}/fc2_bgrad")

                    def w_fc():
                        repops_gemm_strided_batched(a["ln2"], g["dfc"], gl, M=d, N=c.ffn, K=T, lda=d, ldb=c.ffn,
                                                    ldc=c.ffn, sA=(T * d, 0), sB=(T * c.ffn, 0), sC=(self.P, 0),
                                                    batch=(S_loc, 1), transA=True, offC=o("fc.w"))
                        self._hook(f"h{l}/fc_wgrad")
                        repops_sum_cols_seq(g["dfc"], nseg=S_loc, out=gl[:, o("fc.b"):], ldo=self.P)
                        self._hook(f"h{l}/fc_bgrad")

                    def w_ln2():
                        repops_layernorm_backward_params(g["dln2"], a["xmid"], a["mu2"], a["rs2"], nseg=S_loc,
                                                         dgamma=gl[:, o("ln2.g"):], dbeta=gl[:, o("ln2.b"):],
                                                         ldo=self.P)
                        self._hook(f"h{l}/ln2_params")

                    def w_proj():
                        repops_gemm_strided_batched(a["att"], g["dxmid"], gl, M=d, N=d, K=T, lda=d, ldb=d, ldc=d,
                                                    sA=(T * d, 0), sB=(T * d, 0), sC=(self.P, 0), batch=(S_loc, 1),
                                                    transA=True, offC=o("proj.w"))
                        self._hook(f"h{l}/proj_wgrad")
                        repops_sum_cols_seq(g["dxmid"], nseg=S_loc, out=gl[:, o("proj.b"):], ldo=self.P)
                        self._hook(f"h{l}/proj_bgrad")

                    def w_qkv():
                        repops_gemm_strided_batched(a["ln1"], g["dqkv"], gl, M=d, N=3 * d, K=T, lda=d, ldb=3 * d,
                                                    ldc=3 * d, sA=(T * d, 0), sB=(T * 3 * d, 0), sC=(self.P, 0),
                                                    batch=(S_loc, 1), transA=True, offC=o("attn.w"))
                        self._hook(f"h{l}/qkv_wgrad")
                        repops_sum_cols_seq(g["dqkv"], nseg=S_loc, out=gl[:, o("attn.b"):], ldo=self.P)
                        self._hook(f"h{l}/qkv_bgrad")

                    def w_ln1():
                        repops_layernorm_backward_params(g["dln1"], self.x[l], a["mu1"], a["rs1"], nseg=S_loc,
                                                         dgamma=gl[:, o("ln1.g"):], dbeta=gl[:, o("ln1.b"):],
                                                         ldo=self.P)
                        self._hook(f"h{l}/ln1_params")

                    # FC2
                    if self._fault is None and self.fuse_gelu:  # GELU backward fused into the FC2 dgrad
                        self._gemm_tn_post(dout, self.wT[p + "fc2.w"], POST_GELU_BACKWARD, g["dfc"], Xpost=a["fc"],
                                           out=g["dgelu"])
                        self._aux(w_fc2)
                    else:
                        self._gemm_tn(dout, self.wT[p + "fc2.w"], out=g["dgelu"])
                        self._hook(f"h{l}/fc2_dgrad")
                        self._aux(w_fc2)
                        repops_gelu_backward(a["fc"], g["dgelu"], out=g["dfc"])
                        self._hook(f"h{l}/gelu_bwd")
                    # FC
                    self._aux(w_fc)
                    self._gemm_tn(g["dfc"], self.wT[p + "fc.w"], out=g["dln2"])
                    self._hook(f"h{l}/fc_dgrad")
                    # LN2 (+ residual gradient)
                    repops_layernorm_backward(g["dln2"], a["xmid"], W("ln2.g"), a["mu2"], a["rs2"], dres=dout,
                                              out=g["dxmid"])
                    self._hook(f"h{l}/ln2_bwd")
                    self._aux(w_ln2)
                    # proj
                    self._aux(w_proj)
                    self._gemm_tn(g["dxmid"], self.wT[p + "proj.w"], out=g["datt"])
                    self._hook(f"h{l}/proj_dgrad")
                    # attention
                    if self.attn_op and self.attn_dscores and self.attn_probs_ok and self._fault is None:
                        # f4: dP = dO V^T kept in shared memory, softmax backward in the same kernel
                        # (dP is operator-internal under R29); same dS bits as the two launches
                        repops_attention_dscores(g["datt"], a["qkv"], T, hd, d, (T * d, hd), 0, 3 * d,
                                                 (T * 3 * d, hd), 2 * d, a["P"], (H * T * T, T * T), g["dS"],
                                                 (H * T * T, T * T), (S_loc, H), scale=1.0 / np.sqrt(hd))
                    else:
                        repops_gemm_strided_batched(g["datt"], a["qkv"], g["dP"], M=T, N=T, K=hd, lda=d,
                                                    ldb=3 * d, ldc=T, sA=(T * d, hd), sB=(T * 3 * d, hd),
                                                    sC=(H * T * T, T * T), batch=(S_loc, H), transB=True, offB=2 * d)
                        self._hook(f"h{l}/attn_dp")
                        repops_softmax_backward(a["P"], g["dP"], scale=1.0 / np.sqrt(hd), out=g["dS"])
                        self._hook(f"h{l}/softmax_bwd")
                    # dV = P^T dO ; dQ = dS K ; dK = dS^T Q   (into the packed dqkv)
                    repops_gemm_strided_batched(a["P"], g["datt"], g["dqkv"], M=T, N=hd, K=T, lda=T, ldb=d,
                                                ldc=3 * d, sA=(H * T * T, T * T), sB=(T * d, hd),
                                                sC=(T * 3 * d, hd), batch=(S_loc, H), transA=True, offC=2 * d)
                    repops_gemm_strided_batched(g["dS"], a["qkv"], g["dqkv"], M=T, N=hd, K=T, lda=T, ldb=3 * d,
                                                ldc=3 * d, sA=(H * T * T, T * T), sB=(T * 3 * d, hd),
                                                sC=(T * 3 * d, hd), batch=(S_loc, H), offB=d)
                    repops_gemm_strided_batched(g["dS"], a["qkv"], g["dqkv"], M=T, N=hd, K=T, lda=T, ldb=3 * d,
                                                ldc=3 * d, sA=(H * T * T, T * T), sB=(T * 3 * d, hd),
                                                sC=(T * 3 * d, hd), batch=(S_loc, H), transA=True, offC=d)
                    self._hook(f"h{l}/attn_dqkv")
                    # QKV
                    self._aux(w_qkv)
                    self._gemm_tn(g["dqkv"], self.wT[p + "attn.w"], out=g["dln1"])
                    self._hook(f"h{l}/qkv_dgrad")
                    repops_layernorm_backward(g["dln1"], self.x[l], W("ln1.g"), a["mu1"], a["rs1"], dres=g["dxmid"],
                                              out=self.dx[l])
                    self._hook(f"h{l}/ln1_bwd")
                    self._aux(w_ln1)
                    self._aux_join()  # the phase's commit plan hashes every output of the layer
                    if self.p2p is not None and self.bucketed:
                        lo, hi = self._layer_range(l)
                        self._bucket(lo, hi)
                self.launch(bwd)
            pre = f"s{s}/h{l}/"
            t_dout = t_dx
            t_dgelu = T_(pre + "dgelu", V(g["dgelu"], T), s)
            self.node(OP["LINEAR_DGRAD"], s, attrs(layer=l, which=4), [t_dout, P_[p + "fc2.w"][0]], [t_dgelu],
                      pre + "fc2_dgrad")
            fg[p + "fc2.w"] = T_(f"s{s}/grad/{p}fc2.w", G_(p + "fc2.w"), s)
            self.node(OP["LINEAR_WGRAD"], s, attrs(layer=l, which=4), [ids["gelu"], t_dout], [fg[p + "fc2.w"]],
                      pre + "fc2_wgrad")
            fg[p + "fc2.b"] = T_(f"s{s}/grad/{p}fc2.b", G_(p + "fc2.b"), s)
            self.node(OP["BIAS_GRAD"], s, attrs(layer=l, which=4), [t_dout], [fg[p + "fc2.b"]], pre + "fc2_bgrad")
            t_dfc = T_(pre + "dfc", V(g["dfc"], T), s)
            self.node(OP["GELU_BWD"], s, attrs(layer=l), [ids["fc"], t_dgelu], [t_dfc], pre + "gelu_bwd")
            t_dln2 = T_(pre + "dln2", V(g["dln2"], T), s)
            self.node(OP["LINEAR_DGRAD"], s, attrs(layer=l, which=3), [t_dfc, P_[p + "fc.w"][0]], [t_dln2],
                      pre + "fc_dgrad")
            fg[p + "fc.w"] = T_(f"s{s}/grad/{p}fc.w", G_(p + "fc.w"), s)
            self.node(OP["LINEAR_WGRAD"], s, attrs(layer=l, which=3), [ids["ln2"], t_dfc], [fg[p + "fc.w"]],
                      pre + "fc_wgrad")
            fg[p + "fc.b"] = T_(f"s{s}/grad/{p}fc.b", G_(p + "fc.b"), s)
            self.node(OP["BIAS_GRAD"], s, attrs(layer=l, which=3), [t_dfc], [fg[p + "fc.b"]], pre + "fc_bgrad")
            t_dxmid = T_(pre + "dxmid", V(g["dxmid"], T), s)
            self.node(OP["LN_BWD"], s, attrs(layer=l, which=2),
                      [t_dln2, ids["xmid"], P_[p + "ln2.g"][0], ids["mu2"], ids["rs2"], t_dout], [t_dxmid],
                      pre + "ln2_bwd")
            fg[p + "ln2.g"] = T_(f"s{s}/grad/{p}ln2.g", G_(p + "ln2.g"), s)
            fg[p + "ln2.b"] = T_(f"s{s}/grad/{p}ln2.b", G_(p + "ln2.b"), s)
            self.node(OP["LN_PARAM_GRAD"], s, attrs(layer=l, which=2), [t_dln2, ids["xmid"], ids["mu2"], ids["rs2"]],
                      [fg[p + "ln2.g"], fg[p + "ln2.b"]], pre + "ln2_params")
            t_datt = T_(pre + "datt", V(g["datt"], T), s)
            self.node(OP["LINEAR_DGRAD"], s, attrs(layer=l, which=2), [t_dxmid, P_[p + "proj.w"][0]], [t_datt],
                      pre + "proj_dgrad")
            fg[p + "proj.w"] = T_(f"s{s}/grad/{p}proj.w", G_(p + "proj.w"), s)
            self.node(OP["LINEAR_WGRAD"], s, attrs(layer=l, which=2), [ids["att"], t_dxmid], [fg[p + "proj.w"]],
                      pre + "proj_wgrad")
            fg[p + "proj.b"] = T_(f"s{s}/grad/{p}proj.b", G_(p + "proj.b"), s)
            self.node(OP["BIAS_GRAD"], s, attrs(layer=l, which=2), [t_dxmid], [fg[p + "proj.b"]], pre + "proj_bgrad")
            if self.attn_op:
                t_dqkv = T_(pre + "dqkv", V(g["dqkv"], T), s)
                self.node(OP["ATTENTION_BWD"], s, attrs(layer=l, scale=float(1.0 / np.sqrt(hd)), causal=1),
                          [ids["qkv"], t_datt], [t_dqkv], pre + "attention_bwd", label=f"h{l}/attn_dqkv")
            else:
                t_dP = T_(pre + "dP", V(g["dP"], H * T), s)
                self.node(OP["ATTN_DP"], s, attrs(layer=l), [t_datt, ids["qkv"]], [t_dP], pre + "attn_dp")
                t_dS = T_(pre + "dS", V(g["dS"], H * T), s)
                self.node(OP["SOFTMAX_BWD"], s, attrs(layer=l, scale=float(1.0 / np.sqrt(hd))), [ids["P"], t_dP],
                          [t_dS], pre + "softmax_bwd")
                t_dqkv = T_(pre + "dqkv", V(g["dqkv"], T), s)
                self.node(OP["ATTN_DQKV"], s, attrs(layer=l), [t_dS, ids["P"], t_datt, ids["qkv"]], [t_dqkv],
                          pre + "attn_dqkv")
            t_dln1 = T_(pre + "dln1", V(g["dln1"], T), s)
            self.node(OP["LINEAR_DGRAD"], s, attrs(layer=l, which=1), [t_dqkv, P_[p + "attn.w"][0]], [t_dln1],
                      pre + "qkv_dgrad")
            fg[p + "attn.w"] = T_(f"s{s}/grad/{p}attn.w", G_(p + "attn.w"), s)
            self.node(OP["LINEAR_WGRAD"], s, attrs(layer=l, which=1), [ids["ln1"], t_dqkv], [fg[p + "attn.w"]],
                      pre + "qkv_wgrad")
            fg[p + "attn.b"] = T_(f"s{s}/grad/{p}attn.b", G_(p + "attn.b"), s)
            self.node(OP["BIAS_GRAD"], s, attrs(layer=l, which=1), [t_dqkv], [fg[p + "attn.b"]], pre + "qkv_bgrad")
            t_dx = T_(f"s{s}/dx{l}", V(self.dx[l], T), s)
            self.node(OP["LN_BWD"], s, attrs(layer=l, which=1),
                      [t_dln1, ids["x"], P_[p + "ln1.g"][0], ids["mu1"], ids["rs1"], t_dxmid], [t_dx],
                      pre + "ln1_bwd")
            fg[p + "ln1.g"] = T_(f"s{s}/grad/{p}ln1.g", G_(p + "ln1.g"), s)
            fg[p + "ln1.b"] = T_(f"s{s}/grad/{p}ln1.b", G_(p + "ln1.b"), s)
            self.node(OP["LN_PARAM_GRAD"], s, attrs(layer=l, which=1), [t_dln1, ids["x"], ids["mu1"], ids["rs1"]],
                      [fg[p + "ln1.g"], fg[p + "ln1.b"]], pre + "ln1_params")
        # ---------------- embedding backward (accumulates IN PLACE into the tied lm-head
        # gradient, so it runs -- and is committed -- in a global phase after every
        # shard's LM_WGRAD output has been committed; the node keeps its place in
        # the shard's node order)
        fg["wte"] = T_(f"s{s}/grad/wte", G_("wte"), s)
        fg["wpe"] = T_(f"s{s}/grad/wpe", G_("wpe"), s)
        self.node(OP["EMBED_BWD"], s, {}, [t_tok, t_dx, t_gwte_lm], [fg["wte"], fg["wpe"]], f"s{s}/embed_bwd",
                  defer=True)

    def _layer_range(self, l):
        """[lo, hi) of block l's parameters in the flat parameter / gradient layout."""
        c = self.cfg
        lo = self.off[f"h{l}.ln1.g"][0]
        hi = self.off[f"h{l + 1}.ln1.g"][0] if l + 1 < c.n_layer else self.off["lnf.g"][0]
        return lo, hi

    def _bucket(self, lo, hi):
        """combine gradient bucket [lo, hi) on the comm stream, after what the current
        stream has enqueued (the bucket's per-shard gradients)."""
        if hi <= lo:
            return
        if getattr(self, "comm", None) is None:
            self.comm = torch.cuda.Stream(device=self.dev, priority=-1)
        main = torch.cuda.current_stream()
        self.comm.wait_stream(main)
        parts = [self.glocal[q] for q in range(self.S_loc)]
        with torch.cuda.stream(self.comm):
            self.p2p.combine_range(parts, lo, hi, lambda ps, out: repops_tree_sum(ps, out=out), stream=self.comm)

    def _gslice(self, s, name):
        if not self._is_local(s):
            return torch.empty(0, device=self.dev)
        o, shape, _ = self.off[name]
        return self.glocal[s - self.s0, o:o + int(np.prod(shape))].view(*shape)

    def _build_tree_and_adam(self):
        c = self.cfg
        self.phase("embed_bwd")

        def emb_bwd():
            for q in range(self.S_loc):
                repops_embedding_backward(self.tok_in[q], self.dx[0][q * c.seq:(q + 1) * c.seq], c.seq,
                                          self._gslice(self.s0 + q, "wte"), self._gslice(self.s0 + q, "wpe"))
            for q, v, dirty in self._wte_inc:   # chunks of grad/wte the embedding backward rewrote
                verde_dirty_chunks(self.tok_in[q], v.shape[-1] * 4, v.numel() * 4, dirty,
                                   all_chunks=self._fault is not None or self._inject_active)
        self.launch(emb_bwd)
        self._cur[2].extend(self._deferred)
        self.phase("tree")

        def tree():
            parts = [self.glocal[q] for q in range(self.S_loc)]
            if self.p2p is not None:
                if not self.bucketed:
                    self.p2p(parts, lambda ps, out: repops_tree_sum(ps, out=out))
                    return
                # the parameters outside the transformer blocks (wte, wpe before them, lnf
                # after them), then the step's "done" barrier; AdamW waits for the comm stream
                self._bucket(0, self._layer_range(0)[0])
                self._bucket(self._layer_range(c.n_layer - 1)[1], self.P)
                with torch.cuda.stream(self.comm):
                    self.p2p.finish(stream=self.comm)
                torch.cuda.current_stream().wait_stream(self.comm)
                return
            combine = dp_tree_combine_sliced if self.sliced_combine else dp_tree_combine
            combine(parts, self.world, lambda ps, out: repops_tree_sum(ps, out=out), self.pg, out=self.grad)
        self.launch(tree)
        T_ = self._T
        self.grad_out = {}
        for name, shape, kind in self.specs:
            t = T_(f"grad/{name}", self.pview(self.grad, name), REPLICATED)
            ins = [self.final_grad[s][name] for s in range(c.shards)]
            self.node(OP["TREE_SUM"], REPLICATED, {}, ins, [t], f"tree/{name}")
            self.grad_out[name] = t
        self.phase("adamw")

        # one launch for all parameter tensors (they are stored back to back in
        # spec order); per-tensor decay flags, same element chain as repops_adamw
        seg_start = [self.off[name][0] for name, _, _ in self.specs] + [self.P]
        seg_decay = [len(shape) == 2 for _, shape, _ in self.specs]

        def adam():
            if not self.zero1:
                repops_adamw_segments(self.params, self.grad, self.m, self.v, seg_start, seg_decay, self.step_no + 1,
                                      c.lr, c.beta1, c.beta2, c.adam_eps, c.wd)
                return
            # ZeRO-1: the owned tensors' update (same element chain), then every parameter
            # tensor broadcast from its owner (data movement only)
            for name in self.owned:
                shape = self.off[name][1]
                repops_adamw(self.pview(self.params, name), self.pview(self.grad, name), self.mview(self.m, name),
                             self.mview(self.v, name), self.step_no + 1, c.lr, c.beta1, c.beta2, c.adam_eps, c.wd,
                             len(shape) == 2)
            if self.world > 1:
                import torch.distributed as dist
                for name, _, _ in self.specs:
                    dist.broadcast(self.pview(self.params, name), src=self.owner[name], group=self.pg)
        self.launch(adam)
        self.adam_out = {}
        for name, shape, kind in self.specs:
            p_, m_, v_ = self.param_in[name]
            outs = [T_(f"param'/{name}", self.pview(self.params, name), REPLICATED),
                    T_(f"m'/{name}", self.mview(self.m, name), REPLICATED),
                    T_(f"v'/{name}", self.mview(self.v, name), REPLICATED)]
            attrs = {AK["lr"]: f32bits(c.lr), AK["beta1"]: f32bits(c.beta1), AK["beta2"]: f32bits(c.beta2),
                     AK["adam_eps"]: f32bits(c.adam_eps), AK["wd"]: f32bits(c.wd),
                     AK["decay"]: int(len(shape) == 2)}
            self.node(OP["ADAMW"], REPLICATED, attrs, [p_, self.grad_out[name], m_, v_], outs, f"adamw/{name}")
            self.adamw_node[name] = len(self.nodes) - 1
            self.adam_out[name] = outs

    # ------------------------------------------------------------------ finalisation
    def _finalize(self):
        c = self.cfg
        # digest slots: replicated ids first, then shard regions with a common stride
        for i, t in enumerate(self._rep_ids):
            self.tensors[t].slot = i
        n_rep = len(self._rep_ids)
        per = len(self._shard_ids[0])
        assert all(len(v) == per for v in self._shard_ids.values())
        self.rep_slots, self.shard_slots = n_rep, per
        for s in range(c.shards):
            for i, t in enumerate(self._shard_ids[s]):
                self.tensors[t].slot = n_rep + s * per + i
        self.n_slots = n_rep + c.shards * per
        self.digests = torch.zeros((self.n_slots, 32), dtype=torch.uint8, device=self.dev)
        pin = (lambda t: t) if self.structure_only else (lambda t: t.pin_memory())
        self.digests_host = pin(torch.zeros((self.n_slots, 32), dtype=torch.uint8))
        # consumers (output node pointers of the box)
        for nd in self.nodes:
            for t in nd.inputs:
                src = self.tensors[t].producer
                if nd.index not in self.nodes[src].dsts:
                    self.nodes[src].dsts.append(nd.index)
        # token arrays used by the batched launches (staged from the host with the batch)
        self.tok_in = torch.empty((self.S_loc, c.seq), dtype=torch.int32, device=self.dev)
        self.tok_in_flat = self.tok_in.view(-1)
        self.targets = torch.empty((self.S_loc, c.seq), dtype=torch.int32, device=self.dev)
        self.targets_flat = self.targets.view(-1)
        self.tok_host = pin(torch.empty((self.S_loc, c.seq + 1), dtype=torch.int32))
        self.tin_host = pin(torch.empty((self.S_loc, c.seq), dtype=torch.int32))
        self.tgt_host = pin(torch.empty((self.S_loc, c.seq), dtype=torch.int32))
        # Commit plans, one per phase whose launches produce local tensors (all
        # local shards of a batched launch together).  They run on a side stream,
        # each after an event recorded when its phase's kernels are enqueued, so
        # SHA-256 (integer ALU pipe) overlaps the next phases' GEMMs (FMA pipe).
        # A tensor must be hashed before anything modifies it in place; the only
        # in-place writers are the embedding backward (the tied lm-head gradient)
        # and AdamW (parameters / moments) -- run() makes those phases wait for
        # the side stream.
        deferred_phase = next(i for i, p in enumerate(self.phases) if p[0] == "embed_bwd")
        per_phase = {}
        for name, fns, tids in self.phases:
            for t in tids:
                ph = self._tensor_phase.get(t)
                ph = deferred_phase if ph is None else ph
                per_phase.setdefault(ph, []).append(t)
        self.plan_after = {}
        self.plans = []
        # ZeRO-1: a rank commits only the replicated tensors of the parameters it owns; the
        # other replicated digests come from their owners (_gather_rep_digests)
        self._rep_owner = np.zeros(max(n_rep, 1), np.int64)
        for i, t in enumerate(self._rep_ids):
            self._rep_owner[i] = self.owner.get(self.tensors[t].name.split("/", 1)[1], 0)
        not_mine = {t for i, t in enumerate(self._rep_ids) if self.zero1 and self._rep_owner[i] != self.rank}
        # Incremental commitment of the tied embedding gradient (R-TCOMMIT digest unchanged):
        # EMBED_BWD adds into the rows of the shard's tokens of the buffer that already holds
        # LM_WGRAD's output (committed as s/grad/wte_lm), so grad/wte differs from it in at most
        # ntok rows; its commit re-hashes only the 4 KiB chunks those rows meet and takes every
        # other chunk leaf from the wte_lm commit (1.2 GB less SHA-256 per GPT-2 step).  Fault
        # injection (config 5) re-hashes every chunk (an injected flip may sit anywhere).
        inc = {}
        self._wte_inc = []
        if self.delta_commit and not self.structure_only:
            for q in range(self.S_loc):
                s_ = self.s0 + q
                t_lm = next(t for t, tr in enumerate(self.tensors) if tr.name == f"s{s_}/grad/wte_lm")
                t_w = next(t for t, tr in enumerate(self.tensors) if tr.name == f"s{s_}/grad/wte")
                v = self.tensors[t_w].view
                assert v.data_ptr() == self.tensors[t_lm].view.data_ptr() and v.numel() == self.tensors[t_lm].view.numel()
                nch = (v.numel() * 4 + 4095) // 4096
                leaves = torch.empty(nch * 32, dtype=torch.uint8, device=self.dev)
                dirty = torch.ones(nch, dtype=torch.uint8, device=self.dev)
                inc[t_lm] = dict(leaves_out=leaves)
                inc[t_w] = dict(base_leaves=leaves, dirty=dirty)
                self._wte_inc.append((q, v, dirty))
        for ph, tids in sorted(per_phase.items()):
            tids = [t for t in tids if t not in not_mine]
            if tids and not self.structure_only:
                plan = CommitPlan([self.tensors[t].view for t in tids],
                                  [self.digests[self.tensors[t].slot] for t in tids],
                                  incremental={i: inc[t] for i, t in enumerate(tids) if t in inc})
                self.plans.append(plan)
                self.plan_after[ph] = plan
        self.commit_bytes = sum(p.nbytes for p in self.plans)
        self._wait_side_before = {deferred_phase, next(i for i, p in enumerate(self.phases) if p[0] == "adamw")}
        # Commits of the "tree" / "adamw" phases hash buffers (grad, p, m, v) that the
        # next step rewrites only after a _wait_side_before phase, so with join=False
        # they (and the root plan) may run beside the next step's forward; every
        # other commit must finish before the next step rewrites its activations.
        self._tail_from = next(i for i, p in enumerate(self.phases) if p[0] == "tree")
        self._last_act_plan = max(i for i in self.plan_after if i < self._tail_from) if self.plan_after else -1
        self._joined = True
        if not self.structure_only:
            self.side = torch.cuda.Stream(device=self.dev, priority=int(os.environ.get("REPOPS_SIDE_PRIO", "0")))
            self.overlap_commits = True
            self._ev_act = torch.cuda.Event()
            self._ev_root = torch.cuda.Event()
        self._build_node_blob()
        # committed tensors that a later node rewrites in place (same storage): the
        # tied lm-head gradient (EMBED_BWD accumulates into it).  PARAM_IN outputs are
        # excluded: a trainer serves those from its saved starting checkpoint.
        self._overwritten = []
        if not self.structure_only:
            groups = {}
            for tid, t in enumerate(self.tensors):
                if t.view.numel() and t.view.device.type != "meta":  # remote shards hold empty placeholders
                    groups.setdefault((t.view.data_ptr(), t.view.numel()), []).append(tid)
            for tids in groups.values():
                for tid in tids[:-1]:
                    if self.nodes[self.tensors[tid].producer].op != OP["PARAM_IN"]:
                        self._overwritten.append(tid)
        # Targeted waits: an in-place writer waits only for the commit plan that
        # hashed what it overwrites (not for the whole side-stream backlog):
        #   embed_bwd -> the plan holding the tied lm-head gradients (_overwritten),
        #   adamw     -> the plan holding the PARAM_IN tensors (p, m, v).
        ph_of = lambda t: deferred_phase if self._tensor_phase.get(t) is None else self._tensor_phase[t]  # noqa: E731
        adamw_phase = next(i for i, p in enumerate(self.phases) if p[0] == "adamw")
        pin = [t for ids in self.param_in.values() for t in ids]
        self._wait_on = {adamw_phase: max(ph_of(t) for t in pin)}
        if self._overwritten:
            self._wait_on[deferred_phase] = max(ph_of(t) for t in self._overwritten)
        assert all(w in self.plan_after or self.structure_only for w in self._wait_on.values())
        self._plan_ev = {} if self.structure_only else {ph: torch.cuda.Event() for ph in self.plan_after}
        if not self.structure_only:
            from . import RootPlan
            self.root_plan = RootPlan(self.node_blob, self.node_offs, self.node_slots, self.node_soffs,
                                      self.digests, with_nodes=True)
            self.root_host = torch.zeros(32, dtype=torch.uint8).pin_memory()

    def _build_node_blob(self):
        """Static serialisation of every node except its tensor digests (R13)."""
        blob, offs, slots, soffs = bytearray(), [0], [], [0]
        for nd in self.nodes:
            keys = sorted(nd.attrs)
            b = bytearray(b"\x4e")
            b += struct.pack("<IHI", nd.index, nd.op, nd.shard)
            b += struct.pack("<I", len(keys))
            for k in keys:
                b += struct.pack("<IQ", k, nd.attrs[k])
            b += struct.pack("<I", len(nd.inputs))
            for t in nd.inputs:
                b += struct.pack("<II", self.tensors[t].producer, self.tensors[t].pslot)
            b += struct.pack("<I", len(nd.dsts))
            for q in nd.dsts:
                b += struct.pack("<I", q)
            b += struct.pack("<I", len(nd.outputs))
            blob += b
            offs.append(len(blob))
            slots += [self.tensors[t].slot for t in nd.inputs] + [self.tensors[t].slot for t in nd.outputs]
            soffs.append(len(slots))
        self.node_blob = np.frombuffer(bytes(blob), np.uint8).copy()
        self.node_offs = np.asarray(offs, np.int64)
        self.node_slots = np.asarray(slots, np.int64)
        self.node_soffs = np.asarray(soffs, np.int64)

    # ------------------------------------------------------------------ running
    def batch_tokens(self, shard: int, step_index: int):
        """The dataset's batch for `shard` at training step `step_index` (1-based; step t
        consumes synthetic batch t-1), as the committed int32 [T+1] tensor -- what the
        referee checks a disputed TOKENS_IN node against."""
        c = self.cfg
        h = synth.gpt2_tokens(c.vocab, c.seq, shard, step_index - 1, c.seed)
        return torch.from_numpy(np.ascontiguousarray(h, dtype=np.int32))

    def set_tokens(self, step: int | None = None, host_tokens=None):
        """Load this rank's shards' tokens (synthetic recipe, or given host int32 [S_loc, T+1])."""
        c = self.cfg
        if host_tokens is None:
            st = self.step_no if step is None else step
            host_tokens = np.stack([synth.gpt2_tokens(c.vocab, c.seq, self.s0 + q, st, c.seed)
                                    for q in range(self.S_loc)])
        h = np.ascontiguousarray(host_tokens, dtype=np.int32)
        self.tok_host.numpy()[...] = h
        self.tin_host.numpy()[...] = h[:, :c.seq]
        self.tgt_host.numpy()[...] = h[:, 1:]
        self.tok.copy_(self.tok_host, non_blocking=True)     # H2D: the step's input batch
        self.tok_in.copy_(self.tin_host, non_blocking=True)
        self.targets.copy_(self.tgt_host, non_blocking=True)

    @property
    def h2d_bytes(self):
        return 3 * self.tok_host.numel() * 4

    def inject_fault(self, node_index, out_slot=0, elem=0, bit=0):
        """Arm a 1-bit flip of element `elem` of output `out_slot` of node `node_index`,
        applied right after the launch that produces it (so it propagates downstream).
        Used to build a dishonest trainer for the Verde dispute (config 5)."""
        from . import repops_flip_bit
        nd = self.nodes[node_index]
        if nd.label is None or not self._is_local(nd.shard):
            raise ValueError("fault injection needs a local per-shard node with a launch hook")
        view = self.tensors[nd.outputs[out_slot]].view
        self._fault = (nd.label, lambda: repops_flip_bit(view, elem, bit))

    def state_changed(self):
        """The training state (params / m / v) was written outside run(): the next step
        re-hashes its PARAM_IN tensors instead of reusing the last AdamW digests."""
        self._state_digests_valid = False

    def _copy_state_digests(self, stream):
        """PARAM_IN digest slots <- the previous step's AdamW output slots (same bytes)."""
        from . import repops_copy2d
        if not hasattr(self, "_dig_rows"):
            pin = [self.tensors[t].slot for name, _, _ in self.specs for t in self.param_in[name]]
            aout = [self.tensors[t].slot for name, _, _ in self.specs for t in self.adam_out[name]]
            assert pin == list(range(pin[0], pin[0] + len(pin))) and aout == list(range(aout[0], aout[0] + len(aout)))
            self._dig_rows = (pin[0], aout[0], len(pin))
        p0, a0, n = self._dig_rows
        f = self.digests.view(torch.float32)  # [n_slots, 8]: 32 digest bytes as 8 words (bit-exact copy)
        repops_copy2d(f[a0:a0 + n], f[p0:p0 + n], stream=stream)

    def run(self, commit=True, inject=None, join=True):
        """Enqueue one full training step.  inject = (phase_name, fn) runs fn after that
        phase's kernels (coarse fault injection; see inject_fault for per-op points).
        join=False: the main stream only waits for the activation commits, so the
        tail commits (tree / AdamW outputs) overlap the next step; device_root() then
        runs on the side stream and join() waits for everything."""
        main = torch.cuda.current_stream()
        side = self.side if self.overlap_commits else main
        self._inject_active = inject is not None   # a coarse fault may land anywhere: full re-hash
        self.stash = {}
        if side is not main:
            side.wait_stream(main)  # the step's inputs (tokens, checkpoint) are ready
        for i, (name, fns, _) in enumerate(self.phases):
            if commit and side is not main and i in self._wait_on:
                main.wait_event(self._plan_ev[self._wait_on[i]])  # what it overwrites is hashed
            if self.keep_committed and i in self._wait_side_before:
                for tid in self._overwritten:  # first in-place writer of the step comes next
                    if tid not in self.stash:
                        self.stash[tid] = self.tensors[tid].view.clone()
            for fn in fns:
                fn()
            if inject is not None and inject[0] == name:
                inject[1]()
            plan = self.plan_after.get(i)
            if commit and plan is not None:
                reuse = (i == 0 and self.reuse_state_digests and self._state_digests_valid and self._fault is None)
                if side is main:
                    self._copy_state_digests(main) if reuse else plan.run()
                else:
                    side.wait_stream(main)
                    self._copy_state_digests(side) if reuse else plan.run(stream=side)
                    self._plan_ev[i].record(side)
                    if i == self._last_act_plan:
                        self._ev_act.record(side)
        if side is not main:
            if join or not commit:
                main.wait_stream(side)
            else:
                main.wait_event(self._ev_act)
        self._joined = side is main or join or not commit
        # AdamW's outputs of this step were committed iff commit: they are the next PARAM_IN
        self._state_digests_valid = bool(commit)
        self.step_no += 1

    def join(self):
        """Make the current stream wait for every enqueued commit / root launch."""
        if not self.structure_only and self.overlap_commits:
            torch.cuda.current_stream().wait_stream(self.side)
        self._joined = True

    def _gather_rep_digests(self):
        """ZeRO-1: every replicated slot takes its owner's digest (all-gather of the
        replicated region, ≈ 7 x 32 B per parameter tensor per rank)."""
        if not self.zero1 or self.world == 1:
            return
        from .dist import all_gather_rows
        if not hasattr(self, "_rep_sel"):
            self._rep_sel = (torch.from_numpy(self._rep_owner[:self.rep_slots]).to(self.dev),
                             torch.arange(self.rep_slots, device=self.dev))
        allr = all_gather_rows(self.digests[:self.rep_slots].contiguous(), self.world, self.pg)
        self.digests[:self.rep_slots] = allr[self._rep_sel[0], self._rep_sel[1]]

    def gather_digests(self):
        """C2: all-gather the per-shard digest regions; copy the table to the host."""
        gather_shard_digests(self.digests, self.rep_slots, self.shard_slots, self.s0, self.S_loc, self.world, self.pg)
        self._gather_rep_digests()
        self.digests_host.copy_(self.digests, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.digests_host.numpy()

    def device_root(self, sync=True):
        """Step root computed on the GPU (verde_root_plan): C2 gather of the shard digest
        regions (N > 1), node digests, RFC 6962 root; only 32 bytes come back.  After
        run(join=False) this is enqueued on the side stream behind the tail commits;
        with sync=False call root_bytes() later."""
        s = torch.cuda.current_stream() if self._joined else self.side
        with torch.cuda.stream(s):
            gather_shard_digests(self.digests, self.rep_slots, self.shard_slots, self.s0, self.S_loc, self.world,
                                 self.pg)
            self._gather_rep_digests()
            self.root_plan.run(stream=s)
            self.root_host.copy_(self.root_plan.root, non_blocking=True)
            self._ev_root.record(s)
        if sync:
            return self.root_bytes()
        return None

    def root_bytes(self):
        """The last device_root() result (waits for it).  Raises if the step's peer-memory
        gradient exchange timed out (its gradients -- and so this root -- are not valid)."""
        self._ev_root.synchronize()
        self._check_exchange()
        return bytes(self.root_host.numpy())

    def _check_exchange(self):
        if self.p2p is not None:
            torch.cuda.current_stream().synchronize()
            self.p2p.check()

    def step_root(self, table=None):
        """Node digests (R-NODE) and the step's Merkle root (R-MERKLE), host native code."""
        if table is None:
            table = self.gather_digests()
            self._check_exchange()
        n = len(self.nodes)
        out = np.empty((n, 32), np.uint8)
        root = np.empty(32, np.uint8)
        P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        check(lib().verde_node_digests(n, P(self.node_blob), P(self.node_offs), P(self.node_slots),
                                       P(self.node_soffs), P(np.ascontiguousarray(table)), self.n_slots, P(out),
                                       P(root)), "verde_node_digests")
        return root.tobytes(), out

    # ------------------------------------------------------------------ checkpoint commitments
    def checkpoint_commit(self, stream=None):
        """Enqueue the commitment of the training state (every parameter's param, m, v --
        the starting checkpoint C_i of the next step): R-TCOMMIT digests into a
        [3 x n_params, 32] device table, in checkpoint_entries order (verde.py).  This is
        what a trainer logs at the checkpoint steps of Alg. 1 when it does not
        commit every operator output (configs[2] without configs[4])."""
        from . import CommitPlan
        if self.zero1 and self.world > 1:
            raise NotImplementedError("checkpoint_commit with ZeRO-1: the state is partitioned across ranks")
        if getattr(self, "_ckpt_plan", None) is None:
            views = []
            for name, _, _ in self.specs:
                views += [self.pview(self.params, name), self.pview(self.m, name), self.pview(self.v, name)]
            self._ckpt_digests = torch.zeros((len(views), 32), dtype=torch.uint8, device=self.dev)
            self._ckpt_plan = CommitPlan(views, self._ckpt_digests)
        self._ckpt_plan.run(stream=stream)

    def checkpoint_root(self) -> bytes:
        """RFC 6962 root over the last checkpoint_commit()'s digests (waits for them)."""
        from . import verde_merkle_root
        d = self._ckpt_digests.cpu().numpy()
        return verde_merkle_root([d[i].tobytes() for i in range(d.shape[0])])

    def loss(self):
        """Step loss (reported metric): R-SEQ per shard, R-TREE_S over shards, x 1/(S T)."""
        from . import repops_sum_cols_seq as seq
        seq(self.loss_tok.view(-1, 1), nseg=self.S_loc, out=self.shard_loss.view(-1, 1))
        allv = all_gather_rows(self.shard_loss, self.world, self.pg).reshape(-1)
        tot = repops_tree_sum([allv[q:q + 1] for q in range(self.cfg.shards)])
        return float(np.float32(tot.item()) * np.float32(1.0 / (self.cfg.shards * self.cfg.seq)))

    def flops_per_step(self):
        """Algorithmic matmul flops of one full step (all shards): fwd 2*M*N*K, bwd 2x fwd."""
        c = self.cfg
        Ntok = c.shards * c.seq
        lin = 2 * Ntok * (c.d * 3 * c.d + c.d * c.d + 2 * c.d * c.ffn) * c.n_layer
        attn = 2 * 2 * c.shards * c.n_head * c.seq * c.seq * c.hd * c.n_layer
        head = 2 * Ntok * c.d * c.vocab
        return 3 * (lin + attn + head)
