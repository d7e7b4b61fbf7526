"""Verde dispute resolution on top of the RepOps GPT-2 step (BASELINE config 5).

Implements the paper's Phase 2 and the referee's decision algorithm for a
disputed training step (Sec. 2.2-2.3):
  * each trainer commits every node of the step's extended graph
    (AugmentedCGNode, box P:400-406) and the step root = MerkleHash(node hashes)
    (Fig. 2);
  * Alg. 2: the referee checks h_end == MerkleHash(seq) for each
    trainer (line 7) and finds the first differing node d (line 8) -- here by
    descending the two RFC 6962 trees, O(log n) subtree comparisons
    (verde_first_divergence);
  * decision: Case 1 (graph structure differs), Case 2 (an input
    hash differs: the source node's emitted hash decides), Case 3 (an output
    hash differs: the referee recomputes the single operator on the agreed
    inputs with RepOps and compares output hashes).
The referee's recompute uses the same RepOps kernels (bitwise reproducibility
between referee and trainers is the paper's premise).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import (EPI_BIAS, EPI_SCALE, repops_add, repops_adamw, repops_cross_entropy, repops_embedding,
               repops_embedding_backward, repops_gelu, repops_gelu_backward, repops_gemm,
               repops_gemm_strided_batched, repops_layernorm, repops_layernorm_backward,
               repops_layernorm_backward_params, repops_softmax, repops_softmax_backward, repops_sum_cols_seq,
               repops_tree_sum, verde_commit_tensors, verde_first_divergence, verde_merkle_root)
from .gpt2 import AK, OP, REPLICATED, GPT2Step


@dataclass
class Opening:
    """A trainer's opening of node d (Alg. 2 line 10): structure + tensor hashes."""
    index: int
    structure: bytes        # the node's static serialisation (op, attrs, edges)
    in_digests: list
    out_digests: list


class Trainer:
    """A trainer that ran one step and answers the referee's queries."""

    def __init__(self, step: GPT2Step, checkpoint):
        """checkpoint: (params, m, v) flat copies taken BEFORE the step (the trainer keeps
        its starting checkpoint C_i; AdamW updates the live buffers in place)."""
        self.st = step
        self.ckpt = dict(zip(("param", "m", "v"), checkpoint))
        self.root, self.node_digests = step.step_root()
        self.table = step.digests_host.numpy().copy()

    def seq(self) -> bytes:
        return self.node_digests.tobytes()

    def open(self, d: int) -> Opening:
        st = self.st
        nd = st.nodes[d]
        blob = st.node_blob[st.node_offs[d]:st.node_offs[d + 1]].tobytes()
        return Opening(d, blob, [self.table[st.tensors[t].slot].tobytes() for t in nd.inputs],
                       [self.table[st.tensors[t].slot].tobytes() for t in nd.outputs])

    def input_tensors(self, d: int):
        st = self.st
        out = []
        for t in st.nodes[d].inputs:
            name = st.tensors[t].name
            kind, _, pname = name.partition("/")
            if kind in self.ckpt:      # checkpoint input: served from the saved C_i
                out.append(st.pview(self.ckpt[kind], pname))
            else:
                out.append(st.tensors[t].view)
        return out


@dataclass
class Verdict:
    d: int
    case: int               # 1, 2 or 3
    dishonest: int          # 0 or 1
    rounds: int             # subtree comparisons to find d
    detail: str


def phase2(t0: Trainer, t1: Trainer) -> tuple[int, int]:
    """Alg. 2: consistency check (line 7) + first diverging node (line 8)."""
    for t in (t0, t1):
        if verde_merkle_root([t.seq()[i:i + 32] for i in range(0, len(t.seq()), 32)]) != t.root:
            raise ValueError("trainer's node sequence does not hash to its claimed checkpoint")
    return verde_first_divergence(t0.seq(), t1.seq())


def decide(t0: Trainer, t1: Trainer, d: int, rounds: int, program: GPT2Step) -> Verdict:
    o0, o1 = t0.open(d), t1.open(d)
    nd = program.nodes[d]
    ref_struct = program.node_blob[program.node_offs[d]:program.node_offs[d + 1]].tobytes()
    # Case 1: graph structure (inputs, outputs, operator) -- the referee knows the program
    if o0.structure != o1.structure:
        bad = 0 if o0.structure != ref_struct else 1
        return Verdict(d, 1, bad, rounds, "node structure differs from the program")
    # Case 2: an input hash differs -> the source node's emitted hash decides
    for q, (a, b) in enumerate(zip(o0.in_digests, o1.in_digests)):
        if a != b:
            src = program.tensors[nd.inputs[q]]
            # nodes before d agree, so the source node's output hash is common to both
            agreed = t0.open(src.producer).out_digests[src.pslot]
            bad = 0 if a != agreed else 1
            return Verdict(d, 2, bad, rounds, f"input {q} hash differs from source node {src.producer}")
    # Case 3: output hashes differ -> recompute the operator on the agreed inputs
    outs = referee_recompute(program, d, t0.input_tensors(d), o0.in_digests)
    mine = [bytes(x) for x in verde_commit_tensors(outs).cpu().numpy()]
    ok0 = mine == o0.out_digests
    ok1 = mine == o1.out_digests
    if ok0 == ok1:
        raise RuntimeError("referee recompute matches neither / both trainers")
    return Verdict(d, 3, 1 if ok0 else 0, rounds, f"recomputed {nd.name} (op {nd.op})")


def referee_recompute(program: GPT2Step, d: int, inputs, in_digests) -> list:
    """Re-run node d's single operator with RepOps on fresh buffers, after checking
    that the provided input tensors hash to the agreed input digests."""
    ins = [t.clone() for t in inputs]
    got = [bytes(x) for x in verde_commit_tensors(ins).cpu().numpy()] if ins else []
    if got != list(in_digests):
        raise ValueError("provided input tensors do not match the agreed input hashes")
    return replay(program, program.nodes[d], ins)


def replay(st: GPT2Step, nd, x):
    """One operator of the GPT-2 program, for one shard, from its input tensors."""
    c = st.cfg
    T, d, H, hd, V = c.seq, c.d, c.n_head, c.hd, c.vocab
    op, a = nd.op, nd.attrs
    E = lambda *s: torch.empty(*s, device=x[0].device if x else "cuda")  # noqa: E731
    sc = float(np.float32(1.0 / np.sqrt(hd)))
    if op == OP["EMBED"]:
        tok, wte, wpe = x
        return [repops_embedding(tok[:T].contiguous(), wte, wpe, T)]
    if op == OP["LAYERNORM"]:
        y, mu, rs = repops_layernorm(x[0], x[1], x[2], c.ln_eps)
        return [y, mu, rs]
    if op == OP["LINEAR"]:
        return [repops_gemm(x[0], x[1], epi=EPI_BIAS, bias=x[2])]
    if op == OP["ATTN_SCORES"]:
        qkv = x[0]
        S = E(H * T, T)
        repops_gemm_strided_batched(qkv, qkv, S, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T, sA=(0, hd),
                                    sB=(0, hd), sC=(0, T * T), batch=(1, H), transB=True, epi=EPI_SCALE, scale=sc,
                                    offB=d)
        return [S]
    if op == OP["SOFTMAX"]:
        return [repops_softmax(x[0], causal=True)]
    if op == OP["ATTN_PV"]:
        P, qkv = x
        att = E(T, d)
        repops_gemm_strided_batched(P, qkv, att, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d, sA=(0, T * T),
                                    sB=(0, hd), sC=(0, hd), batch=(1, H), offB=2 * d)
        return [att]
    if op == OP["RESIDUAL"]:
        return [repops_add(x[0], x[1])]
    if op == OP["GELU"]:
        return [repops_gelu(x[0])]
    if op == OP["LM_HEAD"]:
        logits = torch.zeros(T, c.vocab_ld, device=x[0].device)
        repops_gemm(x[0], x[1], transB=True, out=logits[:, :V])
        return [logits]
    if op == OP["CROSS_ENTROPY"]:
        logits, tok = x
        tgt = tok[1:].contiguous()
        dl = torch.zeros_like(logits)
        loss, _ = repops_cross_entropy(logits, tgt, scale=1.0 / (c.shards * c.seq), dlogits=dl, V=V)
        return [loss, dl]
    if op == OP["LM_DGRAD"]:
        return [repops_gemm(x[0][:, :V], x[1])]
    if op == OP["LM_WGRAD"]:
        return [repops_gemm(x[0][:, :V], x[1], transA=True)]
    if op == OP["LN_BWD"]:
        dres = x[5] if len(x) > 5 else None
        return [repops_layernorm_backward(x[0], x[1], x[2], x[3], x[4], dres=dres)]
    if op == OP["LN_PARAM_GRAD"]:
        dg, db = repops_layernorm_backward_params(x[0], x[1], x[2], x[3], nseg=1)
        return [dg.view(-1), db.view(-1)]
    if op == OP["LINEAR_DGRAD"]:
        return [repops_gemm(x[0], x[1], transB=True)]
    if op == OP["LINEAR_WGRAD"]:
        return [repops_gemm(x[0], x[1], transA=True)]
    if op == OP["BIAS_GRAD"]:
        return [repops_sum_cols_seq(x[0], nseg=1).view(-1)]
    if op == OP["GELU_BWD"]:
        return [repops_gelu_backward(x[0], x[1])]
    if op == OP["ATTN_DP"]:
        datt, qkv = x
        dP = E(H * T, T)
        repops_gemm_strided_batched(datt, qkv, dP, M=T, N=T, K=hd, lda=d, ldb=3 * d, ldc=T, sA=(0, hd),
                                    sB=(0, hd), sC=(0, T * T), batch=(1, H), transB=True, offB=2 * d)
        return [dP]
    if op == OP["SOFTMAX_BWD"]:
        return [repops_softmax_backward(x[0], x[1], scale=sc)]
    if op == OP["ATTN_DQKV"]:
        dS, P, datt, qkv = x
        dq = E(T, 3 * d)
        kw = dict(M=T, N=hd, K=T, lda=T, ldc=3 * d, sA=(0, T * T), sC=(0, hd), batch=(1, H))
        repops_gemm_strided_batched(P, datt, dq, ldb=d, sB=(0, hd), transA=True, offC=2 * d, **kw)
        repops_gemm_strided_batched(dS, qkv, dq, ldb=3 * d, sB=(0, hd), offB=d, **kw)
        repops_gemm_strided_batched(dS, qkv, dq, ldb=3 * d, sB=(0, hd), transA=True, offC=d, **kw)
        return [dq]
    if op == OP["EMBED_BWD"]:
        tok, dx0, gwte_lm = x
        gwte = gwte_lm.clone()
        gwpe = torch.zeros(c.n_pos, d, device=dx0.device)
        repops_embedding_backward(tok[:T].contiguous(), dx0, T, gwte, gwpe)
        return [gwte, gwpe]
    if op == OP["TREE_SUM"]:
        return [repops_tree_sum([t.contiguous() for t in x])]
    if op == OP["ADAMW"]:
        p, g, m, v = (t.clone() for t in x)
        decay = bool(a.get(AK["decay"], 0))
        repops_adamw(p.view(-1), g.view(-1), m.view(-1), v.view(-1), st.step_no, c.lr, c.beta1, c.beta2,
                     c.adam_eps, c.wd, decay)
        return [p, m, v]
    raise NotImplementedError(f"replay of op {op}")


def dispute(cfg, fault_node: int, elem: int = 0, bit: int = 0, out_slot: int = 0, dishonest: int = 1,
            tokens_step: int = 0):
    """Run an honest and a dishonest trainer (1-bit flip after node `fault_node`'s
    launch) on the same checkpoint and batch; resolve with Phase 2 + decision."""
    honest = GPT2Step(cfg)
    honest.set_tokens(tokens_step)
    ck_h = (honest.params.clone(), honest.m.clone(), honest.v.clone())
    honest.run()
    cheat = GPT2Step(cfg)
    cheat.set_tokens(tokens_step)
    ck_c = (cheat.params.clone(), cheat.m.clone(), cheat.v.clone())
    cheat.inject_fault(fault_node, out_slot, elem, bit)
    cheat.run()
    th, tc = Trainer(honest, ck_h), Trainer(cheat, ck_c)
    t0, t1 = (th, tc) if dishonest == 1 else (tc, th)
    if t0.root == t1.root:
        return None  # no dispute
    d, rounds = phase2(t0, t1)
    return decide(t0, t1, d, rounds, honest)
