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

Beyond one disputed step:
  * Phase 1 (Alg. 1): `TrainingRun` logs checkpoint hashes (= step
    roots, Fig. 2) at k_0 steps while training and keeps those states; `phase1`
    narrows the first diverging step level by level, each trainer re-executing
    only the diverging segment with finer logging (counts k_1, k_2, ...);
  * Case 2(a): a disputed checkpoint tensor (a PARAM_IN output) is
    settled by Merkle membership proofs against the agreed h_start -- the opened
    AdamW node of the previous step plus its RFC 6962 audit path (or, for step 1,
    the entry's path in the C0 tree); training data (TOKENS_IN) against the
    dataset recipe;
  * Case 3 at chunk granularity: the referee checks each trainer's
    4 KiB chunk leaves against its output digest, descends the two data trees to
    the first differing chunk, and recomputes only that chunk's elements (the
    GEMM rows / elementwise slice that produce it).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import synth

from . import (EPI_BIAS, EPI_SCALE, repops_add, repops_adamw, repops_cross_entropy, repops_embedding,
               repops_embedding_backward, repops_flip_bit, repops_gelu, repops_gelu_backward, repops_gemm,
               repops_gemm_strided_batched, repops_layernorm, repops_layernorm_backward,
               repops_layernorm_backward_params, repops_softmax, repops_softmax_backward, repops_sum_cols_seq,
               repops_tree_sum, verde_chunk_leaves, verde_commit_tensors, verde_first_divergence,
               verde_merkle_audit_path, verde_merkle_root, verde_merkle_root_hashed, verde_merkle_verify_path,
               verde_sha256, verde_tensor_digest_from_root)
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

    def __init__(self, step: GPT2Step, checkpoint, prev=None, step_index=None):
        """checkpoint: (params, m, v) flat copies taken BEFORE the step (the trainer keeps
        its starting checkpoint C_i; AdamW updates the live buffers in place).
        prev: what the trainer logged for the previous checkpoint (TrainingRun.log
        entry), used for membership proofs (Case 2(a)); step_index: the step's number."""
        self.st = step
        self.ckpt = dict(zip(("param", "m", "v"), checkpoint))
        self.root, self.node_digests = step.step_root()
        self.table = step.digests_host.numpy().copy()
        self.prev = prev
        self.step_index = step.step_no if step_index is None else step_index

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
            else:                      # as committed (stashed if rewritten in place later)
                out.append(st.stash.get(t, st.tensors[t].view))
        return out

    # ---- Case 2(a): membership of a checkpoint tensor in h_start
    def prove_checkpoint(self, param: str, slot: int):
        """Proof that this trainer's (param, m or v) digest for `param` is committed by
        the agreed starting checkpoint: for step 1 the entry's audit path in the C0
        tree; later, the opening of the previous step's AdamW node for `param` and
        that node digest's audit path in the previous step's node tree."""
        claimed = self.open(self.st.param_in_node[param]).out_digests[slot]
        if self.prev is None:
            raise ValueError("no previous checkpoint log to prove membership from")
        if self.prev["kind"] == "c0":
            idx = self.prev["order"].index(param) * 3 + slot
            return dict(kind="c0", index=idx, n=len(self.prev["entries"]) // 32, claimed=claimed,
                        path=verde_merkle_audit_path(self.prev["entries"], idx))
        st = self.st
        j = st.adamw_node[param]
        nd = st.nodes[j]
        tab = self.prev["table"]
        ins = [tab[st.tensors[t].slot].tobytes() for t in nd.inputs]
        outs = [tab[st.tensors[t].slot].tobytes() for t in nd.outputs]
        blob = st.node_blob[st.node_offs[j]:st.node_offs[j + 1]].tobytes()
        nodes = self.prev["node_digests"].tobytes()
        return dict(kind="node", index=j, n=len(nodes) // 32, claimed=claimed, structure=blob, ins=ins, outs=outs,
                    slot=slot, path=verde_merkle_audit_path(nodes, j))

    # ---- Case 3 at chunk granularity
    def chunk_leaves(self, d: int, q: int) -> bytes:
        """R11 leaf hashes of the 4 KiB chunks of output q of node d (served to the referee)."""
        t = self.st.nodes[d].outputs[q]
        v = self.st.stash.get(t, self.st.tensors[t].view)
        return verde_chunk_leaves(v).cpu().numpy().tobytes()


def verify_checkpoint_proof(proof, h_start: bytes, program: GPT2Step, param: str, slot: int) -> bool:
    """Referee side of Case 2(a): does the proof place the claimed digest of the DISPUTED
    tensor (param, slot) in h_start?  Everything that selects the tree position comes
    from the referee's own program, never from the prover: the C0 entry index
    (parameter order x 3 + slot) and tree size, or the previous step's AdamW node of
    `param` (its index, static structure and the node-tree size) and the output slot."""
    if proof["kind"] == "c0":
        order = [n for n, _, _ in program.specs]
        if param not in order or proof["index"] != order.index(param) * 3 + slot or proof["n"] != 3 * len(order):
            return False
        leaf = verde_sha256(b"\x00" + proof["claimed"])
        return verde_merkle_verify_path(leaf, proof["index"], proof["n"], proof["path"], h_start)
    if proof["kind"] != "node":
        return False
    j = program.adamw_node.get(param)
    blob = program.node_blob[program.node_offs[j]:program.node_offs[j + 1]].tobytes() if j is not None else None
    if j is None or proof["index"] != j or proof["structure"] != blob or proof["slot"] != slot or \
            proof["n"] != len(program.nodes) or not 0 <= slot < len(proof["outs"]):
        return False
    if proof["outs"][slot] != proof["claimed"]:
        return False
    node_digest = verde_sha256(proof["structure"] + b"".join(proof["ins"]) + b"".join(proof["outs"]))
    leaf = verde_sha256(b"\x00" + node_digest)
    return verde_merkle_verify_path(leaf, proof["index"], proof["n"], proof["path"], h_start)


def opening_consistent(t: "Trainer", o: Opening) -> bool:
    """Does the opening of node o.index hash to the node digest the trainer committed in
    its sequence (R-NODE: SHA-256(structure || in-digests || out-digests))?"""
    seq = t.seq()
    if not 0 <= o.index < len(seq) // 32:
        return False
    dig = verde_sha256(o.structure + b"".join(o.in_digests) + b"".join(o.out_digests))
    return dig == seq[32 * o.index:32 * o.index + 32]


@dataclass
class Verdict:
    d: int
    case: int               # 1, 2 or 3; 0 = protocol violation (an opening or served
                            # tensor inconsistent with the trainer's own commitment)
    dishonest: int          # 0 or 1
    rounds: int             # subtree comparisons to find d
    detail: str
    chunk: int = -1         # Case 3: first differing 4 KiB chunk of the disputed output
    chunk_rounds: int = 0   # subtree comparisons to find it
    recomputed: int = 0     # output elements the referee recomputed


def phase2(t0: Trainer, t1: Trainer, h_end=None) -> tuple[int, int]:
    """Alg. 2: consistency check (line 7) + first diverging node (line 8).  h_end: the
    two ending hashes agreed in Phase 1 (default: the trainers' own claims)."""
    for i, t in enumerate((t0, t1)):
        claimed = t.root if h_end is None else h_end[i]
        if verde_merkle_root([t.seq()[i:i + 32] for i in range(0, len(t.seq()), 32)]) != claimed:
            raise ValueError("trainer's node sequence does not hash to its claimed checkpoint")
    return verde_first_divergence(t0.seq(), t1.seq())


def decide(t0: Trainer, t1: Trainer, d: int, rounds: int, program: GPT2Step, h_start=None,
           chunks=True) -> Verdict:
    o0, o1 = t0.open(d), t1.open(d)
    # every opening must match what the trainer committed (its node digest in the
    # sequence whose root Phase 2 checked); one that does not convicts its trainer
    # before any case logic can be steered by forged digests
    ok = [opening_consistent(t0, o0), opening_consistent(t1, o1)]
    if ok[0] != ok[1]:
        return Verdict(d, 0, 0 if not ok[0] else 1, rounds, "opening of the disputed node does not match the "
                       "trainer's committed node digest")
    if not ok[0]:
        raise RuntimeError("neither trainer's opening matches its committed node digest")
    nd = program.nodes[d]
    ref_struct = program.node_blob[program.node_offs[d]:program.node_offs[d + 1]].tobytes()
    # Case 1: graph structure (inputs, outputs, operator) -- the referee knows the program
    if o0.structure != o1.structure:
        bad = 0 if o0.structure != ref_struct else 1
        return Verdict(d, 1, bad, rounds, "node structure differs from the program")
    # Case 2(a): a checkpoint tensor differs -> membership proofs against h_start
    if nd.op == OP["PARAM_IN"]:
        q = next(i for i, (a, b) in enumerate(zip(o0.out_digests, o1.out_digests)) if a != b)
        param = program.tensors[nd.outputs[q]].name.split("/", 1)[1]
        ok = [verify_checkpoint_proof(t.prove_checkpoint(param, q), h_start, program, param, q) for t in (t0, t1)]
        if ok[0] == ok[1]:
            raise RuntimeError("membership proofs verify for neither / both trainers")
        return Verdict(d, 2, 1 if ok[0] else 0, rounds, f"checkpoint tensor {param}[{q}]: membership proof")
    # ... training data: the referee regenerates the batch from the dataset recipe
    if nd.op == OP["TOKENS_IN"]:
        toks = program.batch_tokens(nd.shard, t0.step_index).to(t0.st.dev)
        ref = bytes(verde_commit_tensors([toks]).cpu().numpy()[0])
        ok0, ok1 = o0.out_digests[0] == ref, o1.out_digests[0] == ref
        if ok0 == ok1:
            raise RuntimeError("dataset check matches neither / both trainers")
        return Verdict(d, 2, 1 if ok0 else 0, rounds, "training data differs from the dataset")
    # Case 2(b): an input hash differs -> the source node's emitted hash decides
    for q, (a, b) in enumerate(zip(o0.in_digests, o1.in_digests)):
        if a != b:
            src = program.tensors[nd.inputs[q]]
            # nodes before d have equal digests in both sequences; each trainer opens the
            # source node, and an opening must hash to that common node digest
            srcs = [t.open(src.producer) for t in (t0, t1)]
            sok = [opening_consistent(t, o) for t, o in zip((t0, t1), srcs)]
            if sok[0] != sok[1]:
                return Verdict(d, 0, 0 if not sok[0] else 1, rounds,
                               f"opening of source node {src.producer} does not match the committed digest")
            if not sok[0]:
                raise RuntimeError("neither trainer's opening of the source node matches its commitment")
            agreed = srcs[0].out_digests[src.pslot]
            bad = 0 if a != agreed else 1
            return Verdict(d, 2, bad, rounds, f"input {q} hash differs from source node {src.producer}")
    # Case 3: output hashes differ -> recompute on the agreed inputs
    step = t0.step_index
    # the agreed inputs: from t0, else from t1; a trainer that cannot serve tensors
    # matching the agreed input digests is convicted
    served = []
    for t in (t0, t1):
        try:
            served.append(_check_inputs(t.input_tensors(d), o0.in_digests))
        except ValueError:
            served.append(None)
    if (served[0] is None) != (served[1] is None):
        return Verdict(d, 0, 0 if served[0] is None else 1, rounds,
                       "served input tensors do not match the agreed input digests")
    if served[0] is None:
        raise RuntimeError("neither trainer served inputs matching the agreed input digests")
    agreed_in = served[0]
    if not chunks:
        outs = referee_recompute(program, d, agreed_in, o0.in_digests, step)
        mine = [bytes(x) for x in verde_commit_tensors(outs).cpu().numpy()]
        ok0, ok1 = mine == o0.out_digests, mine == o1.out_digests
        if ok0 == ok1:
            raise RuntimeError("referee recompute matches neither / both trainers")
        return Verdict(d, 3, 1 if ok0 else 0, rounds, f"recomputed {nd.name} (op {nd.op})",
                       recomputed=sum(o.numel() for o in outs))
    q = next(i for i, (a, b) in enumerate(zip(o0.out_digests, o1.out_digests)) if a != b)
    out = program.tensors[nd.outputs[q]].view
    dtype = 2 if out.dtype == torch.int32 else 1
    nbytes = out.numel() * out.element_size()
    leaves = []
    for t, o in ((t0, o0), (t1, o1)):
        L = t.chunk_leaves(d, q)
        # the served leaves must reproduce the trainer's committed output digest
        consistent = verde_tensor_digest_from_root(verde_merkle_root_hashed(L), dtype, out.shape, nbytes) == \
            o.out_digests[q]
        leaves.append(L if consistent else None)
    if (leaves[0] is None) != (leaves[1] is None):
        return Verdict(d, 3, 0 if leaves[0] is None else 1, rounds, "served chunk leaves inconsistent with digest")
    if leaves[0] is None:
        raise RuntimeError("neither trainer served chunk leaves consistent with its digest")
    c, crounds = verde_first_divergence(leaves[0], leaves[1], hashed=True)
    chunk, count = referee_recompute_chunk(program, d, agreed_in, o0.in_digests, q, c, step)
    h = verde_sha256(b"\x00" + chunk)
    ok0, ok1 = h == leaves[0][32 * c:32 * c + 32], h == leaves[1][32 * c:32 * c + 32]
    if ok0 == ok1:
        raise RuntimeError("referee chunk recompute matches neither / both trainers")
    return Verdict(d, 3, 1 if ok0 else 0, rounds, f"recomputed chunk {c} of output {q} of {nd.name} (op {nd.op})",
                   chunk=c, chunk_rounds=crounds, recomputed=count)


def _check_inputs(inputs, in_digests):
    ins = [t.clone() for t in inputs]
    got = [bytes(x) for x in verde_commit_tensors(ins).cpu().numpy()] if ins else []
    if got != list(in_digests):
        raise ValueError("provided input tensors do not match the agreed input hashes")
    return ins


def referee_recompute(program: GPT2Step, d: int, inputs, in_digests, step=None) -> list:
    """Re-run node d's single operator with RepOps on fresh buffers, after checking
    that the provided input tensors hash to the agreed input digests."""
    ins = _check_inputs(inputs, in_digests)
    return replay(program, program.nodes[d], ins, step)


def referee_recompute_chunk(program: GPT2Step, d: int, inputs, in_digests, q: int, c: int, step=None):
    """Bytes of 4 KiB chunk c of output q of node d, recomputing only what produces it:
    the covered output rows of a GEMM-type node (each output element depends only on
    its row of A and column of B, with the same ascending-K fold, so the rows alone
    give the same bits), the covered slice of an elementwise node, otherwise the
    whole operator.  Returns (chunk bytes, number of output elements computed)."""
    ins = _check_inputs(inputs, in_digests)
    nd = program.nodes[d]
    c_ = program.cfg
    out = program.tensors[nd.outputs[q]].view
    n = out.numel()
    e0, e1 = c * 1024, min(c * 1024 + 1024, n)  # float32 / int32 elements of the chunk
    op = nd.op
    x = ins
    if out.dim() == 2:
        cols = out.shape[1]
        r0, r1 = e0 // cols, (e1 - 1) // cols + 1
    sub = None
    if op == OP["LINEAR"]:
        sub = repops_gemm(x[0][r0:r1], x[1], epi=EPI_BIAS, bias=x[2])
    elif op == OP["LINEAR_DGRAD"]:
        sub = repops_gemm(x[0][r0:r1], x[1], transB=True)
    elif op == OP["LINEAR_WGRAD"]:
        sub = repops_gemm(x[0][:, r0:r1], x[1], transA=True)
    elif op == OP["LM_HEAD"]:
        sub = torch.zeros(r1 - r0, c_.vocab_ld, device=x[0].device)
        repops_gemm(x[0][r0:r1], x[1], transB=True, out=sub[:, :c_.vocab])
    elif op == OP["LM_DGRAD"]:
        sub = repops_gemm(x[0][r0:r1, :c_.vocab], x[1])
    elif op in (OP["RESIDUAL"], OP["GELU"], OP["GELU_BWD"]):
        flat = [t.reshape(-1)[e0:e1].contiguous() for t in x]
        y = {OP["RESIDUAL"]: lambda: repops_add(*flat), OP["GELU"]: lambda: repops_gelu(flat[0]),
             OP["GELU_BWD"]: lambda: repops_gelu_backward(*flat)}[op]()
        return y.cpu().numpy().tobytes(), e1 - e0
    if sub is not None:
        flat = sub.reshape(-1)[e0 - r0 * cols:e1 - r0 * cols]
        return flat.cpu().numpy().tobytes(), sub.numel()
    full = replay(program, nd, x, step)[q]
    return full.reshape(-1)[e0:e1].cpu().numpy().tobytes(), full.numel()


def replay(st: GPT2Step, nd, x, step=None):
    """One operator of the GPT-2 program, for one shard, from its input tensors
    (step: the step number, for AdamW's bias corrections)."""
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
    if op == OP["ATTENTION"]:      # R29: scores, causal softmax, PV as one operator
        qkv = x[0]
        S, P, att = E(H * T, T), E(H * T, T), E(T, d)
        repops_gemm_strided_batched(qkv, qkv, S, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T, sA=(0, hd),
                                    sB=(0, hd), sC=(0, T * T), batch=(1, H), transB=True, epi=EPI_SCALE, scale=sc,
                                    offB=d)
        repops_softmax(S, causal=True, out=P)
        repops_gemm_strided_batched(P, qkv, att, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d, sA=(0, T * T),
                                    sB=(0, hd), sC=(0, hd), batch=(1, H), offB=2 * d)
        return [att]
    if op == OP["ATTENTION_BWD"]:  # recomputes the probabilities from qkv (operator-internal)
        qkv, datt = x
        S, P, dP = E(H * T, T), E(H * T, T), E(H * T, T)
        repops_gemm_strided_batched(qkv, qkv, S, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T, sA=(0, hd),
                                    sB=(0, hd), sC=(0, T * T), batch=(1, H), transB=True, epi=EPI_SCALE, scale=sc,
                                    offB=d)
        repops_softmax(S, causal=True, out=P)
        repops_gemm_strided_batched(datt, qkv, dP, M=T, N=T, K=hd, lda=d, ldb=3 * d, ldc=T, sA=(0, hd),
                                    sB=(0, hd), sC=(0, T * T), batch=(1, H), transB=True, offB=2 * d)
        dS = repops_softmax_backward(P, dP, scale=sc)
        dq = E(T, 3 * d)
        kw = dict(M=T, N=hd, K=T, lda=T, ldc=3 * d, sA=(0, T * T), sC=(0, hd), batch=(1, H))
        repops_gemm_strided_batched(P, datt, dq, ldb=d, sB=(0, hd), transA=True, offC=2 * d, **kw)
        repops_gemm_strided_batched(dS, qkv, dq, ldb=3 * d, sB=(0, hd), offB=d, **kw)
        repops_gemm_strided_batched(dS, qkv, dq, ldb=3 * d, sB=(0, hd), transA=True, offC=d, **kw)
        return [dq]
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
        repops_adamw(p.view(-1), g.view(-1), m.view(-1), v.view(-1), st.step_no if step is None else step, c.lr,
                     c.beta1, c.beta2, c.adam_eps, c.wd, decay)
        return [p, m, v]
    raise NotImplementedError(f"replay of op {op}")


def dispute(cfg, fault_node: int, elem: int = 0, bit: int = 0, out_slot: int = 0, dishonest: int = 1,
            tokens_step: int = 0):
    """Run an honest and a dishonest trainer (1-bit flip after node `fault_node`'s
    launch) on the same checkpoint and batch; resolve with Phase 2 + decision."""
    honest = GPT2Step(cfg)
    honest.keep_committed = True
    honest.set_tokens(tokens_step)
    ck_h = (honest.params.clone(), honest.m.clone(), honest.v.clone())
    honest.run()
    cheat = GPT2Step(cfg)
    cheat.keep_committed = True
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


# ---------------------------------------------------------------------- Phase 1 (Alg. 1)
def checkpoint_entries(st: GPT2Step) -> bytes:
    """Entries of the starting-checkpoint tree C0: the digests of every parameter's
    (param, m, v) in parameter order -- exactly what step 1's PARAM_IN nodes emit."""
    views = []
    for name, _, _ in st.specs:
        views += [st.tensors[t].view for t in st.param_in[name]]
    return verde_commit_tensors(views).cpu().numpy().tobytes()


def checkpoint_steps(a: int, b: int, k: int) -> list:
    """k checkpoint steps spread evenly over (a, b], the last one b (every step if b-a <= k)."""
    if b - a <= k:
        return list(range(a + 1, b + 1))
    return sorted({a + -(-(b - a) * (i + 1) // k) for i in range(k)})


class TrainingRun:
    """One trainer's training run of the GPT-2 program from C0.  It logs the checkpoint
    hash (the step root, Fig. 2) and keeps the state at the steps it is asked to
    checkpoint, and re-executes a segment from any kept state (Alg. 1 recursion).
    Dishonest behaviours for tests: fault = (step, node, elem, bit, out_slot) flips one
    bit of a node output during that step; tamper = (step, param, elem, bit) flips a
    parameter bit right before that step (after the previous checkpoint was hashed)."""

    def __init__(self, cfg, fault=None, tamper=None):
        self.st = GPT2Step(cfg)
        self.st.keep_committed = True
        self.fault, self.tamper = fault, tamper
        self.reexecuted = 0
        entries = checkpoint_entries(self.st)
        self.log = {0: dict(kind="c0", root=verde_merkle_root([entries[i:i + 32] for i in range(0, len(entries), 32)]),
                            entries=entries, order=[n for n, _, _ in self.st.specs], state=self._snapshot())}

    def _snapshot(self):
        return tuple(t.clone() for t in (self.st.params, self.st.m, self.st.v))

    def _load(self, t):
        for dst, src in zip((self.st.params, self.st.m, self.st.v), self.log[t]["state"]):
            dst.copy_(src)
        self.st.state_changed()
        self.st.step_no = t

    def _step(self, t):
        st = self.st
        tam = self.tamper if self.tamper is not None and self.tamper[0] == t else None
        if tam is not None and tam[1] == "__tokens__":  # trains on (and commits) an altered batch
            c = st.cfg
            host = np.stack([synth.gpt2_tokens(c.vocab, c.seq, st.s0 + q, t - 1, c.seed) for q in range(st.S_loc)])
            host.reshape(-1)[tam[2]] ^= np.int32(1 << tam[3])
            st.set_tokens(host_tokens=host)
        else:
            st.set_tokens(t - 1)
        if tam is not None and tam[1] != "__tokens__":
            repops_flip_bit(st.pview(st.params, tam[1]).reshape(-1), tam[2], tam[3])
            st.state_changed()
        if self.fault is not None and self.fault[0] == t:
            _, node, elem, bit, slot = self.fault
            st.inject_fault(node, slot, elem, bit)
        st.run()
        st._fault = None
        root, nodes = st.step_root()
        return root, nodes

    def segment(self, a: int, b: int, keep, training=False):
        """Run steps a+1..b from the kept state at a; keep root + state at `keep` steps."""
        self._load(a)
        for t in range(a + 1, b + 1):
            root, nodes = self._step(t)
            if not training:
                self.reexecuted += 1
            if t in keep:
                self.log[t] = dict(kind="nodes", root=root, node_digests=nodes.copy(),
                                   table=self.st.digests_host.numpy().copy(), state=self._snapshot())
        return [self.log[t]["root"] for t in keep]

    def train(self, n_steps: int, k0: int):
        return self.segment(0, n_steps, checkpoint_steps(0, n_steps, k0), training=True)

    def trainer_for_step(self, t: int) -> Trainer:
        """Re-run step t from the kept state t-1 with every node committed (Phase 2)."""
        self._load(t - 1)
        ck = self._snapshot()
        self._step(t)
        self.reexecuted += 1
        return Trainer(self.st, ck, prev=self.log[t - 1], step_index=t)


@dataclass
class Phase1Result:
    step: int               # first diverging training step
    h_start: bytes          # agreed checkpoint hash before it
    h_end: tuple            # the two disputed checkpoint hashes after it
    levels: list            # (a, b, checkpoint steps, diverging index) per level


def phase1(r0: TrainingRun, r1: TrainingRun, n_steps: int, counts) -> Phase1Result | None:
    """Alg. 1 with multi-level checkpointing: level 0 uses the hashes logged while
    training (counts[0] checkpoints); each later level re-executes only the diverging
    segment with counts[l] checkpoints, until the segment is one step."""
    if r0.log[0]["root"] != r1.log[0]["root"]:
        raise ValueError("trainers disagree on the starting checkpoint C0")
    h_end = (r0.log[n_steps]["root"], r1.log[n_steps]["root"])
    if h_end[0] == h_end[1]:
        return None  # no dispute
    a, b, levels = 0, n_steps, []
    for lvl in range(64):
        k = counts[min(lvl, len(counts) - 1)]
        steps = checkpoint_steps(a, b, k)
        if lvl == 0:
            s0 = [r0.log[t]["root"] for t in steps]
            s1 = [r1.log[t]["root"] for t in steps]
        else:
            s0, s1 = r0.segment(a, b, steps), r1.segment(a, b, steps)
        if (s0[-1], s1[-1]) != h_end:
            raise ValueError("checkpoint sequence inconsistent with the disputed ending hashes")
        d = next(j for j in range(len(steps)) if s0[j] != s1[j])
        levels.append((a, b, steps, d))
        a, b = (steps[d - 1] if d else a), steps[d]
        h_end = (s0[d], s1[d])
        if b - a == 1:
            return Phase1Result(b, r0.log[a]["root"], h_end, levels)
    raise RuntimeError("phase 1 did not converge")


def resolve(r0: TrainingRun, r1: TrainingRun, n_steps: int, counts, chunks=True):
    """Full dispute over a training run: Phase 1 -> Phase 2 (with the line-7 check
    against Phase 1's ending hashes) -> decision.  Returns (Phase1Result, Verdict)."""
    p1 = phase1(r0, r1, n_steps, counts)
    if p1 is None:
        return None, None
    t0, t1 = r0.trainer_for_step(p1.step), r1.trainer_for_step(p1.step)
    d, rounds = phase2(t0, t1, h_end=p1.h_end)
    referee_program = GPT2Step(r0.st.cfg, structure_only=True)
    return p1, decide(t0, t1, d, rounds, referee_program, h_start=p1.h_start, chunks=chunks)
