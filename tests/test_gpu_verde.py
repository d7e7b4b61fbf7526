"""Verde dispute resolution (BASELINE config 5): a dishonest trainer flips one
low mantissa bit of one operator output during the GPT-2 step; the referee's
Phase 2 (Alg. 2) must find exactly that node by Merkle
descent, the decision must be Case 3, and the RepOps recompute of
the single operator must convict the dishonest trainer.  The recomputed output
is cross-checked against the CPU oracle (an independent implementation)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def _candidates(st):
    from paper_2502_19405_b200.gpt2 import OP
    skip = {OP["TOKENS_IN"], OP["EMBED"], OP["EMBED_BWD"], OP["PARAM_IN"], OP["TREE_SUM"], OP["ADAMW"]}
    return [nd.index for nd in st.nodes if nd.op not in skip and nd.label is not None]


@pytest.fixture(scope="module")
def tiny_program():
    from paper_2502_19405_b200.gpt2 import GPT2Config, GPT2Step
    return GPT2Config.tiny(), GPT2Step(GPT2Config.tiny(), structure_only=True)


def test_dispute_finds_injected_node_tiny(tiny_program):
    from paper_2502_19405_b200 import verde
    cfg, prog = tiny_program
    cands = _candidates(prog)
    pick = synth.integers(4242, 12, len(cands))
    n_nodes = len(prog.nodes)
    for q, ci in enumerate(pick):
        node = cands[int(ci)]
        nd = prog.nodes[node]
        numel = int(np.prod(prog.tensors[nd.outputs[0]].view.shape))
        elem = int(synth.integers(77 + q, 1, numel)[0])
        v = verde.dispute(cfg, node, elem=elem, bit=0, dishonest=q % 2)
        assert v is not None, nd.name
        assert v.d == node, f"found {v.d}, injected {node} ({nd.name})"
        assert v.case == 3
        assert v.dishonest == q % 2
        assert v.rounds <= 2 + int(np.ceil(np.log2(n_nodes)))


def _oracle_replay(cfg, op, xs):
    """Independent recompute of a few operator types with the CPU oracle."""
    from paper_2502_19405_b200.gpt2 import OP
    if op == OP["LINEAR"]:
        return [oracle.gemm(xs[0], xs[1], epi=1, bias=xs[2])]
    if op == OP["LAYERNORM"]:
        return list(oracle.layernorm(xs[0], xs[1], xs[2], cfg.ln_eps))
    if op == OP["GELU"]:
        return [oracle.gelu(xs[0])]
    if op == OP["RESIDUAL"]:
        return [oracle.add(xs[0], xs[1])]
    if op == OP["LINEAR_DGRAD"]:
        return [oracle.gemm(xs[0], xs[1], transB=True)]
    if op == OP["LINEAR_WGRAD"]:
        return [oracle.gemm(xs[0], xs[1], transA=True)]
    if op == OP["SOFTMAX"]:
        H, T = cfg.n_head, cfg.seq
        return [np.concatenate([oracle.softmax(xs[0][h * T:(h + 1) * T], causal=True) for h in range(H)])]
    if op in (OP["ATTENTION"], OP["ATTENTION_BWD"]):
        H, T, d = cfg.n_head, cfg.seq, cfg.d
        hd = d // H
        sc = float(np.float32(1.0 / np.sqrt(hd)))
        qkv = xs[0]
        c = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
        att = np.empty((T, d), np.float32)
        dq = np.empty((T, 3 * d), np.float32)
        for h in range(H):
            Q, K, Vh = (c(qkv[:, o + h * hd:o + (h + 1) * hd]) for o in (0, d, 2 * d))
            P = oracle.softmax(oracle.gemm(Q, K, transB=True, epi=2, scale=sc), causal=True)
            if op == OP["ATTENTION"]:
                att[:, h * hd:(h + 1) * hd] = oracle.gemm(P, Vh)
                continue
            dO = c(xs[1][:, h * hd:(h + 1) * hd])
            dS = oracle.softmax_backward(P, oracle.gemm(dO, Vh, transB=True), scale=sc)
            dq[:, 2 * d + h * hd:2 * d + (h + 1) * hd] = oracle.gemm(P, dO, transA=True)
            dq[:, h * hd:(h + 1) * hd] = oracle.gemm(dS, K)
            dq[:, d + h * hd:d + (h + 1) * hd] = oracle.gemm(dS, Q, transA=True)
        return [att if op == OP["ATTENTION"] else dq]
    return None


def test_referee_recompute_matches_oracle(tiny_program):
    from paper_2502_19405_b200 import verde
    from paper_2502_19405_b200.gpt2 import OP, GPT2Step
    cfg, prog = tiny_program
    st = GPT2Step(cfg)
    st.set_tokens(0)
    ck = (st.params.clone(), st.m.clone(), st.v.clone())
    st.run()
    tr = verde.Trainer(st, ck)
    wanted = [OP["LINEAR"], OP["LAYERNORM"], OP["GELU"], OP["RESIDUAL"], OP["LINEAR_DGRAD"], OP["LINEAR_WGRAD"],
              OP["ATTENTION"], OP["ATTENTION_BWD"]]
    done = set()
    for nd in st.nodes:
        if nd.op in wanted and nd.op not in done and nd.shard == 3:
            ins = tr.input_tensors(nd.index)
            outs = verde.referee_recompute(st, nd.index, ins, tr.open(nd.index).in_digests)
            gpu_dig = [bytes(x) for x in verde.verde_commit_tensors(outs).cpu().numpy()]
            assert gpu_dig == tr.open(nd.index).out_digests, nd.name
            ref = _oracle_replay(cfg, nd.op, [t.cpu().numpy() for t in ins])
            assert [oracle.commit_tensor(r.reshape(o.shape)) for r, o in zip(ref, outs)] == gpu_dig, nd.name
            done.add(nd.op)
    assert done == set(wanted)


def test_dispute_full_gpt2_mid_network():
    from paper_2502_19405_b200 import verde
    from paper_2502_19405_b200.gpt2 import GPT2Config, GPT2Step
    cfg = GPT2Config()
    prog = GPT2Step(cfg, structure_only=True)
    node = next(nd.index for nd in prog.nodes if nd.name == "s5/h6/fc")
    v = verde.dispute(cfg, node, elem=123457, bit=0)
    assert v.d == node and v.case == 3 and v.dishonest == 1
    assert v.rounds <= 14  # log2(3596) ~ 11.8 levels + root comparison


# ---------------------------------------------------------------------- Phase 1 + Case 2(a) + chunk-level Case 3
def _node_named(prog, name):
    return next(nd.index for nd in prog.nodes if nd.name == name)


def test_phase1_multilevel_then_phase2_chunk_decision(tiny_program):
    """12-step run, a 1-bit fault in step 7: Phase 1 narrows 12 -> 3 -> 2 -> 1 steps with
    re-execution of the diverging segments only; Phase 2 finds the node; the referee
    recomputes just the 4 KiB chunk holding the flipped element."""
    from paper_2502_19405_b200 import verde
    cfg, prog = tiny_program
    node = _node_named(prog, "s3/h1/fc")
    numel = int(np.prod(prog.tensors[prog.nodes[node].outputs[0]].view.shape))
    elem = numel - 5
    for dishonest in (0, 1):
        runs = [verde.TrainingRun(cfg), verde.TrainingRun(cfg, fault=(7, node, elem, 0, 0))]
        if dishonest == 0:
            runs.reverse()
        for r in runs:
            r.train(12, 4)
        p1, v = verde.resolve(runs[0], runs[1], 12, counts=(4, 2))
        assert p1.step == 7
        assert [lv[:2] for lv in p1.levels] == [(0, 12), (6, 9), (6, 8)]
        assert all(r.reexecuted == 3 + 2 + 1 for r in runs)  # levels 1, 2 + the Phase 2 step
        assert v.d == node and v.case == 3 and v.dishonest == dishonest
        assert v.chunk == elem // 1024
        out = prog.tensors[prog.nodes[node].outputs[0]].view
        assert v.recomputed <= out.shape[1] * (1024 // out.shape[1] + 2) < out.numel()


@pytest.mark.parametrize("tamper_step", [1, 4])
def test_case2a_checkpoint_membership_proof(tiny_program, tamper_step):
    """A trainer silently alters one weight between checkpoints: the first diverging
    node is that parameter's PARAM_IN; only the honest trainer can prove membership of
    its digest in h_start (C0 tree for step 1, the previous step's AdamW node later)."""
    from paper_2502_19405_b200 import verde
    cfg, prog = tiny_program
    runs = [verde.TrainingRun(cfg), verde.TrainingRun(cfg, tamper=(tamper_step, "h0.attn.w", 17, 3))]
    for r in runs:
        r.train(6, 3)
    p1, v = verde.resolve(runs[0], runs[1], 6, counts=(3, 2))
    assert p1.step == tamper_step
    assert v.case == 2 and v.dishonest == 1 and "membership" in v.detail
    assert v.d == prog.param_in_node["h0.attn.w"]


def test_case2_training_data_checked_against_dataset(tiny_program):
    from paper_2502_19405_b200 import verde
    cfg, prog = tiny_program
    runs = [verde.TrainingRun(cfg, tamper=(3, "__tokens__", 40, 0)), verde.TrainingRun(cfg)]
    for r in runs:
        r.train(4, 4)
    p1, v = verde.resolve(runs[0], runs[1], 4, counts=(4,))
    assert p1.step == 3 and v.case == 2 and v.dishonest == 0 and "dataset" in v.detail
    assert prog.nodes[v.d].op == 2  # TOKENS_IN


def test_chunk_recompute_equals_full_replay(tiny_program):
    """The referee's partial recompute gives exactly the bytes of the full operator."""
    from paper_2502_19405_b200 import verde
    from paper_2502_19405_b200.gpt2 import GPT2Step
    cfg, prog = tiny_program
    st = GPT2Step(cfg)
    st.set_tokens(0)
    ck = (st.params.clone(), st.m.clone(), st.v.clone())
    st.run()
    tr = verde.Trainer(st, ck)
    for name in ("s2/h0/qkv", "s5/head/lm_head", "s1/h1/fc2_dgrad", "s0/h1/fc_wgrad", "s6/h0/gelu", "s4/h1/res2",
                 "s3/h0/attention", "s2/h1/attention_bwd"):
        d = _node_named(prog, name)
        o = tr.open(d)
        ins = tr.input_tensors(d)
        full = verde.referee_recompute(prog, d, ins, o.in_digests, 1)[0].reshape(-1).cpu().numpy().tobytes()
        n_chunks = (len(full) + 4095) // 4096
        for c in sorted({0, n_chunks // 2, n_chunks - 1}):
            got, count = verde.referee_recompute_chunk(prog, d, ins, o.in_digests, 0, c, 1)
            assert got == full[4096 * c:4096 * (c + 1)], (name, c)


# ---------------------------------------------------------------- dishonest openings / proofs / inputs
def _two_trainers(cfg, node):
    """an honest trainer and one whose node `node` output has a flipped bit"""
    from paper_2502_19405_b200 import verde
    from paper_2502_19405_b200.gpt2 import GPT2Step
    out = []
    for fault in (False, True):
        st = GPT2Step(cfg)
        st.keep_committed = True
        st.set_tokens(0)
        ck = (st.params.clone(), st.m.clone(), st.v.clone())
        if fault:
            st.inject_fault(node, 0, 3, 0)
        st.run()
        out.append(verde.Trainer(st, ck))
    return out


def test_forged_opening_convicts_the_forger(tiny_program):
    """A dishonest trainer opens the disputed node with the honest trainer's digests
    (so the openings look equal): its opening does not hash to the node digest it
    committed, and the referee convicts it before any case logic (ADVICE: an honest
    trainer must never be convicted)."""
    from paper_2502_19405_b200 import verde
    cfg, prog = tiny_program
    node = _node_named(prog, "s2/h1/fc")
    honest, cheat = _two_trainers(cfg, node)

    class Forger(verde.Trainer):
        def open(self, d):
            return honest.open(d)

    forger = Forger.__new__(Forger)
    forger.__dict__.update(cheat.__dict__)
    for dishonest, (t0, t1) in ((1, (honest, forger)), (0, (forger, honest))):
        d, rounds = verde.phase2(t0, t1)
        assert d == node
        v = verde.decide(t0, t1, d, rounds, prog)
        assert v.case == 0 and v.dishonest == dishonest, v


def test_forged_source_opening_in_case2b(tiny_program):
    """Case 2(b): the dishonest trainer claims a different input digest for node d and
    opens the source node with that same forged digest -- both openings are checked
    against its commitments, so it is convicted (not the honest trainer)."""
    from paper_2502_19405_b200 import verde
    cfg, prog = tiny_program
    node = _node_named(prog, "s2/h1/gelu")           # input: s2/h1/fc (source node)
    src = prog.tensors[prog.nodes[node].inputs[0]].producer
    honest, cheat = _two_trainers(cfg, _node_named(prog, "s2/h1/fc"))
    forged = b"\xab" * 32

    class Liar(verde.Trainer):
        def open(self, d):
            o = honest.open(d)
            if d == node:
                o.in_digests = [forged]
            if d == src:
                o.out_digests = [forged]
            return o

        def seq(self):
            return honest.seq()   # claims the honest sequence, so node d is reached with equal digests

    liar = Liar.__new__(Liar)
    liar.__dict__.update(cheat.__dict__)
    v = verde.decide(honest, liar, node, 0, prog)
    assert v.case == 0 and v.dishonest == 1


def test_checkpoint_proof_is_bound_to_the_disputed_tensor(tiny_program):
    """Case 2(a) verifier: a valid proof for one (param, slot) does not verify for
    another parameter, another slot, or with a prover-chosen node index (e.g. the
    previous step's PARAM_IN node instead of its AdamW node)."""
    from paper_2502_19405_b200 import verde
    cfg, prog = tiny_program
    run = verde.TrainingRun(cfg)
    run.train(2, 2)
    t2 = run.trainer_for_step(2)
    h1 = run.log[1]["root"]
    proof = t2.prove_checkpoint("h0.attn.w", 0)
    assert verde.verify_checkpoint_proof(proof, h1, prog, "h0.attn.w", 0)
    assert not verde.verify_checkpoint_proof(proof, h1, prog, "h0.fc.w", 0)
    assert not verde.verify_checkpoint_proof(proof, h1, prog, "h0.attn.w", 1)
    stale = dict(proof)
    j = prog.param_in_node["h0.attn.w"]
    stale["index"] = j
    stale["structure"] = prog.node_blob[prog.node_offs[j]:prog.node_offs[j + 1]].tobytes()
    assert not verde.verify_checkpoint_proof(stale, h1, prog, "h0.attn.w", 0)
    # step-1 proofs from the C0 tree are bound to (param order, slot) the same way
    t1 = run.trainer_for_step(1)
    p0 = t1.prove_checkpoint("h1.fc.b", 2)
    h0 = run.log[0]["root"]
    assert verde.verify_checkpoint_proof(p0, h0, prog, "h1.fc.b", 2)
    assert not verde.verify_checkpoint_proof(p0, h0, prog, "h1.fc.w", 2)
    assert not verde.verify_checkpoint_proof(dict(p0, n=p0["n"] + 1), h0, prog, "h1.fc.b", 2)


def test_case3_trainer_serving_wrong_inputs_is_convicted(tiny_program):
    """Case 3 takes the agreed inputs from t0, else t1; a trainer whose served tensors
    do not hash to the agreed input digests is convicted (the dispute still resolves)."""
    from paper_2502_19405_b200 import verde
    cfg, prog = tiny_program
    node = _node_named(prog, "s1/h0/fc2")
    honest, cheat = _two_trainers(cfg, node)

    class BadServer(verde.Trainer):
        def input_tensors(self, d):
            xs = [x.clone() for x in super().input_tensors(d)]
            xs[0].view(-1)[0] += 1.0
            return xs

    bad = BadServer.__new__(BadServer)
    bad.__dict__.update(cheat.__dict__)
    d, rounds = verde.phase2(bad, honest)
    assert d == node
    v = verde.decide(bad, honest, d, rounds, prog)
    assert v.case == 0 and v.dishonest == 0
    # served correctly by t0, the normal Case 3 decision follows
    v = verde.decide(cheat, honest, d, rounds, prog)
    assert v.case == 3 and v.dishonest == 0
