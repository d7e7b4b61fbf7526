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
              OP["SOFTMAX"]]
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
