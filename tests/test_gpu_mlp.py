"""Config 1 (BASELINE.json configs[0]): the 2-layer MLP data-parallel training step
on the GPU against the oracle step (oracle/mlp_step.py): every committed tensor
element by element (0 ULP), its R-TCOMMIT digest, the step root; the CUDA-graph
replay gives the same bits; and the config's 128^3 GEMM."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import mlp_step as omlp

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def run():
    from paper_2502_19405_b200.mlp import MLPConfig, MLPStep
    cfg = MLPConfig()
    st = MLPStep(cfg)
    st.run()
    torch.cuda.synchronize()
    ref, inp = omlp.run_step(cfg)
    return cfg, st, ref


def test_mlp_step_every_tensor_bit_exact(run):
    cfg, st, ref = run
    table = st.digests.cpu().numpy()
    for i, name in enumerate(st.names):
        r = np.ascontiguousarray(ref[name], np.float32)
        g = st.views[name].cpu().numpy()
        bad = np.flatnonzero(bits(g).ravel() != bits(r).ravel())
        assert bad.size == 0, f"{name}: {bad.size}/{g.size} elements differ"
        assert table[i].tobytes() == oracle.commit_tensor(r.reshape(g.shape)), name


def test_mlp_step_root(run):
    cfg, st, ref = run
    digs = [oracle.commit_tensor(np.ascontiguousarray(ref[n], np.float32).reshape(st.views[n].shape))
            for n in st.names]
    assert st.root() == oracle.merkle_root(digs)


def test_mlp_graph_replay_same_bits(run):
    cfg, st, ref = run
    root1 = st.root()
    st.capture()
    st.replay()
    torch.cuda.synchronize()
    assert st.root() == root1
    st.replay()
    torch.cuda.synchronize()
    assert st.root() == root1


def test_gemm_128_cubed():
    import paper_2502_19405_b200 as R
    A, B = synth.gemm_inputs(128, "bench")
    got = R.repops_gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    assert np.array_equal(bits(got), bits(oracle.gemm(A, B)))
