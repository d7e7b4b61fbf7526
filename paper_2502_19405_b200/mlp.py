"""Config 1 (BASELINE.json configs[0]): one data-parallel training step of a
2-layer MLP (Linear-ReLU-Linear-CE, width 256, batch 32, S = 8 shards of 4 rows)
on RepOps, with every operator output committed (R-TCOMMIT) and a step root.

  h = x W1 + b1   a = relu(h)   z = a W2 + b2   (loss, dz) = CE(z, y, 1/batch)
  da = dz W2^T    dh = relu'(h) da
  per shard s: gW2_s = a_s^T dz_s, gb2_s = SEQ(dz_s), gW1_s = x_s^T dh_s, gb1_s = SEQ(dh_s)
  g = R-TREE_S(g_0..g_7); AdamW (decay on W1, W2)

Row-wise operators run once over all 32 rows (rows are independent, so the bits
equal the per-shard computation of oracle/mlp_step.py); the per-shard weight
gradients are one strided-batched R-GEMM with K = 4 rows.  The step is ~20
launches and launch-latency bound, so `capture()` records it once into a CUDA
graph and `replay()` relaunches the whole step with one call.

Step root: RFC 6962 MTH over the committed tensors' digests in `self.names`
order (the config-1 analogue of the GPT-2 node root; reading R25).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import synth

from . import (EPI_BIAS, CommitPlan, repops_adamw, repops_cross_entropy, repops_gemm, repops_gemm_strided_batched,
               repops_relu, repops_relu_backward, repops_sum_cols_seq, repops_tree_sum, verde_merkle_root)

PARAMS = ("W1", "b1", "W2", "b2")


@dataclass
class MLPConfig:
    batch: int = 32
    width: int = 256
    classes: int = 256
    shards: int = 8
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.95
    adam_eps: float = 1e-8
    wd: float = 0.1
    seed: int = 0


class MLPStep:
    def __init__(self, cfg: MLPConfig = MLPConfig(), device="cuda"):
        assert cfg.batch % cfg.shards == 0
        self.cfg, self.dev = cfg, torch.device(device)
        B, D, Cc, S = cfg.batch, cfg.width, cfg.classes, cfg.shards
        self.R = B // S
        inp = synth.mlp_inputs(B, D, Cc, cfg.seed)
        self.shapes = {"W1": (D, D), "b1": (D,), "W2": (D, Cc), "b2": (Cc,)}
        self.off, o = {}, 0
        for n in PARAMS:
            self.off[n] = o
            o += int(np.prod(self.shapes[n]))
        self.P = o
        host = np.concatenate([inp[n].ravel() for n in PARAMS])
        self.params0 = torch.from_numpy(host).to(self.dev)
        self.params = self.params0.clone()
        self.m = torch.zeros(self.P, device=self.dev)
        self.v = torch.zeros(self.P, device=self.dev)
        self.x = torch.from_numpy(inp["x"]).to(self.dev)
        self.labels = torch.from_numpy(inp["labels"]).to(self.dev)
        E = lambda *s: torch.empty(*s, dtype=torch.float32, device=self.dev)  # noqa: E731
        self.h, self.a, self.da, self.dh = E(B, D), E(B, D), E(B, D), E(B, D)
        self.z, self.dz, self.loss = E(B, Cc), E(B, Cc), E(B)
        self.glocal = E(S, self.P)
        self.grad = E(self.P)
        self.step_no = 0
        # committed tensors, in root order (names follow oracle/mlp_step.py)
        R = self.R
        t = []
        for s in range(S):
            rows = slice(s * R, (s + 1) * R)
            for n, buf in (("h", self.h), ("a", self.a), ("z", self.z), ("loss", self.loss), ("dz", self.dz),
                           ("da", self.da), ("dh", self.dh)):
                t.append((f"s{s}/{n}", buf[rows]))
            for n in PARAMS:
                t.append((f"s{s}/grad/{n}", self.pview(self.glocal[s], n)))
        for n in PARAMS:
            t.append((f"grad/{n}", self.pview(self.grad, n)))
        for n in PARAMS:
            t += [(f"param'/{n}", self.pview(self.params, n)), (f"m'/{n}", self.pview(self.m, n)),
                  (f"v'/{n}", self.pview(self.v, n))]
        self.names = [n for n, _ in t]
        self.views = dict(t)
        self.digests = torch.zeros((len(t), 32), dtype=torch.uint8, device=self.dev)
        self.plan = CommitPlan([v for _, v in t], self.digests)
        self.graph = None

    def pview(self, buf, n):
        o = self.off[n]
        return buf[o:o + int(np.prod(self.shapes[n]))].view(*self.shapes[n])

    def reset(self):
        """Back to the initial parameters / optimizer state (step 1 again)."""
        self.params.copy_(self.params0)
        self.m.zero_()
        self.v.zero_()
        self.step_no = 0

    def _launch(self, step, stream=None):
        c, R, S, P = self.cfg, self.R, self.cfg.shards, self.P
        D, Cc = c.width, c.classes
        W = lambda n: self.pview(self.params, n)  # noqa: E731
        repops_gemm(self.x, W("W1"), epi=EPI_BIAS, bias=W("b1"), out=self.h, stream=stream)
        repops_relu(self.h, out=self.a, stream=stream)
        repops_gemm(self.a, W("W2"), epi=EPI_BIAS, bias=W("b2"), out=self.z, stream=stream)
        repops_cross_entropy(self.z, self.labels, scale=1.0 / c.batch, loss=self.loss, dlogits=self.dz,
                             stream=stream)
        repops_gemm(self.dz, W("W2"), transB=True, out=self.da, stream=stream)
        repops_relu_backward(self.h, self.da, out=self.dh, stream=stream)
        for wn, bn, A, G, M, N in (("W2", "b2", self.a, self.dz, D, Cc), ("W1", "b1", self.x, self.dh, D, D)):
            # per shard: g_W[s] = A_s^T G_s (K = R rows), into row s of glocal
            repops_gemm_strided_batched(A, G, self.glocal, M=M, N=N, K=R, lda=A.shape[1], ldb=N, ldc=N,
                                        sA=(R * A.shape[1], 0), sB=(R * N, 0), sC=(P, 0), batch=(S, 1),
                                        transA=True, offC=self.off[wn], stream=stream)
            repops_sum_cols_seq(G, nseg=S, out=self.glocal[:, self.off[bn]:], ldo=P, stream=stream)
        repops_tree_sum([self.glocal[s] for s in range(S)], out=self.grad, stream=stream)
        for n in PARAMS:
            repops_adamw(self.pview(self.params, n), self.pview(self.grad, n), self.pview(self.m, n),
                         self.pview(self.v, n), step, c.lr, c.beta1, c.beta2, c.adam_eps, c.wd,
                         len(self.shapes[n]) == 2, stream=stream)
        self.plan.run(stream=stream)

    def run(self):
        """One eager step (AdamW step counter = number of steps run so far + 1)."""
        self.step_no += 1
        self._launch(self.step_no)

    def capture(self):
        """Record reset() + step 1 into a CUDA graph; replay() reruns that whole step
        with one call.  (The AdamW step number is a launch argument baked into the
        graph, so the graph restarts from the initial state every time.)"""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm-up: lazy attributes, workspaces
            self.reset()
            self._launch(1, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        self.reset()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.reset()
            self._launch(1, stream=torch.cuda.current_stream())
        self.graph = g
        self.reset()
        return g

    def replay(self):
        self.graph.replay()
        self.step_no = 1

    def root(self) -> bytes:
        d = self.digests.cpu().numpy()
        return verde_merkle_root([bytes(r) for r in d])
