"""bench.py -- RepOps / Verde hot path on B200 (DESIGN.md §7 "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl repops|reference] [--workload gpt2|gemm]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N --steps K --warmup W

Default workload "gpt2" (BASELINE.json configs[2] + [4]): one GPT-2 small (124M)
training step, batch 8 x seq 512, as S = 8 data-parallel shards spread over the
N GPUs: forward, backward, canonical R-TREE_S gradient combine (NCCL all-gather
of partials for N > 1), AdamW, a Verde commitment (SHA-256 / RFC 6962) of every
operator output, the node digests and the step's Merkle root.  This is one pass
of every §8(a) row.  value = algorithmic matmul TFLOP of the step / step time;
ms_per_step is the GPT-2 step time (the metric's second half).

The GEMM sweep of configs[1] (square 1024..8192, M-sharded) runs in the same
invocation and is reported under "gemm_sweep"; --workload gemm makes it the
headline line instead.

Prints ONE JSON line (rank 0).  The oracle (CPU test infrastructure) is only
run by the cpu_baseline leg (rank 0, N = 1) and by --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "RepOps FP32 GEMM TFLOP/s & GPT-2 step time, bit-identical at 1-8 GPUs"
SIZES = (1024, 2048, 4096, 8192)
SWEEP_FLOPS = sum(2 * n ** 3 for n in SIZES)


def fp32_peak_tflops(mhz: float, sms: int = 148) -> float:
    """FP32 CUDA-core FMA peak: SMs x 128 FP32 lanes x 2 flop x clock."""
    return sms * 128 * 2 * mhz * 1e6 / 1e12


# SHA-256 leaf compression (sha256.o, cuobjdump -sass): the all-ALU form is 673 SHF + 352
# LOP3 + 244 IADD3 + 16 PRMT + 2 ISETP per 64-byte block; the default leaf kernel (mode 3)
# moves the round / schedule adds and the schedule shifts to IMAD on the FMA pipe, leaving
# 949 ALU ops per block (the function-wide ALU count drops by 338).  The ALU pipe retires
# 16 lanes / clk / SMSP (rt = 2, B300_MICROARCH "Pipe rates"): the commit's roofline is
# ALU issue, not HBM.
SHA_ALU_OPS_PER_64B = 949


def sha_alu_peak_gbs(mhz: float, sms: int = 148) -> float:
    """bytes/s the ALU pipe allows for SHA-256 leaves: SMs x 64 lanes x clock / ALU ops per byte."""
    return sms * 4 * 16 * mhz * 1e6 / (SHA_ALU_OPS_PER_64B / 64) / 1e9


def profiled_gemm_traffic():
    """DRAM bytes per R-GEMM launch, averaged over one GPT-2 step's GEMM launches in
    the committed ncu launch list (profiles/, tools/profile_round.sh); None if absent."""
    import csv
    path = os.path.join(ROOT, "profiles", "r02_gpt2_step_launches.csv")
    try:
        rows = list(csv.reader(open(path)))
        h = rows[0]
        ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
        byts, ids = 0.0, set()
        for r in rows[1:]:
            if ("gemm_kernel" in r[ki] or "gemm_tn_kernel" in r[ki]) and r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                byts += float(r[vi].replace(",", ""))
                ids.add(r[0])
        return byts / len(ids) if ids else None
    except Exception:
        return None


def measured_hbm_gbs() -> float:
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the timed region runs."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------- distributed
def dist_init():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # timing scalar only (not the data path)
    return float(t.item())


# ---------------------------------------------------------------------- GEMM sweep workload
class GemmSweep:
    """BASELINE config 2: square R-GEMMs 1024..8192, M-sharded, each output committed."""

    def __init__(self, rank, world, device):
        import torch

        import paper_2502_19405_b200 as R
        import synth
        self.R, self.torch = R, torch
        self.rank, self.world = rank, world
        self.items = []
        for n in SIZES:
            A, B = synth.gemm_inputs(n, "bench")
            rows = n // world
            Ar = np.ascontiguousarray(A[rank * rows:(rank + 1) * rows])
            hA = torch.from_numpy(Ar).pin_memory()
            hB = torch.from_numpy(B).pin_memory()
            self.items.append(dict(n=n, rows=rows, hA=hA, hB=hB, A=hA.to(device), B=hB.to(device),
                                   C=torch.empty((rows, n), dtype=torch.float32, device=device)))
        self.roots = torch.empty((len(SIZES), 32), dtype=torch.uint8, device=device)
        self.plan = R.CommitPlan([it["C"] for it in self.items], self.roots, modes=[1] * len(SIZES))
        self.flops = SWEEP_FLOPS

    def step(self):
        for it in self.items:
            self.R.repops_gemm(it["A"], it["B"], out=it["C"])
        self.plan.run()

    def e2e_step(self):
        for it in self.items:
            it["A"].copy_(it["hA"], non_blocking=True)
            it["B"].copy_(it["hB"], non_blocking=True)
        self.step()
        return self.roots.to("cpu")

    @property
    def h2d_bytes(self):
        return sum(it["hA"].numel() * 4 + it["hB"].numel() * 4 for it in self.items)

    d2h_bytes = len(SIZES) * 32

    def digests(self):
        """Tensor digests of the full C matrices (identical at every world size)."""
        from paper_2502_19405_b200.dist import all_gather_rows
        parts = all_gather_rows(self.roots, self.world).cpu().numpy()
        out = []
        for q, it in enumerate(self.items):
            n = it["n"]
            sub = b"".join(parts[r, q].tobytes() for r in range(self.world))
            out.append(self.R.verde_digest_from_subroots(sub, self.R.F32, (n, n), n * n * 4).hex())
        return out


# ---------------------------------------------------------------------- GPT-2 workload
class GPT2Train:
    """mode "every" (configs[2] + [4], the headline): every operator output committed,
    node digests and the step root every step.  mode "checkpoint" (configs[2] alone, as
    Verde's trainers run between disputes, "log checkpoints only at specified
    steps"): no per-operator commitments; every CKPT_EVERY-th step commits the training
    state (param, m, v of every parameter) and its RFC 6962 root."""

    CKPT_EVERY = 10

    def __init__(self, rank, world, device, pg=None, commit=True, overlap=True, combine="p2p", mode="every"):
        from paper_2502_19405_b200.gpt2 import GPT2Config, GPT2Step
        # G > 1: R-TREE_S as one fused peer-memory kernel per rank (CUDA IPC over NVLink)
        self.st = GPT2Step(GPT2Config(), rank=rank, world=world, device=device, pg=pg, combine=combine)
        self.st.overlap_commits = overlap
        self.commit = commit
        self.mode = mode
        self.n_steps = 0
        self.st.set_tokens(0)
        self.flops = self.st.flops_per_step()
        self.root = None

    def step(self):
        with self.stream_ctx():
            if self.mode == "checkpoint":
                self.st.run(commit=False)
                self.n_steps += 1
                if self.commit and self.n_steps % self.CKPT_EVERY == 0:
                    self.st.checkpoint_commit()
                return
            # the tail commits + root of step n run beside step n+1's forward (no host sync)
            self.st.run(commit=self.commit, join=False)
            self.st.device_root(sync=False)   # C2 gather + node digests + step root on the GPU; 32 B D2H

    def stream_ctx(self):
        """the step's main stream: high priority (REPOPS_PRIO=0 turns it off); the commit side
        stream keeps the default, lowest priority, so the block scheduler prefers the step's
        kernels and SHA-256 CTAs fill the gaps they leave (92.5 -> 91.5 ms, same root)"""
        import contextlib

        import torch
        if os.environ.get("REPOPS_PRIO", "1") != "1":
            return contextlib.nullcontext()
        if not hasattr(self, "_hi"):
            self._hi = torch.cuda.Stream(priority=-1)
            self._hi.wait_stream(torch.cuda.current_stream())
        return torch.cuda.stream(self._hi)

    @staticmethod
    def isolated_gemm(wl, world, local, steps=2):
        import torch
        commit = wl.commit
        wl.commit = False
        try:
            for _ in range(1):
                wl.step()
            torch.cuda.synchronize()
            _, tot, _, _ = timed(wl, steps, world, local)
        finally:
            wl.commit = commit
        g_ms, g_fl, _ = tot.get("gemm", (0.0, 0, 0))
        g_ms = max_over_ranks(g_ms, world)
        return g_fl / (g_ms * 1e-3) / 1e12 if g_ms else None

    def join(self):
        with self.stream_ctx():
            self.st.join()
        if hasattr(self, "_hi"):
            import torch
            torch.cuda.current_stream().wait_stream(self._hi)  # the timing events see the step's work
        if self.mode == "every":
            self.root = self.st.root_bytes()

    def e2e_step(self):
        self.st.set_tokens(self.st.step_no)    # H2D of this step's batch from pinned host memory
        if self.mode == "checkpoint":
            self.st.run(commit=False)
            self.n_steps += 1
            if self.commit and self.n_steps % self.CKPT_EVERY == 0:
                self.st.checkpoint_commit()
                self.root = self.st.checkpoint_root()   # 148 x 3 digests D2H, root on the host
            return self.st.loss(), self.root
        self.st.run(commit=self.commit)
        self.root = self.st.device_root()      # 32 B D2H
        return self.st.loss(), self.root       # D2H of the loss

    @property
    def h2d_bytes(self):
        return self.st.h2d_bytes

    @property
    def d2h_bytes(self):
        return 32 + 4  # step root + loss


class LlamaPrefillBench:
    """BASELINE config 4: Llama-3-8B-shaped FP32 prefill, 2048 tokens, TP N-split over the
    N GPUs (8 column blocks), every operator output committed, pass root on the GPU."""

    def __init__(self, rank, world, device, pg=None):
        from paper_2502_19405_b200.llama import LlamaConfig, LlamaPrefill
        self.st = LlamaPrefill(LlamaConfig(), rank=rank, world=world, device=device, pg=pg)
        self.st.load_weights()
        self.st.set_tokens()
        self.flops = self.st.flops()
        self.root = None

    def step(self):
        with GPT2Train.stream_ctx(self):   # high-priority pass stream, commits on the low-priority side
            self.st.run()
            self.root = self.st.device_root()   # waits for the pass (host)

    def e2e_step(self):
        self.st.set_tokens()
        self.step()
        return self.root

    h2d_bytes = 2048 * 4
    d2h_bytes = 32


def ffma2_probe():
    try:
        import paper_2502_19405_b200 as R
        return R.repops_ffma2_probe_tflops()
    except Exception:  # noqa: BLE001 -- diagnostic only
        return None


def verde_dispute_bench(trials=10, with_oracle=True):
    """BASELINE config 5, the dispute half: an honest and a dishonest trainer of the full
    GPT-2 124M step (the dishonest one flips bit 0 of one element of one operator output,
    node and element drawn from the seeded generator) -- Verde Phase 2 (Alg. 2: line-7
    consistency, Merkle descent to the first diverging node) and the decision (Case 3 at
    4 KiB-chunk granularity, the referee recomputing only the rows of the disputed chunk).
    Per trial: found == injected node, case, convicted party, descent rounds, wall time of
    phase 2 + decision (the two trainers' steps are outside it).  Beside it: the oracle's
    SHA-256 commitment rate on one host core."""
    import torch

    import synth
    from paper_2502_19405_b200 import verde
    from paper_2502_19405_b200.gpt2 import OP, GPT2Config, GPT2Step
    cfg = GPT2Config()
    honest = GPT2Step(cfg)
    honest.keep_committed = True
    honest.set_tokens(0)
    ck = (honest.params.clone(), honest.m.clone(), honest.v.clone())
    honest.run()
    th = verde.Trainer(honest, ck)
    cheat = GPT2Step(cfg)
    cheat.keep_committed = True
    skip = {OP["TOKENS_IN"], OP["EMBED"], OP["EMBED_BWD"], OP["PARAM_IN"], OP["TREE_SUM"], OP["ADAMW"]}
    cands = [nd.index for nd in cheat.nodes if nd.op not in skip and nd.label is not None]
    picks = synth.integers(5150, trials, len(cands))
    rows, times = [], []
    for q in range(trials):
        cheat.params.copy_(ck[0])
        cheat.m.copy_(ck[1])
        cheat.v.copy_(ck[2])
        cheat.step_no = 0
        cheat.state_changed()
        cheat.set_tokens(0)
        node = cands[int(picks[q])]
        nd = cheat.nodes[node]
        numel = cheat.tensors[nd.outputs[0]].view.numel()
        elem = int(synth.integers(5151 + q, 1, numel)[0])
        cheat.inject_fault(node, 0, elem, 0)
        cheat.run()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tc = verde.Trainer(cheat, ck)
        d, rnd = verde.phase2(th, tc)
        v = verde.decide(th, tc, d, rnd, honest)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        rows.append(dict(node=nd.name, found=v.d == node, case=v.case, convicted=v.dishonest, rounds=v.rounds,
                         chunk_rounds=v.chunk_rounds, recomputed=v.recomputed))
    cheat._fault = None
    out = {"trials": trials, "nodes": len(cheat.nodes),
           "found": sum(r["found"] for r in rows), "case3": sum(r["case"] == 3 for r in rows),
           "dishonest_convicted": sum(r["convicted"] == 1 for r in rows),
           "rounds_max": max(r["rounds"] for r in rows), "chunk_rounds_max": max(r["chunk_rounds"] for r in rows),
           "resolve_s_median": sorted(times)[len(times) // 2], "resolve_s_max": max(times),
           "trials_detail": rows,
           "config": "GPT-2 124M step (configs[2]) honest vs one-bit-faulted trainer, Phase 2 + Case-3 decision "
                     "(configs[4]); fault node / element from synth.integers(5150 / 5151+q)"}
    del honest, cheat, th
    torch.cuda.empty_cache()
    if with_oracle:
        import oracle
        a = synth.uniform(5152, 8 * 2 ** 20)          # 32 MiB
        t0 = time.perf_counter()
        oracle.commit_tensor(a)
        dt = time.perf_counter() - t0
        out["oracle_sha256_gbs"] = a.nbytes / dt / 1e9
        out["oracle_note"] = "oracle R-TCOMMIT (SHA-256 leaves + RFC 6962 tree + header) of 32 MiB, 1 host core"
    return out


def mlp_extra(with_oracle=True, reps=200):
    """BASELINE config 1 (configs[0]): the 2-layer MLP DP step (fwd, bwd, R-TREE_S,
    AdamW, commit of all 104 outputs) -- launch-latency bound, so reported in us per
    step: eager, and as one CUDA-graph replay; plus the config's 128^3 R-GEMM; beside
    the full oracle step on one host core (seconds)."""
    import torch

    import paper_2502_19405_b200 as R
    import synth
    from paper_2502_19405_b200.mlp import MLPConfig, MLPStep

    def us(fn, n):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3

    st = MLPStep(MLPConfig())
    l0 = R.launch_count()
    st.run()
    launches = R.launch_count() - l0
    eager = us(lambda: (st.reset(), st.run()), reps)
    st.capture()
    graph = us(st.replay, reps)
    torch.cuda.synchronize()
    root = st.root().hex()
    A, B = (torch.from_numpy(t).cuda() for t in synth.gemm_inputs(128, "bench"))
    C = torch.empty(128, 128, device="cuda")
    g128 = us(lambda: R.repops_gemm(A, B, out=C), reps)   # per Python-level call (host-bound)
    # device time per launch: 50 back-to-back launches captured in one CUDA graph
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        R.repops_gemm(A, B, out=C)
        with torch.cuda.graph(g, stream=side):
            for _ in range(50):
                R.repops_gemm(A, B, out=C)
    torch.cuda.synchronize()
    g128_dev = us(g.replay, 20) / 50
    res = {"us_per_step_graph": graph, "us_per_step_eager": eager, "gpu_launches": launches,
           "gemm128_us": g128, "gemm128_device_us": g128_dev, "root": root,
           "config": "Linear-ReLU-Linear-CE, width 256, batch 32 = 8 shards x 4 rows, AdamW, every output "
                     "committed (BASELINE configs[0])"}
    if with_oracle:
        import oracle
        from oracle import mlp_step as omlp
        oracle.lib()
        t0 = time.perf_counter()
        omlp.run_step(MLPConfig())
        res["oracle_s_per_step"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        a_, b_ = synth.gemm_inputs(128, "bench")
        oracle.gemm(a_, b_)
        res["oracle_gemm128_s"] = time.perf_counter() - t0
    return res


# ---------------------------------------------------------------------- cuBLAS context
# the distinct R-GEMM shapes of one GPT-2 step (tools/gpt2_gemm_shapes.py): layout, M, N, K, batch
GPT2_GEMM_SHAPES = [("TN", 4096, 2304, 768, 1), ("TN", 4096, 768, 768, 1), ("TN", 4096, 3072, 768, 1),
                    ("TN", 4096, 768, 3072, 1), ("TN", 4096, 50304, 768, 1), ("TN", 4096, 768, 2304, 1),
                    ("TN", 4096, 768, 50257, 1), ("TN", 768, 2304, 512, 8), ("TN", 768, 768, 512, 8),
                    ("TN", 768, 3072, 512, 8), ("TN", 3072, 768, 512, 8), ("TN", 50257, 768, 512, 8),
                    ("NT", 512, 512, 64, 96), ("NN", 512, 64, 512, 96), ("TN", 512, 64, 512, 96)]


def ulp_stats(got, ref):
    """(elements differing, max ULP distance) of two float32 tensors (same-sign distance in
    units of the last place; a sign mismatch counts as 2^31)."""
    import torch
    a = got.contiguous().view(torch.int32).to(torch.int64)
    b = ref.contiguous().view(torch.int32).to(torch.int64)
    a = torch.where(a < 0, -(a & 0x7FFFFFFF), a)   # sign-magnitude -> ordered integers
    b = torch.where(b < 0, -(b & 0x7FFFFFFF), b)
    d = (a - b).abs()
    return int((d != 0).sum().item()), int(d.max().item()) if d.numel() else 0


def cublas_context():
    """Non-reproducible cuBLAS FP32 SGEMM (torch.mm / bmm, TF32 off) on the same shapes as
    the R-GEMM -- the paper's own overhead comparison (RepOps vs torch::mm) --
    with the ULP differences of its output from the R-GEMM's (which equals the oracle bit
    for bit: tests/test_gpu_parity.py, tests/test_gpu_gpt2_referee.py)."""
    import torch

    import paper_2502_19405_b200 as R
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False

    def ms(fn, iters=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / iters

    gen = torch.Generator(device="cuda").manual_seed(0)
    out = {}
    shapes = [("NN", n, n, n, 1) for n in SIZES] + GPT2_GEMM_SHAPES
    for lay, M, N, K, b in shapes:
        ta, tb = lay[0] == "T", lay[1] == "T"
        # rows padded to a multiple of 4 floats, as the step's buffers are (e.g. the logits'
        # ld 50304 for V = 50257): 16-byte aligned rows for both libraries
        pad = lambda r, c: (torch.rand((b, r, (c + 3) // 4 * 4), device="cuda", generator=gen) * 2 - 1)[:, :, :c]  # noqa: E731
        A = pad(K, M) if ta else pad(M, K)
        B = pad(N, K) if tb else pad(K, N)
        Cr = torch.empty((b, M, N), device="cuda")
        opA = A.transpose(1, 2) if ta else A
        opB = B.transpose(1, 2) if tb else B
        if b == 1:
            rep = lambda: R.repops_gemm(A[0], B[0], transA=ta, transB=tb, out=Cr[0])  # noqa: E731
            lib = lambda: torch.mm(opA[0], opB[0])  # noqa: E731
        else:
            rep = lambda: R.repops_gemm_strided_batched(  # noqa: E731
                A, B, Cr, M=M, N=N, K=K, lda=A.stride(1), ldb=B.stride(1), ldc=N, sA=(A.stride(0), 0),
                sB=(B.stride(0), 0), sC=(M * N, 0), batch=(b, 1), transA=ta, transB=tb)
            lib = lambda: torch.bmm(opA, opB)  # noqa: E731
        t_rep, t_lib = ms(rep), ms(lib)
        Cl = lib()
        rep()
        torch.cuda.synchronize()
        nd, mx = ulp_stats(Cl, Cr)
        fl = 2.0 * M * N * K * b
        out[f"{lay} {M}x{N}x{K}" + (f" x{b}" if b > 1 else "")] = {
            "repops_tflops": round(fl / t_rep / 1e9, 2), "cublas_tflops": round(fl / t_lib / 1e9, 2),
            "time_ratio": round(t_rep / t_lib, 3), "cublas_ulp_diff_frac": round(nd / Cl.numel(), 4),
            "cublas_max_ulp": mx}
        del A, B, Cr, Cl
    torch.cuda.empty_cache()
    return out


def cublas_vs_oracle_1024():
    """cpu_baseline leg (rank 0, N = 1): the full oracle R-GEMM at n = 1024 beside cuBLAS
    SGEMM and the R-GEMM on the same inputs -- ULP-diff counts against the oracle."""
    import torch

    import oracle
    import paper_2502_19405_b200 as R
    import synth
    A, B = synth.gemm_inputs(1024, "bench")
    t0 = time.perf_counter()
    ref = torch.from_numpy(oracle.gemm(A, B)).cuda()
    t_or = time.perf_counter() - t0
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    torch.backends.cuda.matmul.allow_tf32 = False
    nd_c, mx_c = ulp_stats(torch.mm(Ad, Bd), ref)
    nd_r, mx_r = ulp_stats(R.repops_gemm(Ad, Bd), ref)
    return {"n": 1024, "elements": 1024 * 1024, "cublas_ulp_diff": nd_c, "cublas_max_ulp": mx_c,
            "repops_ulp_diff": nd_r, "repops_max_ulp": mx_r, "oracle_s": round(t_or, 2)}


def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None}


# ---------------------------------------------------------------------- oracle legs
def oracle_sample_gemm(seconds_target=10.0):
    """The oracle (as it stands) on a bounded sample of the GEMM sweep: the first r
    rows of each GEMM (full K fold per element), r chosen for ~10 s on one core."""
    import oracle
    import synth
    oracle.lib()
    flops, t_total, rows_done = 0, 0.0, {}
    A, B = synth.gemm_inputs(1024, "bench")
    t0 = time.perf_counter()
    oracle.gemm(A[:2], B)
    per_row_1024 = (time.perf_counter() - t0) / 2
    for n in SIZES:
        A, B = synth.gemm_inputs(n, "bench")
        est_row = per_row_1024 * (n / 1024) ** 2 * (1.6 if n >= 4096 else 1.0)
        r = min(n, max(1, int(seconds_target / len(SIZES) / est_row)))
        t0 = time.perf_counter()
        oracle.gemm(A[:r], B)
        t_total += time.perf_counter() - t0
        flops += 2 * r * n * n
        rows_done[n] = r
    return flops / t_total / 1e12, t_total, f"first rows {rows_done} of each sweep GEMM (full K fold)"


def oracle_sample_gpt2(rows=128):
    """The oracle on a bounded sample of the GPT-2 step: `rows` token rows of shard 0
    through layer 0's four linear GEMMs (full K folds) and the LM head (K = 768 over
    all 50257 vocabulary columns), with their LayerNorm / GELU / softmax row work."""
    import oracle
    import synth
    oracle.lib()
    d, F, V, T = 768, 3072, 50257, 512
    W = {n: synth.gpt2_param(n, s, k) for n, s, k in synth.gpt2_param_specs(1, d, F, V, 1024)}
    x = synth.uniform(11, (rows, d), 1.0)
    t0 = time.perf_counter()
    ln, _, _ = oracle.layernorm(x, W["h0.ln1.g"], W["h0.ln1.b"])
    qkv = oracle.gemm(ln, W["h0.attn.w"], epi=1, bias=W["h0.attn.b"])
    oracle.softmax(qkv[:, :T].copy(), causal=False)
    proj = oracle.gemm(qkv[:, :d].copy(), W["h0.proj.w"], epi=1, bias=W["h0.proj.b"])
    fc = oracle.gemm(proj, W["h0.fc.w"], epi=1, bias=W["h0.fc.b"])
    g = oracle.gelu(fc)
    fc2 = oracle.gemm(g, W["h0.fc2.w"], epi=1, bias=W["h0.fc2.b"])
    oracle.gemm(fc2, W["wte"], transB=True)
    dt = time.perf_counter() - t0
    flops = 2 * rows * (d * 3 * d + d * d + 2 * d * F + d * V)
    return flops / dt / 1e12, dt, f"{rows} token rows through layer 0's linears + LM head (fp32 canonical order)"


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (the only reference this tier has), timed as
    it stands on the host cores, each step a bounded sample of the same workload."""
    if rank != 0:
        return
    import oracle
    oracle.lib()
    if args.workload == "gemm":
        fn = lambda: oracle_sample_gemm(2.0)  # noqa: E731
        cfg = gemm_config(world)
    else:
        fn = lambda: oracle_sample_gpt2(2)  # noqa: E731
        cfg = gpt2_config(world, args.combine)
    for _ in range(args.warmup):
        fn()
    vals, secs, sample = [], 0.0, ""
    for _ in range(args.steps):
        v, s, sample = fn()
        vals.append(v)
        secs += s
    value = statistics.median(vals)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": 1, "kind": "oracle", "sample": sample,
                         **cpu_info()},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------------- timing
def timed(wl, steps, world, local):
    """W warm-up done by the caller; K steps bracketed by barrier + sync, CUDA events
    on the launching stream, kernel families timed live (KernelTimer)."""
    import torch

    import paper_2502_19405_b200 as R
    stream = torch.cuda.current_stream()
    # pass 1 (the reported time): no per-launch instrumentation, one event per step boundary
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        l0 = R.launch_count()
        evs[0].record(stream)
        for k in range(steps):
            wl.step()
            if k + 1 < steps:
                evs[k + 1].record(stream)
        if hasattr(wl, "join"):
            wl.join()                         # side-stream work of the last step is inside the region
        evs[steps].record(stream)
        torch.cuda.synchronize()
        barrier(world)
        launches = (R.launch_count() - l0) // steps
    ms = max_over_ranks(evs[0].elapsed_time(evs[steps]) / steps, world)
    per_step = sorted(evs[k].elapsed_time(evs[k + 1]) for k in range(steps))
    clk = clk.summary()
    stats = {"median_ms": per_step[len(per_step) // 2], "min_ms": per_step[0], "max_ms": per_step[-1],
             "note": "rank-0 per-step intervals of the reported pass (the last one includes the final join)"}
    # pass 2 (same K steps): every R-GEMM / commit launch bracketed by CUDA events for the
    # kernel-family rates (roofline); its wall time is not the reported one
    timer = R.KernelTimer()
    barrier(world)
    torch.cuda.synchronize()
    R.set_timer(timer)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        wl.step()
    if hasattr(wl, "join"):
        wl.join()
    ev1.record(stream)
    torch.cuda.synchronize()
    R.set_timer(None)
    barrier(world)
    stats["instrumented_ms_per_step"] = max_over_ranks(ev0.elapsed_time(ev1) / steps, world)
    stats["instrumented_note"] = ("a second pass of the same K steps with every R-GEMM / commit launch bracketed by "
                                  "CUDA events: the kernel-family rates (roofline, commit) come from it")
    tot = timer.totals()
    if "gemm" in tot:  # GEMMs on the main and aux streams may overlap each other
        tot["gemm_union_ms"] = timer.union_ms("gemm", ev0)
    tot["_stats"] = stats
    return ms, tot, launches, clk


def e2e(wl, steps, world):
    import torch
    for _ in range(2):
        wl.e2e_step()
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        wl.e2e_step()
    torch.cuda.synchronize()
    return max_over_ranks((time.perf_counter() - t0) / steps, world)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="repops", choices=["repops", "reference"])
    ap.add_argument("--workload", default="gpt2", choices=["gpt2", "gemm"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--multi-extras", action="store_true",
                    help="at N > 1 also run the secondary workloads (config 3, the M-split sweep, the TP Llama "
                         "prefill); off by default so a scaling run times only the headline step")
    ap.add_argument("--no-commit", action="store_true", help="diagnostic: skip the Verde commitments")
    ap.add_argument("--no-overlap", action="store_true", help="diagnostic: commits on the main stream")
    ap.add_argument("--combine", default="p2p", choices=["p2p", "sliced", "gather"],
                    help="G > 1 gradient combine transport (same bits): fused peer-memory kernel, "
                         "NCCL all-to-all + all-gather, or NCCL all-gather of partials")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # a bare `python bench.py --gpus N`: relaunch as N ranks (one process per GPU)
        import subprocess
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={29500 + os.getpid() % 1000}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    rank, world, local = dist_init()
    device = torch.device("cuda", local)
    hbm = measured_hbm_gbs()
    out = {"metric": METRIC}
    results = {}
    # the secondary workloads' NCCL paths have only run as gloo processes sharing one GPU: at
    # N > 1 they are opt-in, so an untested collective cannot stall the scaling run's headline
    extras = not args.no_sweep and (world == 1 or args.multi_extras)
    order = [args.workload] + ([] if not extras else
                               [w for w in ("gpt2_ckpt", "gemm", "llama") if w != args.workload])

    def run_workload(wname):
        if wname in ("gpt2", "gpt2_ckpt"):
            wl = GPT2Train(rank, world, device, commit=not args.no_commit, overlap=not args.no_overlap,
                           combine=args.combine, mode="every" if wname == "gpt2" else "checkpoint")
        elif wname == "gemm":
            wl = GemmSweep(rank, world, device)
        else:
            wl = LlamaPrefillBench(rank, world, device)
        head_wl = wname == args.workload
        # the config-3 step (checkpoint commits every CKPT_EVERY steps) is timed over a whole
        # checkpoint interval so the amortised state commitment is inside the region
        steps = args.steps if head_wl else (GPT2Train.CKPT_EVERY if wname == "gpt2_ckpt" else max(2, min(args.steps, 3)))
        for _ in range(args.warmup):   # W >= 3 for every workload of the line, not only the headline
            wl.step()
        torch.cuda.synchronize()
        ms, tot, launches, clk = timed(wl, steps, world, local)
        e2e_s = e2e(wl, steps, world) if head_wl else ms * 1e-3
        gemm_ms, gemm_flops, gemm_n = tot.get("gemm", (0.0, 0, 0))
        gemm_ms = max_over_ranks(gemm_ms, world)
        peak = fp32_peak_tflops(clk["sm_max_mhz"] or 1965.0)
        achieved = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms else 0.0   # per GPU
        g_union = tot.get("gemm_union_ms")
        res = dict(ms=ms, value=wl.flops / (ms * 1e-3) / 1e12, launches=launches, clk=clk, e2e_s=e2e_s,
                   stats=tot.pop("_stats", None),
                   gemm_union=(gemm_flops / (g_union * 1e-3) / 1e12) if g_union else None,
                   e2e_value=wl.flops / e2e_s / 1e12, gemm=(achieved, peak, gemm_ms / steps, gemm_n // steps),
                   h2d=wl.h2d_bytes, d2h=wl.d2h_bytes)
        if "commit" in tot:
            c_ms, c_bytes, c_n = tot["commit"]
            res["commit"] = dict(gbs=c_bytes / (c_ms * 1e-3) / 1e9, ms_per_step=c_ms / steps,
                                 gb_per_step=c_bytes / steps / 1e9, plans_per_step=c_n // steps)
        if wname == "gpt2":
            res["combine"], res["combine_fallback"] = wl.st.combine, wl.st.combine_fallback
            if wl.st.p2p is not None:
                wl.st.p2p.check()   # raises if a peer-memory wait timed out
            res["root"] = wl.root.hex()
            res["loss"] = wl.st.loss()
            # diagnostic (not the headline): the same GEMM launches with the commit side
            # stream idle, i.e. the GEMM kernels' own rate without the SHA-256 sharing the SMs
            iso = GPT2Train.isolated_gemm(wl, world, local)
            if iso:
                res["gemm_isolated"] = iso
        elif wname == "llama":
            res["root"] = wl.root.hex()
        elif wname == "gpt2_ckpt":
            res["loss"] = wl.st.loss()
        else:
            res["digests"] = wl.digests()
        return res, wl


    errors = {}
    for wname in order:
        if wname == args.workload:
            res, wl = run_workload(wname)
        else:
            # a secondary workload of the line must not take the headline down with it
            try:
                res, wl = run_workload(wname)
            except Exception as e:  # noqa: BLE001 -- reported in the JSON line
                errors[wname] = f"{type(e).__name__}: {e}"[:300]
                wl = None
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
                continue
        results[wname] = res
        del wl
        torch.cuda.empty_cache()

    head = results[args.workload]
    achieved, peak, gemm_ms_step, gemm_launches = head["gemm"]
    clk = head["clk"]
    out.update({
        "value": head["value"], "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": head["ms"], "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
    })
    if args.workload == "gpt2":
        out["config"] = gpt2_config(world, head.get("combine", args.combine))
        if head.get("combine_fallback"):
            out["config"]["combine_fallback"] = head["combine_fallback"]
        out["gpt2_step_ms"] = head["ms"]
        out["loss"] = head["loss"]
        out["step_root"] = head["root"]
    else:
        out["config"] = gemm_config(world)
        out["digests"] = head["digests"]
    # primary: the GEMM family's flops over the UNION of its launch intervals (the aux-stream
    # weight-gradient GEMMs overlap the dgrads, so summed per-launch durations double-count)
    per_launch = achieved
    if head.get("gemm_union"):
        achieved = head["gemm_union"]
    out["roofline"] = {"bound": "alu", "kernel": "repops_gemm (FP32 FFMA2 on CUDA cores, sequential K)",
                       "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else 0,
                       "basis": "union of the R-GEMM launch intervals in the timed region" if head.get("gemm_union")
                       else "sum of per-launch CUDA-event durations",
                       "achieved_per_launch": per_launch, "frac_per_launch": per_launch / peak if peak else 0,
                       "peak_note": "148 SM x 128 FP32 lanes x 2 x sm_max_mhz (unit counts of the guides); frac at "
                                    "the median observed clock: %.3f" % (
                                        achieved / fp32_peak_tflops(clk["sm_mhz"]) if clk["sm_mhz"] else -1),
                       "gemm_ms_per_step": gemm_ms_step, "gemm_launches_per_step": gemm_launches,
                       "traffic": profiled_gemm_traffic(),
                       "register_probe_tflops": ffma2_probe(),
                       "register_probe_note": "measured live: register-resident FFMA2 chains over the whole GPU "
                                              "(repops_ffma2_probe) -- the practical FP32 ceiling under the "
                                              "run's clock; peak stays the unit-count figure",
                       "achieved_union": head.get("gemm_union"),
                       "frac_union": (head["gemm_union"] / peak) if head.get("gemm_union") else None,
                       "union_note": "R-GEMM flops / length of the union of the GEMM launch intervals: the "
                                     "backward's weight-gradient GEMMs run on an aux stream beside the dgrads, so "
                                     "per-launch durations (achieved) double-count the overlapped time",
                       "achieved_commit_idle": head.get("gemm_isolated"),
                       "frac_commit_idle": (head["gemm_isolated"] / peak) if head.get("gemm_isolated") else None,
                       "commit_idle_note": "diagnostic: the step's GEMMs timed live in 2 extra steps run with "
                                           "commit=False (no SHA-256 on the side stream sharing the SMs)",
                       "traffic_note": "DRAM bytes (read + write) per R-GEMM launch, mean over one GPT-2 step's "
                                       "GEMM launches, from the committed ncu launch list "
                                       "profiles/r02_gpt2_step_launches.csv (cold-cache replay)"}
    rp = out["roofline"].get("register_probe_tflops")
    out["roofline"]["frac_register_probe"] = (achieved / rp) if rp else None
    if "commit" in head:
        cm = head["commit"]
        cm["hbm_frac"] = cm["gbs"] / hbm
        cm["hbm_peak_gbs"] = hbm
        cm["bound"] = "alu"
        cm["alu_peak_gbs"] = sha_alu_peak_gbs(clk["sm_max_mhz"] or 1965.0)
        cm["alu_frac"] = cm["gbs"] / cm["alu_peak_gbs"]
        cm["note"] = ("SHA-256 is integer-ALU bound (949 ALU-pipe ops per 64 B block); gbs is the commit plans' "
                      "device time on the side stream, sharing the SMs with the step's FFMA2 GEMMs")
        try:
            import paper_2502_19405_b200 as R
            cm["register_probe_gbs"] = R.verde_sha256_probe_gbs()
            cm["frac_register_probe"] = cm["gbs"] / cm["register_probe_gbs"]
            cm["register_probe_note"] = ("measured live: the leaf kernel's compression sequence on register-resident "
                                         "blocks over the whole GPU (verde_sha256_probe) -- the practical ceiling "
                                         "of the commitment kernels, no loads / byte shifts / tree")
        except Exception as e:  # noqa: BLE001 -- diagnostic only
            cm["register_probe_gbs"] = None
            cm["register_probe_note"] = f"{type(e).__name__}: {e}"[:200]
        out["commit"] = cm
    out["clocks"] = clk
    out["step_stats"] = head.get("stats")
    out["gpu_launches"] = head["launches"]
    out["e2e"] = {"value": head["e2e_value"], "unit": "TFLOP/s", "h2d_bytes_per_step": head["h2d"],
                  "d2h_bytes_per_step": head["d2h"],
                  "note": "wall clock per step through the public API: H2D of the batch from pinned host memory, "
                          "the step, D2H of the committed result (max over ranks)"}
    if errors:
        out["workload_errors"] = errors
    for other, res in results.items():
        if other != args.workload:
            key = {"gemm": "gemm_sweep", "llama": "llama_prefill", "gpt2": "gpt2_step",
                   "gpt2_ckpt": "gpt2_train_step"}[other]
            out[key] = {"value": res["value"], "unit": "TFLOP/s", "ms_per_step": res["ms"],
                        "gemm_tflops": res["gemm"][0], "gemm_roofline_frac": res["gemm"][0] / res["gemm"][1],
                        "gemm_union_tflops": res.get("gemm_union"),
                        "gemm_union_frac": (res["gemm_union"] / res["gemm"][1]) if res.get("gemm_union") else None,
                        "digests": res.get("digests"), "root": res.get("root"), "commit": res.get("commit"),
                        "loss": res.get("loss"),
                        "config": {"gemm": "square n=1024..8192, M-split, each output committed",
                                   "gpt2_ckpt": "configs[2]: GPT-2 124M train step B=8 T=512 without per-operator "
                                                "commitments; the training state (param, m, v) committed + RFC 6962 "
                                                f"root every {GPT2Train.CKPT_EVERY} steps (Verde Phase-1 checkpoint "
                                                "logging, P:303-307), timed over one interval",
                                   "llama": "Llama-3-8B-shaped FP32 prefill, 2048 tokens, 32 layers, TP N-split "
                                            f"over {world} GPU(s) (8 column blocks), every output committed",
                                   "gpt2": "GPT-2 124M train step"}[other]}
    def guarded(key, fn):
        try:
            return fn()
        except Exception as e:  # noqa: BLE001 -- reported in the JSON line, the headline stands
            out.setdefault("workload_errors", {})[key] = f"{type(e).__name__}: {e}"[:300]
            return None

    if rank == 0 and world == 1 and not args.no_sweep:
        out["mlp_step"] = guarded("mlp_step", lambda: mlp_extra(with_oracle=not args.no_cpu_baseline))
    if rank == 0 and world == 1 and not args.no_sweep and args.workload == "gpt2":
        out["verde_dispute"] = guarded("verde_dispute",
                                       lambda: verde_dispute_bench(with_oracle=not args.no_cpu_baseline))
    if rank == 0 and world == 1 and not args.no_sweep:
        out["cublas"] = {"note": "non-reproducible cuBLAS FP32 SGEMM (torch.mm/bmm, TF32 off) on the same shapes, "
                                 "as overhead context (the paper's RepOps-vs-torch::mm comparison, P:684-771); "
                                 "time_ratio = R-GEMM time / cuBLAS time; ULP columns: cuBLAS output vs the "
                                 "R-GEMM output (bit-identical to the oracle, tests/)",
                         "shapes": guarded("cublas", cublas_context)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, secs, sample = oracle_sample_gpt2() if args.workload == "gpt2" else oracle_sample_gemm()
        out["cpu_baseline"] = {"value": v, "unit": "TFLOP/s", "cores": 1, "kind": "oracle",
                               "sample": f"{sample}; {secs:.1f} s on 1 host core", **cpu_info()}
        if "cublas" in out:
            out["cublas"]["vs_oracle_1024"] = guarded("cublas_vs_oracle", cublas_vs_oracle_1024)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


GPT2_FLOPS_NOTE = "3 x (2 M N K over every fwd matmul: 12 x [QKV, proj, FC, FC2] + full (unmasked) QK^T, PV + LM head)"


def gpt2_config(world, combine):
    """the headline line's config (both arms print the same object)"""
    return {"workload": "gpt2-124m train step B=8 T=512 (S=8 DP shards) + Verde commit of every operator output "
                        "+ node digests + step Merkle root",
            "global_batch": 8, "seq_len": 512, "parallelism": f"dp{world} (canonical R-TREE_S)",
            "combine": (f"{combine}: " + {"p2p": "per-layer buckets, one fused peer-memory kernel per rank (CUDA IPC)",
                                          "sliced": "NCCL all-to-all + all-gather",
                                          "gather": "NCCL all-gather of partials"}[combine])
            if world > 1 else "local tree (G=1)",
            "l2": "per-step working set ~17 GB >> 126 MB L2 (no explicit flush)",
            "inputs": "synthetic tokens + U(std 0.02) weights (synth.gpt2_*)",
            "flops_per_step": GPT2_FLOPS_NOTE}


def gemm_config(world):
    return {"workload": "gemm-sweep: R-GEMM square n=1024..8192 + Verde commit of every output",
            "sizes": list(SIZES), "sharding": f"M-split over {world} GPU(s), full K per rank",
            "l2": "step working set 1.07 GB > 126 MB L2 (no explicit flush)"}

if __name__ == "__main__":
    main()
