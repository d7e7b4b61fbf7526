"""bench.py -- RepOps / Verde hot path on B200 (see DESIGN.md §7 "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl repops|reference] [--workload gemm]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N --steps K --warmup W

Workload "gemm" (BASELINE.json configs[1]: reproducible FP32 GEMM sweep, square
1024..8192, M-sharded over N GPUs, 0-ULP vs the oracle).  One step = the whole
hot path of that config over one batch of synthetic inputs:
  for n in (1024, 2048, 4096, 8192):
      C_r = R-GEMM(A[rows_r], B)            (rank r owns n/N rows, full K)
      root_r = Verde data-root commit of C_r (SHA-256 leaves + RFC 6962 levels)
  all_gather(root_r) -> tensor digest of C   (identical at every N)
value = sum of 2 n^3 over the sweep / max-over-ranks device time per step.

Prints ONE JSON line (rank 0).  The oracle (CPU, test infrastructure) is only
executed by the cpu_baseline leg (rank 0, N = 1) and by --impl reference.
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


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the timed region runs."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

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
                    if r & bit and name != "gpu_idle":
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
    if world > 1:
        torch.cuda.set_device(local)
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
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
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
            dA = hA.to(device)
            dB = hB.to(device)
            dC = torch.empty((rows, n), dtype=torch.float32, device=device)
            self.items.append(dict(n=n, rows=rows, hA=hA, hB=hB, A=dA, B=dB, C=dC))
        self.roots = torch.empty((len(SIZES), 32), dtype=torch.uint8, device=device)
        self.ws = R.CommitWorkspace(device)
        self.stream = torch.cuda.current_stream()
        self.gemm_ms = []  # per-launch device times of the dominant kernel
        self.gemm_flops = 0

    def step(self, time_gemm=False):
        R, torch = self.R, self.torch
        for it in self.items:
            if time_gemm:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
            R.repops_gemm(it["A"], it["B"], out=it["C"])
            if time_gemm:
                e1.record(self.stream)
                self.gemm_ms.append((e0, e1, 2 * it["rows"] * it["n"] * it["n"]))
        R.verde_commit_tensors([it["C"] for it in self.items], digests=self.roots, ws=self.ws, mode=1)

    def e2e_step(self):
        """Same step through the public API from pinned HOST buffers: H2D of the
        inputs, the step, D2H of the committed result (the slab roots)."""
        for it in self.items:
            it["A"].copy_(it["hA"], non_blocking=True)
            it["B"].copy_(it["hB"], non_blocking=True)
        self.step()
        return self.roots.to("cpu", non_blocking=False)

    @property
    def h2d_bytes(self):
        return sum(it["hA"].numel() * 4 + it["hB"].numel() * 4 for it in self.items)

    @property
    def d2h_bytes(self):
        return self.roots.numel()

    def digests(self):
        """Tensor digests of the full C matrices (identical at every world size)."""
        torch = self.torch
        roots = self.roots
        if self.world > 1:
            import torch.distributed as dist
            parts = [torch.empty_like(roots) for _ in range(self.world)]
            dist.all_gather(parts, roots)
        else:
            parts = [roots]
        out = []
        for q, it in enumerate(self.items):
            sub = b"".join(bytes(p[q].cpu().numpy().tobytes()) for p in parts)
            n = it["n"]
            out.append(self.R.verde_digest_from_subroots(sub, self.R.F32, (n, n), n * n * 4).hex())
        return out

    def kernel_times(self):
        ms = sum(e0.elapsed_time(e1) for e0, e1, _ in self.gemm_ms)
        flops = sum(f for _, _, f in self.gemm_ms)
        return ms, flops, len(self.gemm_ms)


# ---------------------------------------------------------------------- oracle legs
def cpu_sample_gemm(seconds_target=10.0):
    """Time the oracle (as it stands) on a bounded sample of the workload: the first
    r rows of each GEMM in the sweep (full K fold per element), r chosen for ~10 s."""
    import oracle
    import synth
    oracle.lib()
    flops, t_total, rows_done = 0, 0.0, {}
    # calibrate on the 1024 problem
    A, B = synth.gemm_inputs(1024, "bench")
    t0 = time.perf_counter()
    oracle.gemm(A[:2], B)
    per_row_1024 = (time.perf_counter() - t0) / 2
    for n in SIZES:
        A, B = synth.gemm_inputs(n, "bench")
        est_row = per_row_1024 * (n / 1024) ** 2 * (1.6 if n >= 4096 else 1.0)
        r = max(1, int(seconds_target / len(SIZES) / est_row))
        r = min(r, n)
        t0 = time.perf_counter()
        oracle.gemm(A[:r], B)
        t_total += time.perf_counter() - t0
        flops += 2 * r * n * n
        rows_done[n] = r
    return flops / t_total / 1e12, t_total, rows_done


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (the only reference this tier has), timed as
    it stands on the host cores, each step a bounded sample of the same workload."""
    if rank != 0:
        return
    import oracle
    import synth
    oracle.lib()
    inputs = [synth.gemm_inputs(n, "bench") for n in SIZES]
    rows = {1024: 16, 2048: 4, 4096: 1, 8192: 1}

    def ref_step():
        f = 0
        for (A, B), n in zip(inputs, SIZES):
            r = rows[n]
            C = oracle.gemm(A[:r], B)
            oracle.data_root(C)
            f += 2 * r * n * n
        return f

    for _ in range(args.warmup):
        ref_step()
    t0 = time.perf_counter()
    flops = 0
    for _ in range(args.steps):
        flops += ref_step()
    dt = time.perf_counter() - t0
    value = flops / dt / 1e12
    sample = f"rows {rows} of each n^3 GEMM (full K fold per element) + RFC 6962 data root of those rows"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": "gemm-sweep 1024-8192 (oracle sample)", "sizes": list(SIZES)},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="repops", choices=["repops", "reference"])
    ap.add_argument("--workload", default="gemm", choices=["gemm"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local = (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                          int(os.environ.get("LOCAL_RANK", "0")))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    rank, world, local = dist_init()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    import paper_2502_19405_b200 as R

    wl = GemmSweep(rank, world, device)
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, device time via CUDA events, max over ranks
    stream = torch.cuda.current_stream()
    l0 = R.launch_count()
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            wl.step(time_gemm=True)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    launches = (R.launch_count() - l0) // args.steps
    ms = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms, world)
    value = SWEEP_FLOPS / (ms * 1e-3) / 1e12

    gemm_ms, gemm_flops, nl = wl.kernel_times()
    gemm_ms = max_over_ranks(gemm_ms, world)
    achieved = gemm_flops * world / (gemm_ms * 1e-3) / 1e12  # all ranks' GEMM flops over the (max) GEMM time
    achieved_per_gpu = achieved / world

    # ---- e2e through the public API from pinned host buffers
    for _ in range(2):
        wl.e2e_step()
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        wl.e2e_step()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps, world)
    e2e_value = SWEEP_FLOPS / e2e_s / 1e12

    digests = wl.digests()
    c = clk.summary()
    peak_max = fp32_peak_tflops(c["sm_max_mhz"] or 1965.0)
    out = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "gemm-sweep: R-GEMM square n=1024,2048,4096,8192 + Verde commit of every output",
                   "sizes": list(SIZES), "sharding": f"M-split over {world} GPU(s), full K per rank",
                   "l2": "step working set 1.07 GB > 126 MB L2 (no explicit flush)",
                   "inputs": "A,B ~ U[-1,1) on a 24-bit grid (synth.gemm_inputs, SplitMix64)"},
        "roofline": {"bound": "alu", "kernel": "repops_gemm (FP32 FFMA, sequential K)",
                     "achieved": achieved_per_gpu, "peak": peak_max, "unit": "TFLOP/s",
                     "frac": achieved_per_gpu / peak_max,
                     "peak_note": "148 SM x 128 FP32 lanes x 2 x sm_max_mhz (guide unit counts); "
                                  "frac at the median observed clock: %.3f" % (
                                      achieved_per_gpu / fp32_peak_tflops(c["sm_mhz"]) if c["sm_mhz"] else -1),
                     "traffic": None, "launches_timed": nl},
        "clocks": c,
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": wl.h2d_bytes,
                "d2h_bytes_per_step": wl.d2h_bytes,
                "note": "pinned host A,B -> device, step, committed roots -> host (wall clock, max over ranks)"},
        "digests": digests,
    }
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            out["roofline"]["traffic"] = json.load(open(tp)).get("repops_gemm_8192")
        except Exception:
            pass
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, secs, rows = cpu_sample_gemm()
        out["cpu_baseline"] = {"value": v, "unit": "TFLOP/s", "cores": 1, "kind": "oracle",
                               "sample": f"first rows {rows} of each sweep GEMM, {secs:.1f} s on 1 host core"}
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
