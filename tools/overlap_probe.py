"""Co-residency probe: does SHA-256 commit work (ALU pipe) overlap an FFMA2 GEMM
(FMA pipe) when both run on separate streams?  Times GEMM chain alone, commit
chain alone, and both together, for GEMM occupancy variants (bits-neutral knobs:
tile cfg, shared-memory floor capping CTAs/SM)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_19405_b200 as R
from paper_2502_19405_b200._lib import lib

M, N, K = 4096, 3072, 768
torch.manual_seed(0)
A = torch.rand(M, K, device="cuda") - 0.5
B = torch.rand(K, N, device="cuda") - 0.5
C = torch.empty(M, N, device="cuda")
x = torch.rand(256 * 1024 * 1024, device="cuda")  # 1 GiB
d = torch.empty((1, 32), dtype=torch.uint8, device="cuda")
plan = R.CommitPlan([x], d)
sg, sc = torch.cuda.Stream(), torch.cuda.Stream()
NG, NC = 40, 12


def gem(cfg):
    for _ in range(NG):
        R.repops_gemm(A, B, out=C, stream=sg, cfg=cfg)


def com():
    for _ in range(NC):
        plan.run(stream=sc)


def timed(fns):
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    sg.wait_event(s)
    sc.wait_event(s)
    for f in fns:
        f()
    eg, ec = torch.cuda.Event(), torch.cuda.Event()
    eg.record(sg)
    ec.record(sc)
    torch.cuda.current_stream().wait_event(eg)
    torch.cuda.current_stream().wait_event(ec)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


for cfg, floor, cap in [(6, 0, 16), (6, 80 * 1024, 16), (6, 80 * 1024, 3), (6, 80 * 1024, 2), (6, 0, 1),
                        (9, 80 * 1024, 3), (6, 110 * 1024, 4), (6, 110 * 1024, 6)]:
    lib().repops_gemm_smem_floor(floor)
    lib().repops_commit_ctas_per_sm(cap)
    timed([lambda: gem(cfg)])
    tg = timed([lambda: gem(cfg)])
    tc = timed([com])
    tb = timed([lambda: gem(cfg), com])
    fl = 2 * M * N * K * NG / tg / 1e9
    print(f"cfg{cfg} smem_floor {floor // 1024:3d}K sha_cap {cap:2d}: gemm {tg:7.2f} ms ({fl:5.1f} TFLOP/s)  commit {tc:7.2f} ms  "
          f"both {tb:7.2f} ms  (serial {tg + tc:7.2f}, saved {100 * (tg + tc - tb) / min(tg, tc):5.1f}% of the shorter)",
          flush=True)
lib().repops_gemm_smem_floor(0)
lib().repops_commit_ctas_per_sm(16)
