"""Co-residency probe for the gemm_tn kernel (cfg 20) and the SHA-256 commit: GEMM alone
(2 or 1 CTAs / SM via the shared-memory floor hook), commit alone, both on two streams."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_19405_b200 as R
from paper_2502_19405_b200._lib import lib

M, N, K = 4096, 4096, 2048
At = torch.rand(K, M, device="cuda") - 0.5
B = torch.rand(K, N, device="cuda") - 0.5
C = torch.empty(M, N, device="cuda")
x = torch.rand(256 * 1024 * 1024, device="cuda")  # 1 GiB
d = torch.empty((1, 32), dtype=torch.uint8, device="cuda")
plan = R.CommitPlan([x], d)
sg, sc = torch.cuda.Stream(priority=-1), torch.cuda.Stream()
NG, NC = 20, 4


def gem():
    for _ in range(NG):
        R.repops_gemm(At, B, transA=True, out=C, stream=sg, cfg=20)


def com():
    for _ in range(NC):
        plan.run(stream=sc)


def timed(fns):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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


for floor, cap in [(0, 16), (120 * 1024, 16), (120 * 1024, 4), (120 * 1024, 2)]:
    lib().repops_gemm_smem_floor(floor)
    lib().repops_commit_ctas_per_sm(cap)
    timed([gem])
    tg = timed([gem])
    tc = timed([com])
    tb = timed([gem, com])
    fl = 2 * M * N * K * NG / tg / 1e9
    print(f"gemm_tn smem_floor {floor // 1024:3d}K sha_cap {cap:2d}: gemm {tg:7.2f} ms ({fl:5.1f} TFLOP/s)  "
          f"commit {tc:7.2f} ms ({NC / tc:5.3f} GiB/ms) both {tb:7.2f} ms (serial {tg + tc:7.2f}, saved "
          f"{100 * (tg + tc - tb) / min(tg, tc):5.1f}% of the shorter)", flush=True)
lib().repops_gemm_smem_floor(0)
lib().repops_commit_ctas_per_sm(16)
