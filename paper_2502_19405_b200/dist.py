"""Multi-GPU host logic (one process per GPU, torch.distributed for the plumbing).

Only order-insensitive dimensions are split; the paper
leaves the collective's combine order to future work, and this
build fixes it (reading R14):
  * DP: S fixed shards; rank r owns the aligned block [r*S/G, (r+1)*S/G).  The
    per-shard gradients are combined by R-TREE_S, evaluated as the aligned local
    subtree on each rank, an all-gather of the G partials (data movement only --
    NCCL reductions and in-switch NVLS reduction are never used on floats), and
    the top log2(G) levels on every rank.  Because the tree is balanced and the
    blocks are aligned, the bits equal the single-GPU tree over S parts.
  * GEMM: M (or N) slabs with the full K on every rank.
  * Commitments: every rank hashes what it produced; digests (32 B each) are
    all-gathered so that every rank builds the identical step root.
The arithmetic of the tree is a parameter (`tree`) so the same host logic is
exercised by the product (repops_tree_sum on the GPU) and by the CPU gloo tests.
"""
from __future__ import annotations

import torch


def shard_block(rank: int, world: int, shards: int) -> tuple[int, int]:
    """(first shard, count) owned by `rank`; requires shards % world == 0 and both powers of two."""
    if shards % world or world & (world - 1) or shards & (shards - 1):
        raise ValueError(f"need power-of-two world ({world}) dividing power-of-two shards ({shards})")
    per = shards // world
    return rank * per, per


def all_gather_rows(x: torch.Tensor, world: int, pg=None) -> torch.Tensor:
    """[world, *x.shape] with row r = rank r's x (rank order)."""
    if world == 1:
        return x.unsqueeze(0)
    import torch.distributed as dist
    out = torch.empty((world, *x.shape), dtype=x.dtype, device=x.device)
    if dist.get_backend(pg) == "nccl":
        dist.all_gather_into_tensor(out, x.contiguous(), group=pg)
    else:
        dist.all_gather(list(out.unbind(0)), x.contiguous(), group=pg)
    return out


def dp_tree_combine(local_parts, world: int, tree, pg=None, out=None):
    """R-TREE_S over all S shards' gradients, given this rank's aligned block.

    local_parts: list of this rank's S/G per-shard tensors (equal shapes);
    tree(parts, out) -> out evaluates the balanced tree over its parts."""
    if world == 1:
        return tree(local_parts, out)
    partial = tree(local_parts, None)                 # aligned local subtree
    allp = all_gather_rows(partial, world, pg)         # C1: G partials, data movement only
    return tree([allp[r] for r in range(world)], out)  # top levels, identical on every rank


def dp_tree_combine_sliced(local_parts, world: int, tree, pg=None, out=None):
    """Bandwidth-optimal R-TREE_S: the same bits as dp_tree_combine with
    2(G-1)/G x P instead of (G-1) x P bytes received per rank.  Each rank reduces its
    aligned local subtree, an all-to-all hands rank r slice r of every rank's partial,
    rank r applies the top levels to its slice (elementwise, so slicing cannot change
    a bit), and an all-gather of the summed slices rebuilds the full gradient."""
    if world == 1:
        return tree(local_parts, out)
    import torch.distributed as dist
    partial = tree(local_parts, None).reshape(-1)
    n = partial.numel()
    per = -(-n // world)
    send = torch.zeros(world * per, dtype=partial.dtype, device=partial.device)
    send[:n] = partial
    recv = torch.empty_like(send)
    if send.is_cuda and dist.get_backend(pg) != "nccl":  # gloo test transport: stage through the host
        rh = torch.empty(recv.shape, dtype=recv.dtype)
        dist.all_to_all_single(rh, send.cpu(), group=pg)
        recv.copy_(rh)
    else:
        dist.all_to_all_single(recv, send, group=pg)    # recv[j] = slice r of rank j's partial
    mine = tree([recv[j * per:(j + 1) * per] for j in range(world)], None)
    full = all_gather_rows(mine, world, pg).reshape(-1)[:n]
    if out is None:
        return full.reshape(local_parts[0].shape)
    out.copy_(full.reshape(out.shape))
    return out


def p2p_slice(rank: int, world: int, n: int, align: int = 4) -> tuple[int, int]:
    """[lo, hi) of the n-element gradient that `rank` combines in the peer-memory path:
    equal slices rounded up to `align` elements (16-byte float4 boundaries), the last
    one ragged; slices are disjoint and cover [0, n) for any n >= 0."""
    per = -(-n // world)
    per = -(-per // align) * align
    lo = min(rank * per, n)
    return lo, min(lo + per, n)


class P2PUnavailable(RuntimeError):
    """Peer-memory setup failed on some rank (raised on every rank, after agreeing)."""


class P2PTreeCombine:
    """R-TREE_S across G ranks as ONE fused kernel per rank over NVLink peer memory
    (the combine order is the paper's future work, fixed by
    reading R14).  Same bits as dp_tree_combine / dp_tree_combine_sliced.

    Setup (once): every rank allocates, with CUDA IPC, a partial buffer [P], a gradient
    buffer [P] (what AdamW reads) and a flag array [2, G]; the 64-byte handles are
    all-gathered over the process group and every peer buffer is mapped.
    Per bucket (`epoch` = bucket count, all on the caller's stream, no host sync):
      1. tree(local parts) -> my partial (the aligned local subtree);
      2. signal "partial ready" into every peer's flags[0][me]; wait for all G;
      3. repops_p2p_tree_combine on my slice p2p_slice(me): loads the slice of all G
         partials (P2P), top log2(G) levels, stores the sum into all G gradient buffers;
      4. signal "slice written" into flags[1][me] of every peer; wait for all G.
    After 4 every rank's gradient buffer holds the full combined gradient, and no peer
    will touch my partial again until I signal the next epoch (so buffers are reused).

    sync="host" replaces the device flags by stream synchronisation + a process-group
    barrier: the transport for tests where several processes share one GPU (their
    contexts time-slice, so one rank's spinning wait kernel would stall the others)."""

    def __init__(self, n: int, rank: int, world: int, pg=None, sync: str = "device", timeout_ms: int = 60000):
        import torch.distributed as dist
        from . import repops_ipc_alloc, repops_ipc_open
        if world & (world - 1) or world > 8:
            raise ValueError("P2PTreeCombine: world must be 1, 2, 4 or 8")
        self.n, self.rank, self.world, self.pg, self.sync = n, rank, world, pg, sync
        self.timeout_ms = timeout_ms
        self.lo, self.hi = p2p_slice(rank, world, n)
        self.partial, hp = repops_ipc_alloc(n)
        self.grad, hg = repops_ipc_alloc(n)
        self.flags, hf = repops_ipc_alloc(2 * world, torch.int32)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.grad.device)
        handles = [None] * world
        dist.all_gather_object(handles, (hp, hg, hf), group=pg)
        self._opened = []

        def peer(r, k, n_, dt):
            if r == rank:
                return (self.partial, self.grad, self.flags)[k]
            t = repops_ipc_open(handles[r][k], n_, dt)
            self._opened.append(t)
            return t
        err = None
        try:
            self.peer_partial = [peer(r, 0, n, torch.float32) for r in range(world)]
            self.peer_grad = [peer(r, 1, n, torch.float32) for r in range(world)]
            peer_flags = [peer(r, 2, 2 * world, torch.int32) for r in range(world)]
        except Exception as e:  # noqa: BLE001 -- agreed on below, then raised on every rank
            err = f"rank {rank}: {type(e).__name__}: {e}"[:300]
        errs = [None] * world
        dist.all_gather_object(errs, err, group=pg)   # every rank reaches this: same decision everywhere
        bad = [e for e in errs if e]
        if bad:
            raise P2PUnavailable(bad[0])
        self.peer_ready = [f[:world] for f in peer_flags]
        self.peer_done = [f[world:] for f in peer_flags]
        self.epoch = 0

    def _barrier(self, phase: int, stream):
        from . import repops_p2p_signal, repops_p2p_wait
        if self.sync == "host":
            import torch.distributed as dist
            (stream or torch.cuda.current_stream()).synchronize()
            dist.barrier(group=self.pg)
            return
        peers = self.peer_ready if phase == 0 else self.peer_done
        repops_p2p_signal(peers, self.rank, self.epoch, stream)
        repops_p2p_wait(peers[self.rank], self.world, self.epoch, self.timeout_ms, self.status, stream)

    def combine_range(self, local_parts, lo: int, hi: int, tree, stream=None):
        """One bucket [lo, hi) of the gradient (a layer's parameters): local subtree ->
        my partial[lo:hi]; "ready" signal / wait (next epoch); the fused kernel on my
        sub-slice of the bucket.  Buckets of one step are disjoint and issued in the
        same order on every rank; finish() closes the step."""
        from . import repops_p2p_tree_combine
        self.epoch += 1
        tree([q[lo:hi] for q in local_parts], self.partial[lo:hi])
        self._barrier(0, stream)
        slo, shi = p2p_slice(self.rank, self.world, hi - lo)
        # a timed-out "ready" wait leaves self.status set: the kernel then stores nothing
        repops_p2p_tree_combine(self.peer_partial, lo + slo, lo + shi, self.peer_grad, stream,
                                status=None if self.sync == "host" else self.status)

    def finish(self, stream=None):
        """ "done" signal / wait: every rank's slices of every bucket are in every gradient
        buffer, and no peer reads my partial again until the next step's first bucket."""
        self._barrier(1, stream)
        return self.grad

    def __call__(self, local_parts, tree, stream=None):
        """combine the whole gradient as one bucket; returns self.grad (the IPC gradient
        buffer, identical on every rank)."""
        self.combine_range(local_parts, 0, self.n, tree, stream)
        return self.finish(stream)

    def check(self):
        """raise if a device wait timed out (call after synchronising)."""
        if int(self.status.item()) != 0:
            raise RuntimeError("P2PTreeCombine: a peer did not signal within the timeout")

    def close(self):
        from . import repops_ipc_close, repops_ipc_free
        torch.cuda.synchronize()
        for t in self._opened:
            repops_ipc_close(t)
        self._opened = []
        for t in (self.partial, self.grad, self.flags):
            repops_ipc_free(t)


def gather_shard_digests(table: torch.Tensor, rep_slots: int, shard_slots: int, s0: int, s_loc: int, world: int,
                         pg=None) -> torch.Tensor:
    """C2: fill every shard region of the digest table from the rank that owns it.
    table: [rep_slots + S*shard_slots, 32] uint8; regions are shard-major."""
    if world == 1:
        return table
    lo = rep_slots + s0 * shard_slots
    mine = table[lo:lo + s_loc * shard_slots]
    allr = all_gather_rows(mine, world, pg)
    table[rep_slots:].copy_(allr.reshape(-1, table.shape[1]))
    return table
