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
