"""Multi-GPU row-block sharding of the ball matmul.

One process per GPU (torch.distributed, NCCL over NVLink on the GPU box; gloo
for the CPU tests).  Rank r owns rows [r*M/W, (r+1)*M/W) of A and C; B is
replicated.  The only collectives move operand and result tiles:

    scatter   A row blocks            (root -> ranks)
    broadcast B                       (root -> ranks)
    all_reduce(min) of the per-rank "single-block plan" flag
    gather    C row blocks            (ranks -> root)

Bit-identity with the single call block_matmul_ball(A, B, p): the per-row
scale exponents e_i, the recombine and the radius row centring are row-local
and f_j is B-only (src/matmul.cpp:163-203, 397-422), so a shard's rows are
computed exactly as in the full product whenever the full product's plan is a
single block.  If every rank's LOCAL plan is single-block (midpoint h uses the
shard's entry precision <= the global one, radius h = 900 is fixed), the global
plan is single-block too; otherwise the ranks fall back to gathering A on the
root, which runs the full product (multi-block plans need the global greedy
split, src/matmul.cpp:74-114).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

FIELDS = ("mant", "exp", "kind", "rad_man", "rad_exp")


def row_range(M: int, world: int, rank: int):
    per = (M + world - 1) // world
    lo = min(M, rank * per)
    return lo, min(M, lo + per), per


def to_tensors(arr, device):
    """BallArray (numpy) or DeviceBallArray (torch) -> dict of torch tensors on `device`"""
    import torch
    from .balls import BallArray
    if isinstance(arr, BallArray):
        t = {"mant": torch.from_numpy(arr.mant.view(np.int64)), "exp": torch.from_numpy(arr.exp),
             "kind": torch.from_numpy(arr.kind), "rad_man": torch.from_numpy(arr.rad_man.view(np.int32)),
             "rad_exp": torch.from_numpy(arr.rad_exp)}
    else:
        t = {f: getattr(arr, f) for f in FIELDS}
    return {k: v.to(device).contiguous() for k, v in t.items()}


def from_tensors(t, on_device: bool):
    from .balls import BallArray, DeviceBallArray
    if on_device:
        return DeviceBallArray(t["mant"], t["exp"], t["kind"], t["rad_man"], t["rad_exp"])
    return BallArray(t["mant"].cpu().numpy().view(np.uint64), t["exp"].cpu().numpy(),
                     t["kind"].cpu().numpy(), t["rad_man"].cpu().numpy().view(np.uint32),
                     t["rad_exp"].cpu().numpy())


def _empty_like_rows(rows, L, device):
    import torch
    return {"mant": torch.zeros((rows, L), dtype=torch.int64, device=device),
            "exp": torch.zeros(rows, dtype=torch.int64, device=device),
            "kind": torch.zeros(rows, dtype=torch.uint8, device=device),
            "rad_man": torch.zeros(rows, dtype=torch.int32, device=device),
            "rad_exp": torch.zeros(rows, dtype=torch.int64, device=device)}


@dataclass
class PlanInfo:
    blocks: int
    radius_single: bool


def device_plan_info(A, B, prec) -> PlanInfo:
    """plan of the local shard through the CUDA library"""
    from . import ops
    info = ops.plan_info(A, B, prec)
    return PlanInfo(blocks=info["n_blocks"] if not info["special"] else 2,
                    radius_single=bool(info["radius_single"]))


def sharded_matmul(A, B, M: int, K: int, N: int, prec: int, *, group=None, root: int = 0,
                   device="cuda", compute=None, plan_info=None):
    """C = A B by output row blocks over the ranks of `group`.

    A, B: ball arrays (host BallArray or DeviceBallArray) significant on `root`
    only; M, K, N, prec known everywhere.  `compute(A_rows, B, rows, K, N, prec)`
    returns the local product as a ball array (default: the CUDA block matmul);
    `plan_info(A_rows, B, rows, K, N, prec)` reports the local plan.  Returns C
    (M x N ball array) on root, None elsewhere."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    on_device = device != "cpu"
    if compute is None or plan_info is None:
        from . import ops

        def compute(a, b, r, k, n, p):  # noqa: F811
            return ops.block_matmul_ball(ops.BallMatrix(a, r, k), ops.BallMatrix(b, k, n), p).balls

        def plan_info(a, b, r, k, n, p):  # noqa: F811
            return device_plan_info(ops.BallMatrix(a, r, k), ops.BallMatrix(b, k, n), p)
    from .balls import limbs_for
    # limb slot counts travel with the metadata
    Ls = torch.zeros(2, dtype=torch.int64, device=device)
    if rank == root:
        Ls[0], Ls[1] = A.L, B.L
    dist.broadcast(Ls, root, group=group)
    LA, LB = int(Ls[0]), int(Ls[1])
    lo, hi, per = row_range(M, world, rank)
    # scatter A row blocks (padded to `per` rows)
    mine = _empty_like_rows(per * K, LA, device)
    if rank == root:
        full = to_tensors(A, device)
        chunks = {}
        for f in FIELDS:
            parts = []
            for r in range(world):
                rl, rh, _ = row_range(M, world, r)
                part = full[f][rl * K:rh * K]
                pad = per * K - part.shape[0]
                if pad:
                    part = torch.cat([part, torch.zeros((pad,) + tuple(part.shape[1:]), dtype=part.dtype,
                                                        device=device)])
                parts.append(part.contiguous())
            chunks[f] = parts
    for f in FIELDS:
        dist.scatter(mine[f], chunks[f] if rank == root else None, src=root, group=group)
    rows = hi - lo
    a_loc = {f: v[:rows * K] for f, v in mine.items()}
    # broadcast B
    b_t = to_tensors(B, device) if rank == root else _empty_like_rows(K * N, LB, device)
    for f in FIELDS:
        dist.broadcast(b_t[f], root, group=group)
    a_arr, b_arr = from_tensors(a_loc, on_device), from_tensors(b_t, on_device)
    # every local plan single-block <=> the global plan is (module docstring)
    single = 1
    if rows:
        info = plan_info(a_arr, b_arr, rows, K, N, prec)
        single = int(info.blocks <= 1 and info.radius_single)
    flag = torch.tensor([single], dtype=torch.int64, device=device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    Lc = limbs_for(prec)
    if int(flag.item()) == 1:
        c_loc = _empty_like_rows(per * N, Lc, device)
        if rows:
            c_arr = to_tensors(compute(a_arr, b_arr, rows, K, N, prec), device)
            for f in FIELDS:
                c_loc[f][:rows * N] = c_arr[f].reshape(c_loc[f][:rows * N].shape)
        gathered = {f: [torch.zeros_like(c_loc[f]) for _ in range(world)] if rank == root else None
                    for f in FIELDS}
        for f in FIELDS:
            dist.gather(c_loc[f], gathered[f], dst=root, group=group)
        if rank != root:
            return None
        out = {}
        for f in FIELDS:
            parts = []
            for r in range(world):
                rl, rh, _ = row_range(M, world, r)
                parts.append(gathered[f][r][:(rh - rl) * N])
            out[f] = torch.cat(parts)
        return from_tensors(out, on_device)
    # fallback: the root runs the full product on the A it scattered (no gather)
    if rank != root:
        return None
    return compute(from_tensors(full, on_device), b_arr, M, K, N, prec)
