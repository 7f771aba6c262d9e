"""Env-slice data parallelism across the GPUs of one box.

Environments are independent worlds sharing immutable geometry
(scene.py:150-157), and every random draw is keyed by the global env index
(rng.py:1-12), so the render step shards with no collective: rank r of R owns
the contiguous slice ``env_slice(total, r, R)``, replicates the BVHs, and
passes ``env_offset`` to its Scene. The only communication is the optional
frame gather to a policy rank (``gather_frames``).
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_slice(total_envs: int, rank: int, world: int) -> tuple[int, int]:
    """(start, count) of rank's contiguous env block; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(int(total_envs), world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def init_from_env(backend: str | None = None):
    """torchrun-style init: returns (rank, world, local_rank, device)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
        device = torch.device("cuda", local)
    else:
        device = torch.device("cpu")
    if world > 1 and not dist.is_initialized():
        be = backend or ("nccl" if device.type == "cuda" else "gloo")
        kw = {"device_id": device} if be == "nccl" else {}
        dist.init_process_group(be, **kw)
    return rank, world, local, device


def gather_frames(obs: torch.Tensor, dst: int | None = 0, group=None) -> torch.Tensor | None:
    """Concatenate every rank's (N_r, C, H, W) observation block in rank order.

    dst=None: all ranks receive the full tensor (all_gather); otherwise only
    ``dst`` does (others get None). Requires equal N_r on all ranks. NCCL uses
    all_gather_into_tensor / grouped P2P; gloo uses all_gather / gather.
    """
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return obs
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obs = obs.contiguous()
    full_shape = (world * obs.shape[0],) + tuple(obs.shape[1:])
    nccl = dist.get_backend(group) == "nccl"
    if dst is None:
        out = torch.empty(full_shape, dtype=obs.dtype, device=obs.device)
        if nccl:
            dist.all_gather_into_tensor(out, obs, group=group)
        else:
            dist.all_gather(list(out.chunk(world)), obs, group=group)
        return out
    if nccl:
        ops = []
        out = None
        if rank == dst:
            out = torch.empty(full_shape, dtype=obs.dtype, device=obs.device)
            parts = out.chunk(world)
            parts[rank].copy_(obs)
            for r in range(world):
                if r != rank:
                    ops.append(dist.P2POp(dist.irecv, parts[r], r, group))
        else:
            ops.append(dist.P2POp(dist.isend, obs, dst, group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        return out
    if rank == dst:
        out = torch.empty(full_shape, dtype=obs.dtype, device=obs.device)
        dist.gather(obs, list(out.chunk(world)), dst=dst, group=group)
        return out
    dist.gather(obs, None, dst=dst, group=group)
    return None
