"""Env-slice data parallelism across the GPUs of one box.

Environments are independent worlds sharing immutable geometry
(scene.py:150-157), and every random draw is keyed by the global env index
(rng.py:1-12), so the render step shards with no collective: rank r of R owns
the contiguous slice ``env_slice(total, r, R)``, replicates the BVHs, and
passes ``env_offset`` to its Scene. The only communication is the optional
frame gather to a policy rank: ``gather_frames`` (NCCL all_gather / grouped
P2P, a copy after the step) or ``PeerFrameSink`` (the fused path: each rank's
render epilogue stores its block straight into the destination rank's buffer
over peer memory, so the transfer overlaps the traversal tile by tile and no
gather kernel runs).
"""

from __future__ import annotations

import ctypes
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


def gpu_numa_node(device: torch.device) -> int | None:
    """NUMA node of a GPU's PCI function (sysfs), or None when unknown."""
    try:
        p = torch.cuda.get_device_properties(device)
        path = f"/sys/bus/pci/devices/{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0/numa_node"
        node = int(open(path).read().strip())
        return node if node >= 0 else None
    except (OSError, ValueError, AttributeError, RuntimeError):
        return None


def _cpulist(text: str) -> set[int]:
    cpus = set()
    for part in text.strip().split(","):
        if not part:
            continue
        lo, _, hi = part.partition("-")
        cpus.update(range(int(lo), int(hi or lo) + 1))
    return cpus


def bind_to_gpu_numa(device: torch.device) -> dict:
    """Pin the calling thread (and the threads it starts afterwards) to the CPUs of
    its GPU's NUMA node.

    Call early, before allocating pinned host buffers: cudaHostAlloc first-touches
    its pages from the calling thread, so they then live on the GPU's node and the
    per-step H2D/D2H copies do not cross the socket interconnect. Returns
    {"node", "cpus"} (node None and every allowed CPU when the topology is
    unknown or has a single node).
    """
    allowed = os.sched_getaffinity(0)
    node = gpu_numa_node(device)
    if node is None:
        return {"node": None, "cpus": len(allowed)}
    try:
        cpus = _cpulist(open(f"/sys/devices/system/node/node{node}/cpulist").read()) & allowed
    except OSError:
        cpus = set()
    if cpus:
        os.sched_setaffinity(0, cpus)
    return {"node": node, "cpus": len(cpus) or len(allowed)}


def rank_sizes(n_local: int, group=None, device=None) -> list[int]:
    """Every rank's leading (env) size, in rank order (one small all_gather)."""
    world = dist.get_world_size(group)
    dev = device if device is not None and dist.get_backend(group) == "nccl" else torch.device("cpu")
    mine = torch.tensor([int(n_local)], dtype=torch.int64, device=dev)
    allv = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    return [int(v.item()) for v in allv]


def gather_frames(obs: torch.Tensor, dst: int | None = 0, group=None, sizes: list[int] | None = None
                  ) -> torch.Tensor | None:
    """Concatenate every rank's (N_r, C, H, W) observation block in rank order.

    dst=None: all ranks receive the full tensor (all_gather); otherwise only
    ``dst`` does (others get None). Blocks may differ in N_r (``env_slice``
    gives slices that differ by one when the env count does not divide):
    ``sizes`` (every rank's N_r) is exchanged first unless the caller passes
    it. NCCL uses grouped P2P for dst, all_gather_into_tensor for equal blocks
    (padded to the largest block otherwise); gloo stages through the CPU.
    """
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return obs
    if dist.get_backend(group) == "gloo" and obs.device.type == "cuda":
        # gloo collectives are host-side: stage through the CPU
        res = gather_frames(obs.cpu(), dst, group, sizes)
        return None if res is None else res.to(obs.device)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obs = obs.contiguous()
    if sizes is None:
        sizes = rank_sizes(obs.shape[0], group, obs.device)
    sizes = [int(x) for x in sizes]
    if len(sizes) != world or sizes[rank] != obs.shape[0]:
        raise ValueError(f"sizes {sizes} do not match world {world} / local block {obs.shape[0]}")
    tail = tuple(obs.shape[1:])
    total = sum(sizes)
    offs = [sum(sizes[:r]) for r in range(world)]
    nccl = dist.get_backend(group) == "nccl"
    if nccl and dst is not None:
        ops = []
        out = None
        if rank == dst:
            out = torch.empty((total,) + tail, dtype=obs.dtype, device=obs.device)
            out[offs[rank]:offs[rank] + sizes[rank]].copy_(obs)
            for r in range(world):
                if r != rank and sizes[r]:
                    ops.append(dist.P2POp(dist.irecv, out[offs[r]:offs[r] + sizes[r]], r, group))
        elif obs.shape[0]:
            ops.append(dist.P2POp(dist.isend, obs, dst, group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return out
    # collectives with equal blocks: pad every block to the largest one
    mx = max(sizes)
    blk = obs
    if obs.shape[0] != mx:
        blk = torch.zeros((mx,) + tail, dtype=obs.dtype, device=obs.device)
        blk[:obs.shape[0]].copy_(obs)
    if dst is None or rank == dst:
        padded = torch.empty((world * mx,) + tail, dtype=obs.dtype, device=obs.device)
        parts = list(padded.chunk(world))
    if dst is None:
        if nccl:
            dist.all_gather_into_tensor(padded, blk, group=group)
        else:
            dist.all_gather(parts, blk, group=group)
    elif rank == dst:
        dist.gather(blk, parts, dst=dst, group=group)
    else:
        dist.gather(blk, None, dst=dst, group=group)
        return None
    if mx * world == total:
        return padded
    return torch.cat([parts[r][:sizes[r]] for r in range(world)])


# ---------------------------------------------------------------------------
# Fused gather over peer memory (second mechanism)
# ---------------------------------------------------------------------------

class _DLDevice(ctypes.Structure):
    _fields_ = [("device_type", ctypes.c_int32), ("device_id", ctypes.c_int32)]


class _DLDataType(ctypes.Structure):
    _fields_ = [("code", ctypes.c_uint8), ("bits", ctypes.c_uint8), ("lanes", ctypes.c_uint16)]


class _DLTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("device", _DLDevice), ("ndim", ctypes.c_int32),
                ("dtype", _DLDataType), ("shape", ctypes.POINTER(ctypes.c_int64)),
                ("strides", ctypes.POINTER(ctypes.c_int64)), ("byte_offset", ctypes.c_uint64)]


class _DLManagedTensor(ctypes.Structure):
    pass


_DL_DELETER = ctypes.CFUNCTYPE(None, ctypes.POINTER(_DLManagedTensor))
_DLManagedTensor._fields_ = [("dl_tensor", _DLTensor), ("manager_ctx", ctypes.c_void_p),
                             ("deleter", _DL_DELETER)]
_KDL_CPU, _KDL_CUDA = 1, 2
_noop_deleter = _DL_DELETER(lambda _p: None)


def wrap_pointer(ptr: int, shape, device: torch.device, keepalive: list) -> torch.Tensor:
    """A float32 tensor over raw memory at ``ptr`` that torch places on ``device``.

    Used for peer mappings: torch's own pointer query would attribute an
    IPC-mapped buffer to the GPU that owns it, but kernels on the local GPU
    address it through the peer mapping, so the tensor must claim the local
    device. The DLPack structs are appended to ``keepalive``; the caller keeps
    that list (and the mapping) alive for the tensor's lifetime.
    """
    shape = tuple(int(x) for x in shape)
    shp = (ctypes.c_int64 * len(shape))(*shape)
    mt = _DLManagedTensor()
    mt.dl_tensor.data = ctypes.c_void_p(int(ptr))
    if device.type == "cuda":
        mt.dl_tensor.device = _DLDevice(_KDL_CUDA, device.index if device.index is not None else 0)
    else:
        mt.dl_tensor.device = _DLDevice(_KDL_CPU, 0)
    mt.dl_tensor.ndim = len(shape)
    mt.dl_tensor.dtype = _DLDataType(2, 32, 1)   # float32
    mt.dl_tensor.shape = shp
    mt.dl_tensor.strides = None                  # C-contiguous
    mt.dl_tensor.byte_offset = 0
    mt.deleter = _noop_deleter
    keepalive.extend([shp, mt])
    new_capsule = ctypes.pythonapi.PyCapsule_New
    new_capsule.restype = ctypes.py_object
    new_capsule.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
    return torch.utils.dlpack.from_dlpack(new_capsule(ctypes.addressof(mt), b"dltensor", None))


def peer_block_offsets(full_envs: int, env_start: int, env_count: int, frame_elems_per_env: int) -> tuple[int, int]:
    """(byte offset, byte length) of an env block inside the destination buffer."""
    if not 0 <= env_start <= env_start + env_count <= full_envs:
        raise ValueError(f"env block [{env_start}, {env_start + env_count}) outside [0, {full_envs})")
    return 4 * env_start * frame_elems_per_env, 4 * env_count * frame_elems_per_env


class PeerFrameSink:
    """Destination-rank observation buffers that every rank's render writes into directly.

    The destination rank (``dst``) allocates ``slots`` buffers of shape
    (N_total, C, H, W) with ``mdrt_peer_alloc`` and broadcasts their CUDA IPC
    handles; the other ranks map them (``mdrt_peer_open``). ``local(k)`` is the
    tensor to pass as ``render_pipeline(out=...)`` on every rank: this rank's
    env rows of slot ``k`` (on ``dst`` a plain view of its own buffer, on the
    others a peer view whose stores travel over NVLink inside the render
    epilogue). ``full(k)`` (dst only) is the gathered (N_total, C, H, W) batch.

    ``publish()`` makes the stores of the steps enqueued so far visible on
    ``dst``: with NCCL it is a one-element all_reduce on the current stream
    (kernel completion on every rank orders their peer stores before the
    collective finishes; no host sync); with gloo it synchronises the stream
    and runs a host barrier. Use at least two slots and alternate them so a
    producer never overwrites a slot the destination is still reading: the
    consumer must enqueue its use of slot k before the ``publish()`` that
    follows the step writing slot k+1.
    """

    def __init__(self, frame_shape_per_env, total_envs: int, env_start: int, env_count: int, *,
                 dst: int = 0, slots: int = 2, group=None, device: torch.device | None = None):
        from . import _native
        self._native = _native
        self.group = group
        self.dst = dst
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.per_env = tuple(int(x) for x in frame_shape_per_env)
        self.total_envs = int(total_envs)
        self.env_start, self.env_count = int(env_start), int(env_count)
        elems = 1
        for x in self.per_env:
            elems *= x
        self.elems_per_env = elems
        self.off, _ = peer_block_offsets(self.total_envs, self.env_start, self.env_count, elems)
        nbytes = 4 * self.total_envs * elems
        lib = _native.lib()
        dev = self.device.index if self.device.index is not None else 0
        self._owned, self._mapped, self._keep = [], [], []
        handles = None
        if self.rank == dst:
            handles = []
            for _ in range(slots):
                p = ctypes.c_void_p()
                h = ctypes.create_string_buffer(64)
                _native.check(lib.mdrt_peer_alloc(dev, nbytes, ctypes.byref(p), h))
                self._owned.append(p.value)
                handles.append(h.raw)
        if self.world > 1:
            box = [handles]
            dist.broadcast_object_list(box, src=dst, group=group)
            handles = box[0]
        bases = list(self._owned)
        if self.rank != dst:
            for h in handles:
                p = ctypes.c_void_p()
                _native.check(lib.mdrt_peer_open(dev, h, ctypes.byref(p)))
                self._mapped.append(p.value)
                _native.register_remote(p.value, nbytes)   # renders into it use MDRT_WIDE_STORES
            bases = list(self._mapped)
        self._local = [wrap_pointer(b + self.off, (self.env_count,) + self.per_env, self.device, self._keep)
                       for b in bases]
        self._full = ([wrap_pointer(b, (self.total_envs,) + self.per_env, self.device, self._keep)
                       for b in bases] if self.rank == dst else None)
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.device) if self.world > 1 else None

    @property
    def slots(self) -> int:
        return len(self._local)

    def local(self, k: int) -> torch.Tensor:
        return self._local[k % self.slots]

    def full(self, k: int) -> torch.Tensor:
        if self._full is None:
            raise RuntimeError(f"rank {self.rank} is not the destination rank {self.dst}")
        return self._full[k % self.slots]

    def publish(self) -> None:
        if self.world == 1:
            return
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.current_stream(self.device).synchronize()
            dist.barrier(group=self.group)

    def close(self) -> None:
        """Unmap / free the buffers (call on every rank, after the last use)."""
        lib = self._native.lib()
        torch.cuda.synchronize(self.device)
        self._local, self._full = [], None
        for p in self._mapped:
            self._native.unregister_remote(p)
            self._native.check(lib.mdrt_peer_close(ctypes.c_void_p(p)))
        if self.world > 1:
            dist.barrier(group=self.group)   # every mapping closed before the owner frees
        for p in self._owned:
            self._native.check(lib.mdrt_peer_free(ctypes.c_void_p(p)))
        self._mapped, self._owned, self._keep = [], [], []
