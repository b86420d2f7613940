"""Per-GPU batch sharder (SURVEY.md 8 e).

Images are independent, so a batch shards by image with NO data-path
collective: GPU g owns images [start_g, stop_g) (contiguous, balanced), runs
one flat-batch launch on its own stream, and the per-pixel maps plus the
exact per-image min/max make outputs bit-identical for any GPU count (the
multi-GPU analogue of the reference's thread-count invariance,
test_core.py:201-206). Two drivers:

* one process per GPU (``torch.distributed``, the bench / torchrun layout):
  :func:`shard_range` picks the rank's images; :func:`gather_to_root` is the
  optional final gather (an all-gather of equal-size padded shards, timed
  separately from the device metric);
* one process driving several GPUs: :func:`run_on_devices` fans the shards
  of a host batch out to ``wg_host_*`` calls, one host thread per device.

The gather can also be part of the launch itself: :class:`PeerBuffer` is the
whole batch's output allocated on the root and mapped into every rank over
CUDA IPC (NVLink peer access); a rank passes ``peer.view(first, count)`` as the
``out=`` of its decolor call and the kernel stores its shard straight into
the root's memory -- no staging copy, no separate collective.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from typing import Callable, Sequence

import numpy as np


def shard_range(n_items: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split: the first ``n % world`` ranks get one extra item."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} for world size {world_size}")
    if n_items < 0:
        raise ValueError(f"n_items must be >= 0, got {n_items}")
    base, extra = divmod(n_items, world_size)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_sizes(n_items: int, world_size: int) -> list[int]:
    return [b - a for a, b in (shard_range(n_items, world_size, r) for r in range(world_size))]


def gather_to_root(local, n_items: int, group=None, root: int = 0):
    """Assemble every rank's shard (leading axis = items) on ``root``.

    Shards are padded to the largest shard size and sent to ``root`` with one
    ``gather`` (NCCL send/recv over NVLink on GPUs: only the root receives and
    holds the whole batch; gloo on CPU falls back to an all-gather); the root
    trims the padding and concatenates in rank order. Returns the full batch
    on ``root`` and ``None`` elsewhere.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = shard_sizes(n_items, world)
    if local.shape[0] != sizes[rank]:
        raise ValueError(f"rank {rank} holds {local.shape[0]} items, expected {sizes[rank]}")
    cap = max(sizes) if sizes else 0
    padded = torch.zeros((cap, *local.shape[1:]), dtype=local.dtype, device=local.device)
    if local.shape[0]:
        padded[: local.shape[0]] = local
    if dist.get_backend(group) == "gloo":
        full = torch.empty((world * cap, *local.shape[1:]), dtype=local.dtype, device=local.device)
        parts = list(full.chunk(world)) if world else []
        dist.all_gather(parts, padded, group=group)
    else:
        full = torch.empty((world * cap, *local.shape[1:]), dtype=local.dtype, device=local.device) \
            if rank == root else None
        dist.gather(padded, list(full.chunk(world)) if full is not None else None, dst=root, group=group)
    if rank != root:
        return None
    pieces = [full[r * cap: r * cap + sizes[r]] for r in range(world)]
    return torch.cat(pieces, dim=0) if pieces else full[:0]


def run_on_devices(fn: Callable[[np.ndarray, int], np.ndarray], batch: np.ndarray,
                   devices: Sequence[int]) -> np.ndarray:
    """Shard a host batch by image over ``devices``; ``fn(shard, device)`` -> per-shard result.

    One host thread per device (each ``wg_host_*`` call is synchronous on
    its own device's streams); results are concatenated in image order.
    """
    if not devices:
        raise ValueError("need at least one device")
    n = batch.shape[0]
    spans = [shard_range(n, len(devices), r) for r in range(len(devices))]
    with ThreadPoolExecutor(max_workers=len(devices)) as pool:
        futs = [pool.submit(fn, batch[a:b], d) for (a, b), d in zip(spans, devices) if b > a]
        parts = [f.result() for f in futs]
    return np.concatenate(parts, axis=0) if parts else fn(batch[:0], devices[0])


class _CudaArray:
    """A raw device pointer as a ``__cuda_array_interface__`` object (torch.as_tensor)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class PeerBuffer:
    """The full batch's output on ``root``, mapped into every rank (SURVEY.md 8 e).

    The root allocates ``n_items`` items of ``item_shape`` (``wg_ipc_alloc``,
    its own cudaMalloc) and broadcasts the 64-byte CUDA IPC handle; the other
    ranks map it (``wg_ipc_open``, peer access over NVLink). ``view(first,
    count)`` is a tensor over items [first, first + count) of the root's buffer
    on every rank: given as ``out=`` to ``decolor`` / ``decolor_tone``, the
    kernel's stores land in the root's HBM. Call :meth:`close` on every rank
    (collective) when done; the root's full batch is :meth:`full` until then.
    """

    def __init__(self, n_items: int, item_shape, device: int, dtype: str = "uint8", group=None, root: int = 0):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib

        if dtype not in ("uint8", "float32"):
            raise ValueError(f"unsupported dtype {dtype}")
        self._torch = torch
        self.device = int(device)
        self.item_shape = tuple(int(x) for x in item_shape)
        self.dtype = dtype
        self.itemsize = 1 if dtype == "uint8" else 4
        self.item_elems = int(np.prod(self.item_shape)) if self.item_shape else 1
        self.n_items = int(n_items)
        self.group, self.root = group, root
        self.rank = dist.get_rank(group)
        nbytes = max(1, self.n_items * self.item_elems * self.itemsize)
        handle = (ctypes.c_uint8 * 64)()
        ptr = ctypes.c_void_p()
        if self.rank == root:
            _lib.call("wg_ipc_alloc", nbytes, self.device, ctypes.byref(ptr), handle)
        box = [bytes(handle)]
        dist.broadcast_object_list(box, src=root, group=group)
        err = None
        if self.rank != root:
            ctypes.memmove(handle, box[0], 64)
            try:
                _lib.call("wg_ipc_open", handle, self.device, ctypes.byref(ptr))
            except Exception as e:  # every rank learns of it below (no rank left waiting)
                err = f"rank {self.rank}: {e}"
        errs = [None] * dist.get_world_size(group)
        dist.all_gather_object(errs, err, group=group)
        if any(errs):
            if self.rank == root:
                _lib.call("wg_ipc_free", ptr.value, self.device)
            elif err is None:
                _lib.call("wg_ipc_close", ptr.value)
            raise RuntimeError("peer buffer mapping failed: " + "; ".join(e for e in errs if e))
        self.ptr = int(ptr.value)
        self._open = True

    def ptr_at(self, first: int) -> int:
        """Device address of item ``first`` of the root's buffer in this rank's mapping
        (for the C ABI's ``out`` pointer: the launch's device is the caller's)."""
        if not 0 <= first <= self.n_items:
            raise ValueError(f"item {first} outside [0, {self.n_items}]")
        return self.ptr + first * self.item_elems * self.itemsize

    def view(self, first: int, count: int):
        """Items [first, first + count) of the root's buffer, as a tensor on this rank's device.

        (torch infers the tensor's device from the pointer; when a peer mapping
        reports the root's device instead, use :meth:`ptr_at` with the C ABI.)
        """
        if not (0 <= first and first + count <= self.n_items):
            raise ValueError(f"items [{first}, {first + count}) outside [0, {self.n_items})")
        typestr = "|u1" if self.dtype == "uint8" else "<f4"
        with self._torch.cuda.device(self.device):
            t = self._torch.as_tensor(_CudaArray(self.ptr_at(first), (count, *self.item_shape), typestr),
                                      device=f"cuda:{self.device}")
        if t.device.index != self.device:
            raise RuntimeError(f"peer view landed on {t.device}, not cuda:{self.device}: use ptr_at()")
        return t

    def full(self):
        """The whole batch (root only)."""
        if self.rank != self.root:
            raise ValueError("full() is the root's view; other ranks use view()")
        return self.view(0, self.n_items)

    def close(self):
        """Collective: every rank's stores are complete, then unmap / free."""
        import torch.distributed as dist

        from . import _lib

        if not self._open:
            return
        self._torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        if self.rank != self.root:
            _lib.call("wg_ipc_close", self.ptr)
        dist.barrier(group=self.group)  # every mapping closed before the root frees
        if self.rank == self.root:
            _lib.call("wg_ipc_free", self.ptr, self.device)
        self._open = False
