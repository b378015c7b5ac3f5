"""Multi-GPU plumbing: spatial-slab sharding of the points and the one
exchange step of the path, a sum-allreduce of the partial systems.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Each rank
assembles its slab of points against the full, replicated centre set and
pattern; the device buffer [values | rhs | hits] is then summed in place across
ranks (B and A^T h are sums over points, so partial sums add).  On CPU the same
code runs over gloo on host copies (tests/test_multirank.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native


def partition_slabs(points: np.ndarray, n_slabs: int, axis: int | None = None):
    """Equal-count slabs along `axis` (default: x in 2-D, z in 3-D).
    Returns (bounds[n_slabs+1], slab_of[n])."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    dim = pts.shape[1]
    axis = (0 if dim == 2 else 2) if axis is None else axis
    bounds = np.empty(n_slabs + 1)
    slab = np.empty(pts.shape[0], dtype=np.uint32)
    st = _native.lib().rbg_partition_slabs(dim, pts.ctypes.data, pts.shape[0], axis, n_slabs,
                                          bounds.ctypes.data, slab.ctypes.data)
    _native.check(st)
    return bounds, slab


class _CudaArray:
    """Zero-copy __cuda_array_interface__ view of a device fp64 buffer."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3, "strides": None}


def system_tensor(engine):
    """torch view (no copy) of the engine's device system buffer."""
    import torch

    ptr, count = engine.system_device()
    return torch.as_tensor(_CudaArray(ptr, count), device="cuda")


def allreduce_system(engine, group=None) -> None:
    """In-place sum of [values | rhs | hits] across the ranks of `group`.
    The engine must run on torch's current stream (Engine(stream=...)), so the
    collective is ordered after the assembly without a host sync."""
    import torch.distributed as dist

    dist.all_reduce(system_tensor(engine), op=dist.ReduceOp.SUM, group=group)


def allreduce_host(arrays: list[np.ndarray], group=None) -> None:
    """CPU/gloo variant on host arrays (tests and host-side reduction)."""
    import torch
    import torch.distributed as dist

    for a in arrays:
        t = torch.from_numpy(a)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
