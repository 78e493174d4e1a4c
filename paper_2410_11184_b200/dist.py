"""Exchange callbacks for the sharded many-ciphertext Softmax.

The library calls ``exchange(user, partial, gathered, words, stream)`` once
per Softmax iteration with this rank's degree-2 partial aux sum; the callback
must leave the partials of all ranks, in rank order, in ``gathered``.  The
library then adds them mod q (exact, order-independent), so every rank holds
bit-identical aux ciphertexts and the result equals the single-GPU run.

PyTorch is the plumbing here: the process group (NCCL over NVLink on GPUs,
gloo on CPU for tests) performs the all-gather.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import EXCHANGE_FN


class _CudaBuf:
    """A raw device pointer exposed through __cuda_array_interface__."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (int(ptr), False),
                                         "version": 2, "strides": None}


def nccl_exchange(group=None):
    """all_gather_into_tensor over the default (NCCL) process group."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)

    def fn(user, partial, gathered, words, stream):
        try:
            src = torch.as_tensor(_CudaBuf(partial, words), device="cuda")
            dst = torch.as_tensor(_CudaBuf(gathered, words * world), device="cuda")
            # order the collective on the library's stream, not torch's current one
            ext = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
            with torch.cuda.stream(ext):
                dist.all_gather_into_tensor(dst, src, group=group)
            return 0
        except Exception as e:  # pragma: no cover - surfaced as HS_ENCCL
            print("nccl_exchange failed:", e)
            return 1

    return EXCHANGE_FN(fn)


def host_exchange(group=None):
    """The same contract on host buffers with a gloo group (CPU tests of the
    multi-rank path; the GPU library itself always passes device buffers)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)

    def fn(user, partial, gathered, words, stream):
        try:
            src = torch.from_numpy(np.ctypeslib.as_array((C.c_int64 * words).from_address(partial)))
            dst = torch.from_numpy(np.ctypeslib.as_array((C.c_int64 * (words * world)).from_address(gathered)))
            parts = [torch.empty_like(src) for _ in range(world)]
            dist.all_gather(parts, src, group=group)
            dst.copy_(torch.cat(parts))
            return 0
        except Exception as e:  # pragma: no cover
            print("host_exchange failed:", e)
            return 1

    return EXCHANGE_FN(fn)


def gloo_device_exchange(group=None):
    """The device-buffer contract over a gloo (host) process group: the
    partial is staged through host memory, all-gathered by gloo and copied
    back.  For hosts without NCCL, and for the multi-process GPU test that
    runs two ranks on one GPU -- every wait is host-side (no kernel waits on
    another rank's kernel)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)

    def fn(user, partial, gathered, words, stream):
        try:
            ext = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
            src = torch.as_tensor(_CudaBuf(partial, words), device="cuda")
            dst = torch.as_tensor(_CudaBuf(gathered, words * world), device="cuda")
            with torch.cuda.stream(ext):
                host = src.cpu()  # synchronises the library's stream
                parts = [torch.empty_like(host) for _ in range(world)]
                dist.all_gather(parts, host, group=group)
                dst.copy_(torch.cat(parts).to("cuda"))
            ext.synchronize()
            return 0
        except Exception as e:  # pragma: no cover - surfaced as HS_ENCCL
            print("gloo_device_exchange failed:", e)
            return 1

    return EXCHANGE_FN(fn)
