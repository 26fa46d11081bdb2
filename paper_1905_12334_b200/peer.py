"""Peer-memory plumbing for the data-parallel exchange on one node.

``PeerBuffer`` is a device buffer every rank of the process group maps
(``fp8b_peer_alloc`` = cudaMalloc + IPC handle; the 64-byte handles travel over
the group with ``all_gather_object``). ``reduce_quantize`` launches the fused
rank-order sum + Q node kernel (``csrc/peer.cu``) over the ranks' mappings: the
owner of a shard reads every rank's FP32 partial straight over NVLink / NVSwitch
and writes E5M2 codes -- no FP32 sum makes a round trip through HBM and no NCCL
reduce-scatter runs. Kernels never wait on a peer; ``fence`` orders the steps on
the host (stream sync + group barrier).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import torch
import torch.distributed as dist

from . import _lib
from . import Counters, _BITS, _fmt, _mode, _stream
from ._lib import LIB, check

HANDLE_BYTES = 64


class _Raw:
    """__cuda_array_interface__ view of raw device memory (bytes)."""

    def __init__(self, ptr: int, nbytes: int, owner):
        self.owner = owner
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 2}


class PeerBuffer:
    """nbytes of device memory mapped by every rank of `group` (one node)."""

    def __init__(self, nbytes: int, group=None):
        self.nbytes = int(nbytes)
        self.group = group
        distributed = dist.is_initialized()
        self.world = dist.get_world_size(group) if distributed else 1
        self.rank = dist.get_rank(group) if distributed else 0
        p = C.c_void_p()
        h = C.create_string_buffer(HANDLE_BYTES)
        check(LIB.fp8b_peer_alloc(C.byref(p), self.nbytes, h), "peer_alloc")
        self._own = p.value
        self.ptrs: List[int] = [0] * self.world
        self.ptrs[self.rank] = self._own
        self._opened: List[int] = []
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(h.raw), group=group)
            for r, hr in enumerate(handles):
                if r == self.rank:
                    continue
                q = C.c_void_p()
                check(LIB.fp8b_peer_open(hr, C.byref(q)), "peer_open")
                self.ptrs[r] = q.value
                self._opened.append(q.value)
        self._views = {}

    def view(self, rank: Optional[int] = None) -> torch.Tensor:
        """uint8 tensor over rank's buffer (own buffer by default)."""
        r = self.rank if rank is None else rank
        if r not in self._views:
            self._views[r] = torch.as_tensor(_Raw(self.ptrs[r], self.nbytes, self),
                                             device=torch.device("cuda", torch.cuda.current_device()))
        return self._views[r]

    def close(self) -> None:
        self._views.clear()
        for q in self._opened:
            LIB.fp8b_peer_close(q)
        self._opened = []
        if self._own:
            LIB.fp8b_peer_free(self._own)
            self._own = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fence(group=None) -> None:
    """Every rank's queued work is done and visible before any rank goes on."""
    torch.cuda.synchronize()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.barrier(group=group)


def reduce_quantize(peer_ptrs: List[int], i0: int, n: int, codes: torch.Tensor, *,
                    fmt: str = "fp8", mode: str = "nearest-even", seed: int = 1,
                    block_offset: int = 0, saturate: bool = False,
                    counters: Optional[Counters] = None,
                    sum_out: Optional[torch.Tensor] = None, stream=None) -> None:
    """codes[i] = Q(sum_r peers[r][i0 + i]) for i in [0, n), ranks summed in order
    (fp8b_peer_reduce_quantize). peer_ptrs: device pointers to every rank's FP32
    buffer (PeerBuffer.ptrs)."""
    world = len(peer_ptrs)
    arr = (C.c_void_p * world)(*peer_ptrs)
    cfg = _lib.QuantConfig(_mode(mode), _BITS["counter"], int(seed), int(bool(saturate)), 0,
                           int(block_offset), None)
    check(LIB.fp8b_peer_reduce_quantize(arr, world, int(i0), int(n),
                                        sum_out.data_ptr() if sum_out is not None else None,
                                        codes.data_ptr(), _fmt(fmt), cfg,
                                        counters.ptr if counters is not None else None,
                                        _stream(stream)), "peer_reduce_quantize")
