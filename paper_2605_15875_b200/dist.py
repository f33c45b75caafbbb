"""Partition-per-GPU runs over torch.distributed.

The reference runs one worker thread per partition and a controller that
exchanges messages over a Transport (proj/src/runtime.cpp:110-694,
proj/include/dabd/transport.hpp:15-40). Here each rank (one process per GPU)
owns a contiguous range of partitions and its engine calls two hooks of
`dabd_gpu_comm` (include/dabd_gpu.h):

* ``halo``      -- once per ADMM iteration, the split-body replicas (q, u, rho)
                   a neighbouring rank pairs with: point-to-point with rank-1
                   and rank+1 only (NVLink P2P under NCCL);
* ``allgather`` -- once per ADMM iteration the controller fan-in record
                   (per partition dq, r, s, earliest merge TOI and a failure
                   flag), and once per frame the committed global state.

With the NCCL backend the engine's device buffers go to NCCL on the engine's
own stream. With gloo (the CPU tests, or several ranks sharing one GPU) they
are staged through host memory. The exchange carries no arithmetic: both
ranks of a split body evaluate the consensus in the same order, so a run on
N ranks is bitwise the run of the same partitions on one GPU.
"""

from __future__ import annotations

import ctypes as C
from contextlib import nullcontext
from typing import List, Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L


def partition_offsets(num_workers: int, world: int) -> List[int]:
    """Contiguous near-equal split of the partitions over the ranks."""
    if world < 1 or num_workers < world:
        raise ValueError(f"need at least one partition per rank ({num_workers} < {world})")
    base, extra = divmod(num_workers, world)
    out = [0]
    for r in range(world):
        out.append(out[-1] + base + (1 if r < extra else 0))
    return out


class _CudaArray:
    def __init__(self, ptr: int, n: int) -> None:
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class TorchComm:
    """dabd_gpu_comm over a torch.distributed process group."""

    def __init__(self, num_workers: int, device: Optional[int] = None, group=None) -> None:
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = str(dist.get_backend(group))
        self.device = device
        self.offsets = partition_offsets(num_workers, self.world)
        self.part_begin = self.offsets[self.rank]
        self.part_end = self.offsets[self.rank + 1]
        self.error: Optional[BaseException] = None
        self._halo_cb = L.HaloFn(self._halo_c)
        self._allgather_cb = L.AllgatherFn(self._allgather_c)
        self._offs = (C.c_int * (self.world + 1))(*self.offsets)
        self.struct = L.Comm(None, self._halo_cb, self._allgather_cb, self.rank, self.world,
                             C.cast(self._offs, C.POINTER(C.c_int)))

    # ---- tensor-level exchange (testable on CPU tensors) --------------------
    def _peer(self, r: int) -> int:
        return r if self.group is None else dist.get_global_rank(self.group, r)

    def halo(self, send_lo: torch.Tensor, recv_lo: torch.Tensor, send_hi: torch.Tensor,
             recv_hi: torch.Tensor) -> None:
        """send_lo -> rank-1, rank-1 -> recv_lo; send_hi -> rank+1, rank+1 -> recv_hi."""
        pairs = []
        if send_lo.numel():
            pairs.append((send_lo, recv_lo, self.rank - 1))
        if send_hi.numel():
            pairs.append((send_hi, recv_hi, self.rank + 1))
        if not pairs:
            return
        staged = self.backend != "nccl" and pairs[0][0].is_cuda
        ops, back = [], []
        for s, r, peer in pairs:
            if not 0 <= peer < self.world:
                raise RuntimeError(f"halo: rank {self.rank} has no neighbour {peer}")
            if staged:
                s_, r_ = s.cpu(), torch.empty(r.numel(), dtype=r.dtype)
                back.append((r, r_))
            else:
                s_, r_ = s, r
            ops.append(dist.P2POp(dist.isend, s_, self._peer(peer), self.group))
            ops.append(dist.P2POp(dist.irecv, r_, self._peer(peer), self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for r, r_ in back:
            r.copy_(r_)

    def allgather(self, send: torch.Tensor, recv: torch.Tensor) -> None:
        """recv[r * n:(r + 1) * n] = send of rank r."""
        n = send.numel()
        if self.backend == "nccl":
            dist.all_gather_into_tensor(recv, send, group=self.group)
            return
        src = send.cpu() if send.is_cuda else send
        parts = [torch.empty(n, dtype=send.dtype) for _ in range(self.world)]
        dist.all_gather(parts, src, group=self.group)
        recv.copy_(torch.cat(parts))

    # ---- C callbacks (device pointers on the engine's stream) ----------------
    def _view(self, ptr: Optional[int], n: int) -> torch.Tensor:
        if n == 0 or not ptr:
            return torch.empty(0, dtype=torch.float64, device=self._dev())
        return torch.as_tensor(_CudaArray(ptr, n), device=self._dev())

    def _dev(self) -> torch.device:
        return torch.device("cuda", torch.cuda.current_device() if self.device is None else self.device)

    def _on(self, stream: int):
        if not stream:
            return nullcontext()
        return torch.cuda.stream(torch.cuda.ExternalStream(stream, device=self._dev()))

    def _halo_c(self, _user, s_lo, r_lo, n_lo, s_hi, r_hi, n_hi, stream) -> int:
        try:
            with self._on(stream):
                self.halo(self._view(s_lo, n_lo), self._view(r_lo, n_lo),
                          self._view(s_hi, n_hi), self._view(r_hi, n_hi))
            return 0
        except BaseException as e:  # no exception may cross the C ABI
            self.error = e
            return 1

    def _allgather_c(self, _user, send, recv, count, stream) -> int:
        try:
            with self._on(stream):
                self.allgather(self._view(send, count), self._view(recv, count * self.world))
            return 0
        except BaseException as e:
            self.error = e
            return 1


def run_partitioned(scene, workers: int, frames: int, device: int = 0, group=None, **solver):
    """This rank's share of a `workers`-partition consensus-ADMM run
    (runtime.cpp:110-694 semantics); every rank returns the same committed
    global trajectory and trace. rho is NaN outside this rank's partitions."""
    from . import api

    comm = TorchComm(workers, device=device, group=group)
    sc = api.Scene(scene)
    ctx = api.Context(sc, device=device, num_workers=workers, part_begin=comm.part_begin,
                      part_end=comm.part_end, **solver)
    ctx.set_comm(comm)
    run_partitioned.last_comm_mode = ctx.comm_mode()
    qs, qds, hs, stats = [], [], [], []
    for _ in range(frames):
        st = ctx.run_frames(1)[0]
        q, qd = ctx.state()
        qs.append(q)
        qds.append(qd)
        hs.append(st["h"])
        stats.append(st)
    return api.Trajectory(np.array(qs).reshape(frames, sc.n, 6),
                          np.array(qds).reshape(frames, sc.n, 6), np.array(hs), stats,
                          ctx.take_trace(), ctx.rho())
