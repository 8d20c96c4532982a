"""NCCL communicator behind the C ABI (``ut_comm_*``, ``ut_allgather_f64``,
``ut_allreduce_f32/f64`` in include/undertext_b200.h).

The row-sharded pipelines exchange two small records per step (SURVEY.md
§8(e)): the per-class moment records (an all-gather, combined in rank order
inside K3) and the 2K min/max record (a MAX all-reduce).  With a ``Comm`` both
go through the library's own collective entry points on the current stream,
so a rank's step is a single stream of our kernels and NCCL collectives (and
can be captured into a CUDA graph); without one the pipelines fall back to
``torch.distributed`` collectives (any backend -- gloo for the CPU tests).

    comm = Comm.from_group()            # after torch.distributed.init_process_group
    pipe = CvaPipeline(shard, xs, ys, labels, k=5, comm=comm)
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from . import device as dev


def available() -> int:
    """NCCL version code seen by the library (0: NCCL not loadable)."""
    return int(_lib.lib().ut_comm_available())


class Comm:
    """One NCCL communicator (``world`` ranks, this process is ``rank``)."""

    def __init__(self, unique_id: bytes, world: int, rank: int, device=None):
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.world, self.rank = int(world), int(rank)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        handle = C.c_void_p()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _lib.check(_lib.lib().ut_comm_init(buf, self.world, self.rank, self.device.index or 0,
                                           C.byref(handle)), "ut_comm_init")
        self.handle = handle

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _lib.check(_lib.lib().ut_comm_unique_id(buf), "ut_comm_unique_id")
        return buf.raw

    @classmethod
    def from_group(cls, group=None, device=None) -> "Comm":
        """Create the communicator of a torch.distributed group: group rank 0
        makes the NCCL id, the group's own transport broadcasts it."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        return cls(obj[0], world, rank, device)

    @classmethod
    def single(cls, device=None) -> "Comm":
        """A one-rank communicator (tests, and graph capture of the sharded code)."""
        return cls(cls.unique_id(), 1, 0, device)

    def allgather_f64(self, send: torch.Tensor, recv: torch.Tensor) -> None:
        if send.dtype != torch.float64 or recv.dtype != torch.float64:
            raise TypeError("allgather_f64 needs float64 tensors")
        if recv.numel() != send.numel() * self.world:
            raise ValueError(f"recv has {recv.numel()} elements, need {send.numel() * self.world}")
        _lib.check(_lib.lib().ut_allgather_f64(self.handle, send.data_ptr(), recv.data_ptr(),
                                               send.numel(), dev.stream_handle()),
                   "ut_allgather_f64")

    def allreduce(self, t: torch.Tensor, op: str = "sum") -> None:
        code = {"sum": _lib.UT_OP_SUM, "min": _lib.UT_OP_MIN, "max": _lib.UT_OP_MAX}[op]
        if t.dtype == torch.float64:
            fn, what = _lib.lib().ut_allreduce_f64, "ut_allreduce_f64"
        elif t.dtype == torch.float32:
            fn, what = _lib.lib().ut_allreduce_f32, "ut_allreduce_f32"
        else:
            raise TypeError(f"allreduce supports float32 / float64, got {t.dtype}")
        _lib.check(fn(self.handle, t.data_ptr(), t.numel(), code, dev.stream_handle()), what)

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            _lib.check(_lib.lib().ut_comm_destroy(self.handle), "ut_comm_destroy")
            self.handle = C.c_void_p()

    def __del__(self):  # pragma: no cover - best effort at interpreter exit
        try:
            self.close()
        except Exception:
            pass
