"""One process per GPU: NCCL communicator for the per-batch exchange.

The communicator's unique id is created on rank 0 by the C ABI
(``lcb_comm_unique_id``) and distributed with ``torch.distributed`` (plumbing
only); the exchange itself — allreduce(max) of the packed (cut, ~member) key and
of the owner's winner bits — runs inside ``libliftcut_b200.so`` on the solve's own
stream (lcb_runtime.cu, Solver::run_batch).

Member sharding: rank r owns global members [r*B, (r+1)*B) of every batch, so an
N-rank solve with batch_size=B is the reference's solve with batch_size=N*B
(member streams are keyed by the global index, init.cpp:80).
"""
from __future__ import annotations

import ctypes as C

from . import _abi


def pack_key(cut: int, global_member: int) -> int:
    """(cut << 32) | (0xffffffff - member): max key = first max (solver.cpp:132-134)."""
    return int(_abi.lib().lcb_pack_key(cut, global_member))


def unpack_key(key: int):
    c, m = C.c_int64(), C.c_int64()
    _abi.lib().lcb_unpack_key(key, C.byref(c), C.byref(m))
    return c.value, m.value


def shard(global_batch: int, nranks: int, rank: int):
    """Contiguous member range of `rank`."""
    if global_batch % nranks:
        raise ValueError("global batch must divide evenly over ranks")
    b = global_batch // nranks
    return rank * b, (rank + 1) * b


class Comm:
    """NCCL communicator over the ranks of one box."""

    def __init__(self, nranks: int, rank: int, device: int, uid: bytes):
        self.nranks, self.rank, self.device = nranks, rank, device
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        st = _abi.lib().lcb_comm_create(buf, nranks, rank, device, C.byref(h))
        if st != 0:
            raise RuntimeError(f"lcb_comm_create: {_abi.last_error()}")
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        st = _abi.lib().lcb_comm_unique_id(buf)
        if st != 0:
            raise RuntimeError(f"lcb_comm_unique_id: {_abi.last_error()}")
        return bytes(buf)

    @classmethod
    def from_torch(cls, device: int):
        """Build the communicator of the current torch.distributed group."""
        import torch.distributed as dist

        world, rank = dist.get_world_size(), dist.get_rank()
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(world, rank, device, obj[0])

    @classmethod
    def loopback(cls, group: "LoopbackGroup", rank: int, device: int = 0) -> "Comm":
        """Rank `rank` of an in-process loopback group (lcb_comm_create_loopback)."""
        c = cls.__new__(cls)
        c.nranks, c.rank, c.device = group.nranks, rank, device
        h = C.c_void_p()
        if _abi.lib().lcb_comm_create_loopback(group.handle, rank, device, C.byref(h)) != 0:
            raise RuntimeError(f"lcb_comm_create_loopback: {_abi.last_error()}")
        c.handle = h
        return c

    def close(self):
        if self.handle:
            _abi.lib().lcb_comm_destroy(self.handle)
            self.handle = None


class LoopbackGroup:
    """`nranks` ranks that are threads of this process (lcb_loopback_create): the solver's
    per-batch collectives run through device staging buffers and a host barrier.  Used to
    run the member-sharded solve on fewer GPUs than ranks (tests)."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        h = C.c_void_p()
        if _abi.lib().lcb_loopback_create(nranks, C.byref(h)) != 0:
            raise RuntimeError(f"lcb_loopback_create: {_abi.last_error()}")
        self.handle = h

    def close(self):
        if self.handle:
            _abi.lib().lcb_loopback_destroy(self.handle)
            self.handle = None
