"""Multi-GPU plumbing for ``Context.solve(dist=...)``.

One process per GPU, each holding the full instance.  The library owns the
algorithm (item ownership by agent index, record pack / merge, replicated
commit); this module only supplies the exchange step it calls once per scan:

* :class:`TorchDistExchange` -- ``torch.distributed.all_gather_into_tensor`` on
  the solver's own CUDA stream (NCCL over NVLink / NVSwitch when the process
  group backend is ``nccl``).
* :class:`ThreadExchange` -- several ranks as threads of one process on one
  device (device-to-device copies through a barrier): exercises the exact
  multi-rank code path on a single GPU, for tests.
"""
from __future__ import annotations

import threading

from . import _native as N


class _Exchange:
    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world
        self._cb = N.ALLGATHER_FN(self._call)
        self._error = None
        self.send = self.recv = None
        self.calls = 0

    def _buffers(self, ctx):
        import torch
        nbytes = int(N.LIB.lsapgpu_dist_exchange_bytes(ctx.n, self.world))
        if self.send is None or self.send.numel() != nbytes:
            dev = torch.device("cuda", ctx.device)
            self.send = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
            self.recv = torch.zeros(nbytes * self.world, dtype=torch.uint8, device=dev)
            torch.cuda.synchronize(dev)
        return nbytes

    def struct(self, ctx) -> "N.Dist":
        self._buffers(ctx)
        d = N.Dist()
        d.rank, d.world = self.rank, self.world
        d.allgather = self._cb
        d.user = None
        d.send_dev = self.send.data_ptr()
        d.recv_dev = self.recv.data_ptr()
        return d

    def _call(self, user, send, recv, nbytes, stream):
        try:
            self.calls += 1
            self.exchange(int(nbytes), int(stream or 0))
            return 0
        except BaseException as e:  # noqa: BLE001 -- surfaced by raise_pending
            self._error = e
            return 1

    def raise_pending(self):
        if self._error is not None:
            e, self._error = self._error, None
            raise e

    def exchange(self, nbytes: int, stream: int):
        raise NotImplementedError


class TorchDistExchange(_Exchange):
    """Allgather over the default torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        super().__init__(dist.get_rank(group), dist.get_world_size(group))
        self.group = group

    def exchange(self, nbytes: int, stream: int):
        import torch
        import torch.distributed as dist
        s = torch.cuda.ExternalStream(stream, device=self.send.device)
        if dist.get_backend(self.group) == "nccl":
            with torch.cuda.stream(s):
                dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
            return
        # host-staged exchange for CPU backends (gloo: several ranks per GPU in tests)
        s.synchronize()
        send = self.send.cpu()
        recv = torch.empty(send.numel() * self.world, dtype=send.dtype)
        dist.all_gather_into_tensor(recv, send, group=self.group)
        with torch.cuda.stream(s):
            self.recv.copy_(recv, non_blocking=False)


class ThreadExchange(_Exchange):
    """Ranks as threads of one process (one context each, same or different devices)."""

    def __init__(self, rank: int, world: int, shared: dict):
        super().__init__(rank, world)
        self.shared = shared  # {"barrier": threading.Barrier(world), "peers": [exchange objects]}

    @staticmethod
    def group(world: int):
        shared = {"barrier": threading.Barrier(world), "peers": [None] * world}
        ex = [ThreadExchange(r, world, shared) for r in range(world)]
        shared["peers"] = ex
        return ex

    def exchange(self, nbytes: int, stream: int):
        import torch
        s = torch.cuda.ExternalStream(stream, device=self.send.device)
        s.synchronize()  # our packed records are complete
        self.shared["barrier"].wait()
        with torch.cuda.stream(s):
            for r, peer in enumerate(self.shared["peers"]):
                self.recv[r * nbytes:(r + 1) * nbytes].copy_(peer.send[:nbytes], non_blocking=True)
        s.synchronize()
        self.shared["barrier"].wait()  # nobody repacks before every peer copied
