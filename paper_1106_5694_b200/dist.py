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
* :class:`TorchPeerExchange` / :class:`ThreadPeerExchange` -- the peer-memory
  transport: no allgather call at all; the library's pack kernel stores each
  rank's records straight into every replica (NVLink P2P through CUDA IPC
  mappings, or plain pointers for ranks sharing a device) and raises a flag
  there.
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


class _PeerExchange(_Exchange):
    """Peer-memory transport: every rank's receive buffer and flag array mapped here."""

    def __init__(self, rank: int, world: int):
        super().__init__(rank, world)
        self.precv = self.pflags = None
        self._peer_ptrs = None
        self._dev = 0
        self._nbytes = 0
        self.recv_ptr = self.flags_ptr = self.send_ptr = None

    def _alloc(self, ctx):
        """This rank's receive buffer and flags: library allocations (cudaMalloc
        bases, so a CUDA IPC handle maps exactly them), zeroed."""
        import ctypes as C
        nbytes = int(N.LIB.lsapgpu_dist_p2p_bytes(ctx.n, self.world))
        if self._nbytes == nbytes:
            return False
        self.free()
        self._dev = ctx.device
        for attr, size in (("recv_ptr", nbytes), ("flags_ptr", 8 * self.world), ("send_ptr", 16)):
            p = C.c_void_p()
            if N.LIB.lsapgpu_dev_alloc(self._dev, size, C.byref(p)) != 0:
                raise RuntimeError("device allocation for the peer exchange failed")
            setattr(self, attr, p.value)
        self._nbytes = nbytes
        self._peer_ptrs = None
        return True

    def free(self):
        for attr in ("recv_ptr", "flags_ptr", "send_ptr"):
            p = getattr(self, attr, None)
            if p:
                N.LIB.lsapgpu_dev_free(self._dev, p)
            setattr(self, attr, None)
        self._nbytes = 0

    def _peers(self, ctx):  # -> (recv pointers, flag pointers) of every rank
        raise NotImplementedError

    def struct(self, ctx) -> "N.Dist":
        import ctypes as C
        fresh = self._alloc(ctx)
        if fresh or self._peer_ptrs is None:
            rp, fp = self._peers(ctx)
            self.precv = (C.c_void_p * self.world)(*rp)
            self.pflags = (C.c_void_p * self.world)(*fp)
            self._peer_ptrs = (rp, fp)
        d = N.Dist()
        d.rank, d.world = self.rank, self.world
        d.allgather = self._cb
        d.user = None
        d.send_dev = self.send_ptr
        d.recv_dev = self.recv_ptr
        d.peer_recv = C.cast(self.precv, C.POINTER(C.c_void_p))
        d.peer_flags = C.cast(self.pflags, C.POINTER(C.c_void_p))
        return d

    def exchange(self, nbytes: int, stream: int):  # never called: no allgather in this transport
        raise RuntimeError("peer transport has no allgather step")


class ThreadPeerExchange(_PeerExchange):
    """Peer transport for ranks that are threads of one process (tests on one GPU)."""

    def __init__(self, rank: int, world: int, shared: dict):
        super().__init__(rank, world)
        self.shared = shared

    @staticmethod
    def group(world: int):
        shared = {"barrier": threading.Barrier(world), "peers": [None] * world}
        ex = [ThreadPeerExchange(r, world, shared) for r in range(world)]
        shared["peers"] = ex
        return ex

    def _peers(self, ctx):
        self.shared["barrier"].wait()  # every rank allocated its buffers
        peers = self.shared["peers"]
        return [p.recv_ptr for p in peers], [p.flags_ptr for p in peers]


class TorchPeerExchange(_PeerExchange):
    """Peer transport across processes: CUDA IPC handles exchanged over torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist
        super().__init__(dist.get_rank(group), dist.get_world_size(group))
        self.group = group
        self._opened = []

    def _peers(self, ctx):
        import ctypes as C
        import torch.distributed as dist
        mine = []
        for ptr in (self.recv_ptr, self.flags_ptr):
            h = (C.c_char * 64)()
            if N.LIB.lsapgpu_ipc_handle(C.c_void_p(ptr), h) != 0:
                raise RuntimeError("cudaIpcGetMemHandle failed")
            mine.append(bytes(h))
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.group)
        rp, fp = [], []
        for r, (hr, hf) in enumerate(allh):
            if r == self.rank:
                rp.append(self.recv_ptr)
                fp.append(self.flags_ptr)
                continue
            ptrs = []
            for h in (hr, hf):
                p = C.c_void_p()
                if N.LIB.lsapgpu_ipc_open(C.c_char_p(h), C.byref(p)) != 0:
                    raise RuntimeError("cudaIpcOpenMemHandle failed")
                self._opened.append(p.value)
                ptrs.append(p.value)
            rp.append(ptrs[0])
            fp.append(ptrs[1])
        dist.barrier(group=self.group)
        return rp, fp

    def close(self):
        for p in self._opened:
            N.LIB.lsapgpu_ipc_close(p)
        self._opened = []
        self.free()
