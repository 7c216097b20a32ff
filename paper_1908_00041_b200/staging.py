"""Host <-> device copies of the drop-in entry points' numpy arrays.

``forward_favest`` / ``adjoint_favest`` take and return ordinary (pageable)
numpy arrays, as the reference does.  A pageable array cannot be DMA'd
directly, so a plain ``torch.from_numpy(x).to(dev)`` makes the driver stage it
through its own small pinned buffers one block at a time, and the reverse copy
likewise.  ``Stager`` does the staging itself, pipelined: the array is cut into
chunks; chunk k is memcpy'd (torch's multi-threaded CPU copy) into one of a few
resident pinned slots while chunk k-1's DMA runs on the caller's stream, and on
the way back chunk k's DMA overlaps the host copy of chunk k-1 out of its slot.
Results are written into fresh pageable numpy arrays, so nothing the caller
keeps stays page-locked; the pinned slots (``SLOTS`` x ``CHUNK`` bytes per
device) are the only pinned memory and are reused by every call.

One stager per device, serialised by its lock (the slots are shared).
"""

from __future__ import annotations

import threading
from collections import deque

import numpy as np

CHUNK = 16 << 20
SLOTS = 3
SMALL = 4 << 20  # below this a direct copy is as fast

_STAGERS: dict = {}
_STAGERS_LOCK = threading.Lock()


def _torch():
    import torch

    return torch


def _bytes_view(t):
    torch = _torch()
    return t.reshape(-1).view(torch.uint8)


class Stager:
    def __init__(self, device):
        torch = _torch()
        self.device = device
        self.lock = threading.Lock()
        self.slots = [torch.empty(CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(SLOTS)]
        self.ready = [None] * SLOTS  # event: the slot's last DMA has completed

    def to_device(self, arr: np.ndarray, out=None):
        """numpy array -> new (or ``out``) contiguous device tensor, same shape / dtype.
        The copies are enqueued on the current stream; the call returns once the
        host side is done (the array may then be modified)."""
        torch = _torch()
        src = torch.from_numpy(np.ascontiguousarray(arr))
        if out is None:
            out = torch.empty(src.shape, dtype=src.dtype, device=self.device)
        nbytes = src.numel() * src.element_size()
        if nbytes < SMALL:
            out.copy_(src)
            return out
        sb, db = _bytes_view(src), _bytes_view(out)
        stream = torch.cuda.current_stream(self.device)
        with self.lock:
            for k, off in enumerate(range(0, nbytes, CHUNK)):
                s = k % SLOTS
                n = min(CHUNK, nbytes - off)
                if self.ready[s] is not None:
                    self.ready[s].synchronize()  # the slot's previous DMA has read it
                slot = self.slots[s][:n]
                slot.copy_(sb[off:off + n])
                db[off:off + n].copy_(slot, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                self.ready[s] = ev
            # the slots stay owned by the enqueued DMAs; the next call waits on self.ready
        return out

    def to_host(self, x) -> np.ndarray:
        """Device tensor -> new pageable numpy array (waits for the copy)."""
        torch = _torch()
        x = x.contiguous()
        out = np.empty(tuple(x.shape), dtype=torch.empty((), dtype=x.dtype).numpy().dtype)
        nbytes = x.numel() * x.element_size()
        if nbytes < SMALL:
            torch.from_numpy(out).copy_(x)
            return out
        sb, db = _bytes_view(x), _bytes_view(torch.from_numpy(out))
        stream = torch.cuda.current_stream(self.device)
        with self.lock:
            pending = deque()

            def drain_one():
                s, off, n, ev = pending.popleft()
                ev.synchronize()
                db[off:off + n].copy_(self.slots[s][:n])

            for k, off in enumerate(range(0, nbytes, CHUNK)):
                s = k % SLOTS
                n = min(CHUNK, nbytes - off)
                if len(pending) == SLOTS:
                    drain_one()  # frees slot s (its previous chunk)
                if self.ready[s] is not None:
                    self.ready[s].synchronize()  # an upload's DMA may still read the slot
                self.slots[s][:n].copy_(sb[off:off + n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                self.ready[s] = ev
                pending.append((s, off, n, ev))
            while pending:
                drain_one()
        return out


def stager(device) -> Stager:
    with _STAGERS_LOCK:
        st = _STAGERS.get(str(device))
        if st is None:
            st = _STAGERS[str(device)] = Stager(device)
        return st
