"""Host-resident field batches through the device transforms, overlapped.

A serving loop whose fields live in host memory pays the host link once per
batch in each direction (for the round trip: the samples in, the synthesised
field out), which on a PCIe-attached B200 costs several times the transforms
themselves.  ``HostPipeline`` hides what can be hidden: batch k+1's
host->device copy, batch k's transforms and batch k-1's device->host copy run
on three CUDA streams against ``depth`` device staging slots (default 3: with
two, batch k+2's upload has to wait for batch k's download, which waits for
batch k's transforms, so the compute is exposed every period), so a stream of
batches is bound by the slower link direction instead of the sum of both
directions plus the compute.  Every batch's bytes still cross the link once
each way (nothing is cached between batches).

The transforms themselves are the plan's (one compute stream, so the plan's
workspaces are never shared by two calls in flight).
"""

from .plan import GridPlan


def _torch():
    import torch

    return torch


class HostPipeline:
    """Pipelined forward / adjoint / round trip of pinned host batches.

    ``submit_*`` calls return immediately; results land in the caller's pinned
    output buffers once :meth:`synchronize` returns (or the returned event
    completes).  The caller must not overwrite an input buffer, or read an
    output buffer, before then.
    """

    def __init__(self, plan: GridPlan, depth: int = 3):
        torch = _torch()
        self.plan = plan
        self.depth = max(1, int(depth))
        dev = plan.device
        B, N, K = plan.max_batch, plan.n_points, plan.n_coeffs
        self.h2d = torch.cuda.Stream(dev)
        self.comp = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        c128 = torch.complex128
        self._slots = []
        for _ in range(self.depth):
            self._slots.append({
                "T": torch.empty((B, N, 3), dtype=c128, device=dev),
                "Tout": torch.empty((B, N, 3), dtype=c128, device=dev),
                "a": torch.empty((B, K), dtype=c128, device=dev),
                "b": torch.empty((B, K), dtype=c128, device=dev),
                "loaded": torch.cuda.Event(), "done": torch.cuda.Event(), "free": torch.cuda.Event(),
            })
        self._k = 0

    @staticmethod
    def _pinned(x, name):
        if x.device.type != "cpu" or not x.is_pinned():
            raise ValueError(f"{name} must be a pinned host tensor (torch.empty(..., pin_memory=True))")
        return x

    def _slot(self):
        s = self._slots[self._k % self.depth]
        self._k += 1
        return s

    def _stage(self, s, srcs):
        torch = _torch()
        with torch.cuda.stream(self.h2d):
            self.h2d.wait_event(s["free"])  # the slot's previous batch has fully drained
            for dst, src in srcs:
                dst.copy_(src, non_blocking=True)
            s["loaded"].record(self.h2d)

    def _drain(self, s, pairs):
        torch = _torch()
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(s["done"])
            for dst, src in pairs:
                dst.copy_(src, non_blocking=True)
            s["free"].record(self.d2h)
        return s["free"]

    def submit_roundtrip(self, T_host, T_out_host):
        """forward then adjoint of a (B, N, 3) pinned batch -> (B, N, 3) pinned output."""
        torch = _torch()
        self._pinned(T_host, "T_host")
        self._pinned(T_out_host, "T_out_host")
        B = int(T_host.shape[0])
        s = self._slot()
        self._stage(s, [(s["T"][:B], T_host)])
        with torch.cuda.stream(self.comp):
            self.comp.wait_event(s["loaded"])
            a, b = self.plan.forward(s["T"][:B], s["a"][:B], s["b"][:B])
            self.plan.adjoint(a, b, s["Tout"][:B])
            s["done"].record(self.comp)
        return self._drain(s, [(T_out_host, s["Tout"][:B])])

    def submit_forward(self, T_host, a_host, b_host):
        """(B, N, 3) pinned samples -> (B, K) pinned div / curl coefficients."""
        torch = _torch()
        for x, n in ((T_host, "T_host"), (a_host, "a_host"), (b_host, "b_host")):
            self._pinned(x, n)
        B = int(T_host.shape[0])
        s = self._slot()
        self._stage(s, [(s["T"][:B], T_host)])
        with torch.cuda.stream(self.comp):
            self.comp.wait_event(s["loaded"])
            self.plan.forward(s["T"][:B], s["a"][:B], s["b"][:B])
            s["done"].record(self.comp)
        return self._drain(s, [(a_host, s["a"][:B]), (b_host, s["b"][:B])])

    def submit_adjoint(self, a_host, b_host, T_out_host):
        """(B, K) pinned coefficients -> (B, N, 3) pinned field."""
        torch = _torch()
        for x, n in ((a_host, "a_host"), (b_host, "b_host"), (T_out_host, "T_out_host")):
            self._pinned(x, n)
        B = int(a_host.shape[0])
        s = self._slot()
        self._stage(s, [(s["a"][:B], a_host), (s["b"][:B], b_host)])
        with torch.cuda.stream(self.comp):
            self.comp.wait_event(s["loaded"])
            self.plan.adjoint(s["a"][:B], s["b"][:B], s["Tout"][:B])
            s["done"].record(self.comp)
        return self._drain(s, [(T_out_host, s["Tout"][:B])])

    def synchronize(self):
        self.d2h.synchronize()
