"""CPU stand-in for ``paper_1908_00041_b200.dist.CudaStages`` built on the numpy
oracle (TEST INFRASTRUCTURE: lets the order-sharded driver — partition,
transposes, compact bins, halos — run under gloo on CPU against the oracle)."""

import numpy as np
import torch

import oracle as O


class OracleStages:
    def __init__(self, L, ring_thetas, ring_weights, n_phi):
        self.L, self.th, self.w, self.n = L, ring_thetas, ring_weights, n_phi

    def fft_fields(self, T_local, S_loc):
        B, nloc, n = S_loc.shape[1], S_loc.shape[2], S_loc.shape[3]
        T = T_local.numpy().reshape(B, nloc, n, 3)
        S_loc.copy_(torch.from_numpy(np.fft.fft(T, axis=2).transpose(3, 0, 1, 2).copy()))

    def ifft_fields(self, S_loc, T_local):
        B, nloc, n = S_loc.shape[1], S_loc.shape[2], S_loc.shape[3]
        T = np.fft.ifft(S_loc.numpy(), axis=3) * n  # favest/scalar.py:178
        T_local.copy_(torch.from_numpy(T.transpose(1, 2, 3, 0).reshape(B, nloc * n, 3).copy()))

    def forward_orders(self, S_own, bin_lo, nb, a, b, legendre, coef):
        B, nth, n = S_own.shape[1], S_own.shape[2], self.n
        Sn = S_own.numpy()
        spec = np.zeros((B, nth, n, 3), dtype=np.complex128)
        for j, m in enumerate(range(bin_lo, bin_lo + nb)):
            spec[:, :, (n - m) % n, :] = Sn[:, :, :, nb + j].transpose(1, 2, 0)
            spec[:, :, m, :] = Sn[:, :, :, j].transpose(1, 2, 0)
        T = np.fft.ifft(spec, axis=2).reshape(B, nth * n, 3)
        ls, ms = O.degrees_orders(self.L)
        sel = (np.abs(ms) >= coef[0]) & (np.abs(ms) < coef[1])
        for f in range(B):
            ra, rb = O.vsht_forward_grid(T[f], self.th, self.w, n, self.L, orders=range(coef[0], coef[1]))
            a[f, torch.from_numpy(sel)] = torch.from_numpy(ra[sel])
            b[f, torch.from_numpy(sel)] = torch.from_numpy(rb[sel])

    def adjoint_orders(self, a, b, orders, S_own):
        B, n = S_own.shape[1], self.n
        nb = orders[1] - orders[0]
        for f in range(B):
            spec = O.vsht_adjoint_grid(a[f].numpy(), b[f].numpy(), self.L, self.th, n,
                                       orders=range(orders[0], orders[1]), spectrum=True)
            for j, m in enumerate(range(orders[0], orders[1])):
                S_own[:, f, :, j] = torch.from_numpy(spec[:, m, :].T.copy())
                if m:
                    S_own[:, f, :, nb + j] = torch.from_numpy(spec[:, (n - m) % n, :].T.copy())

    # packed spectra (dist.py ring-offset tables): gather / scatter around the dense stages
    def _dense_index(self, rtab, B, nb):
        n = len(self.th)
        base = rtab.view(3, B, n, 1)
        return base + torch.arange(2 * nb, dtype=torch.long).view(1, 1, 1, -1)

    def forward_orders_packed(self, flat, rtab, B, bin_lo, nb, a, b, legendre, coef):
        S_own = flat[self._dense_index(rtab, B, nb)]
        self.forward_orders(S_own, bin_lo, nb, a, b, legendre, coef)

    def adjoint_orders_packed(self, a, b, B, orders, flat, rtab, nb):
        S_own = torch.zeros((3, B, len(self.th), 2 * nb), dtype=torch.complex128)
        self.adjoint_orders(a, b, orders, S_own)
        flat[self._dense_index(rtab, B, nb).reshape(-1)] = S_own.reshape(-1)
