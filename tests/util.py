"""Seeded inputs and small oracles shared by the tests (test infrastructure)."""

import numpy as np


def gauss(n, m, seed, cplx=False):
    g = np.random.default_rng(seed)
    x = g.standard_normal((n, m))
    if cplx:
        x = x + 1j * g.standard_normal((n, m))
    return x


def orthonormal(n, m, seed, cplx=False):
    return np.linalg.qr(gauss(n, m, seed, cplx))[0]


def sym_matrix(n, seed, cplx=False):
    a = gauss(n, n, seed, cplx)
    return 0.5 * (a + a.conj().T)


def hpd_matrix(n, seed, cplx=False):
    g = gauss(n, n + 3, seed, cplx)
    return g @ g.conj().T + 0.1 * np.eye(n)


class HostCsr:
    """numpy/scipy operator for the oracle (the product's operators run on the GPU)."""

    def __init__(self, csr):
        self.csr = csr.tocsr()
        self.n = csr.shape[0]
        self.dtype = self.csr.dtype

    def apply(self, block):
        return self.csr @ block


class HostDense:
    def __init__(self, a):
        self.a = 0.5 * (a + a.conj().T)
        self.n = a.shape[0]
        self.dtype = self.a.dtype

    def apply(self, block):
        return self.a @ block


class HostDiag:
    def __init__(self, d):
        self.d = np.asarray(d, dtype=np.float64)
        self.n = self.d.shape[0]

    def apply(self, block):
        return self.d[:, None] * block


def sine_angle(v1, v2):
    """max principal angle (sine form) between orthonormal bases: ||V2 - V1 (V1^H V2)||_2."""
    return float(np.linalg.norm(v2 - v1 @ (v1.conj().T @ v2), 2))
