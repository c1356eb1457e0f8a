"""Seeded synthetic workloads shaped like the paper's datasets.

This module is shared by the tests, the bench and the oracle's inputs.  It
holds NONE of the method's arithmetic: it only draws vectors.  The real
datasets of the paper (Table 2) are not available; these
generators stand in for them.

All generators are torch-based so the same code runs on CPU (tests) and on the
GPU (bench, large configs).  Determinism: every chunk of ``CHUNK`` rows draws
from its own ``torch.Generator`` seeded by (config seed, stream, chunk), so the
output does not depend on how many rows are requested at once.  The CPU and
CUDA generators produce different (but each deterministic) streams; a given
test or bench run uses one device for generation and copies to the other.
"""
from __future__ import annotations

import math

import torch

CHUNK = 4096

# BASELINE.json configs (index 0..4) -> shape and seed
CONFIGS = {
    1: dict(name="cfg1-pr1", N=20_000, D=256, Q=100, k=10, seed=0, modes=(0,)),
    2: dict(name="cfg2-gist-like", N=1_000_000, D=960, Q=10_000, k=10, seed=1, modes=(0, 1)),
    3: dict(name="cfg3-isotropic", N=1_000_000, D=1024, Q=10_000, k=10, seed=2, modes=(1,)),
    4: dict(name="cfg4-text-like", N=2_000_000, D=3072, Q=10_000, k=100, seed=3, modes=(0, 1)),
    5: dict(name="cfg5-descriptor-like", N=2_000_000, D=4096, Q=10_000, k=10, seed=4, modes=(0, 1)),
}

S_BASE, S_QUERY, S_BASIS, S_SPECTRUM, S_CENTERS, S_LABELS, S_SIGNS = 11, 12, 13, 14, 15, 16, 17


def _gen(device, seed: int, stream: int, chunk: int = 0) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + stream * 7_919 + chunk * 104_729) & 0x7FFF_FFFF_FFFF_FFFF)
    return g


def _basis(D: int, r: int, seed: int, device) -> torch.Tensor:
    """U = Q of QR(Gaussian D x r), diag(R) > 0 (App. B common rules)."""
    g = _gen("cpu", seed, S_BASIS)
    G = torch.randn(D, r, generator=g, dtype=torch.float64)
    Qm, Rm = torch.linalg.qr(G)
    Qm = Qm * torch.sign(torch.diagonal(Rm)).unsqueeze(0)
    return Qm.to(device)


def _fwht(x: torch.Tensor) -> torch.Tensor:
    """Normalised Walsh-Hadamard transform along the last dim (power of two)."""
    n = x.shape[-1]
    h = 1
    y = x.clone()
    while h < n:
        y = y.view(*x.shape[:-1], n // (2 * h), 2, h)
        a, b = y[..., 0, :], y[..., 1, :]
        y = torch.stack((a + b, a - b), dim=-2).reshape(*x.shape[:-1], n)
        h *= 2
    return y / math.sqrt(n)


class Workload:
    """Generator for one config; ``rows(start, n, kind)`` draws rows [start, start+n)."""

    def __init__(self, cfg: int, device="cpu", D: int | None = None):
        self.cfg = cfg
        c = CONFIGS[cfg]
        self.D = D or c["D"]
        self.seed = c["seed"]
        self.device = torch.device(device)
        D, seed, dev = self.D, self.seed, self.device
        if cfg == 1:
            self.r = 16
            self.U = _basis(D, self.r, seed, dev)
            self.lam = torch.arange(1, self.r + 1, dtype=torch.float64, device=dev) ** -1.5
        elif cfg == 2:
            self.r = max(1, D // 20)  # top 5% of dimensions
            self.U = _basis(D, self.r, seed, dev)
            self.sig_s = math.sqrt(0.9 * D / self.r)
            self.sig_n = math.sqrt(0.1 * D / (D - self.r))
            g = _gen("cpu", seed, S_CENTERS)
            gc = torch.randn(64, self.r, generator=g, dtype=torch.float64).to(dev)
            self.mu = 2.0 * (gc * self.sig_s) @ self.U.T  # 64 x D
        elif cfg == 3:
            g = _gen("cpu", seed, S_SPECTRUM)
            self.lam = (0.8 + 0.4 * torch.rand(D, generator=g, dtype=torch.float64)).to(dev)
        elif cfg == 4:
            self.r = min(256, D)
            self.U = _basis(D, self.r, seed, dev)
            self.lam = torch.arange(1, self.r + 1, dtype=torch.float64, device=dev) ** -1.0
            # noise variance per dim so that noise carries f = 0.1 of the total variance
            f = 0.1
            self.sig_n = math.sqrt(f / (1 - f) * float(self.lam.sum()) / D)
        elif cfg == 5:
            assert D & (D - 1) == 0, "cfg5 needs a power-of-two D (Walsh-Hadamard)"
            self.lam = torch.arange(1, D + 1, dtype=torch.float64, device=dev) ** -1.0
            g = _gen("cpu", seed, S_SIGNS)
            self.signs = (torch.randint(0, 2, (D,), generator=g) * 2 - 1).to(torch.float64).to(dev)
        else:
            raise ValueError(cfg)

    def _chunk(self, n: int, stream: int, chunk: int) -> torch.Tensor:
        g = _gen(self.device, self.seed, stream, chunk)
        dev, D, f64 = self.device, self.D, torch.float64
        if self.cfg == 1:
            z = torch.randn(n, self.r, generator=g, device=dev, dtype=f64)
            e = torch.randn(n, D, generator=g, device=dev, dtype=f64)
            x = (z * self.lam.sqrt()) @ self.U.T + 0.05 * e
        elif self.cfg == 2:
            lab = torch.randint(0, 64, (n,), generator=g, device=dev)
            z = torch.randn(n, self.r, generator=g, device=dev, dtype=f64)
            e = torch.randn(n, D, generator=g, device=dev, dtype=f64)
            x = self.mu[lab] + (z * self.sig_s) @ self.U.T + self.sig_n * e
        elif self.cfg == 3:
            z = torch.randn(n, D, generator=g, device=dev, dtype=f64)
            x = z * self.lam.sqrt()
            x = x / x.norm(dim=1, keepdim=True)
        elif self.cfg == 4:
            z = torch.randn(n, self.r, generator=g, device=dev, dtype=f64)
            e = torch.randn(n, D, generator=g, device=dev, dtype=f64)
            x = (z * self.lam.sqrt()) @ self.U.T + self.sig_n * e
            x = x / x.norm(dim=1, keepdim=True)
        else:
            z = torch.randn(n, D, generator=g, device=dev, dtype=f64)
            x = torch.relu(self.signs * _fwht(z * self.lam.sqrt()))
        return x.to(torch.float32)

    def rows(self, start: int, n: int, kind: str = "base", out: torch.Tensor | None = None) -> torch.Tensor:
        stream = S_BASE if kind == "base" else S_QUERY
        if out is None:
            out = torch.empty(n, self.D, dtype=torch.float32, device=self.device)
        pos = 0
        while pos < n:
            gi = start + pos
            ch, off = divmod(gi, CHUNK)
            take = min(CHUNK - off, n - pos)
            block = self._chunk(CHUNK, stream, ch) if (off or take < CHUNK) else None
            if block is None:
                out[pos:pos + take] = self._chunk(CHUNK, stream, ch)
            else:
                out[pos:pos + take] = block[off:off + take]
            pos += take
        return out

    def base(self, N: int, out=None):
        return self.rows(0, N, "base", out)

    def queries(self, Q: int, out=None):
        return self.rows(0, Q, "query", out)
