"""Seeded synthetic stand-ins for the BASELINE.json configs (the paper's datasets are not in the
container).  Generators follow the shapes and value distributions BASELINE.json states; they are
workload definitions, not part of the factorisation path.

  C1  exact low-rank 2000 x 1000, rank 20, fp64, k=20 p=10 q=2, 100 sweeps
  C2  face-image-like 32256 x 2410 (192x168 px), 16 Gaussian "parts", fp32, k=16 p=20 q=2, 200 sweeps
  C3  spectral-unmixing-like 1,048,576 x 256, 10 endmembers, fp32, k=10 p=10 q=2, 300 sweeps
  C4  noisy low-rank 200,000 x 20,000, rank 40, fp32, k=40 p=20 q=2, 200 sweeps
  C5  box-scale 500,000 x 100,000, rank 64, fp32 (multi-GPU only), k=64 p=32 q=3, 100 sweeps
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    k: int
    p: int
    q: int
    iters: int
    dtype: str


CONFIGS = {
    "C1": Config("C1-exact-lowrank-2000x1000-r20", 2000, 1000, 20, 10, 2, 100, "f64"),
    "C2": Config("C2-faces-32256x2410-k16", 32256, 2410, 16, 20, 2, 200, "f32"),
    "C3": Config("C3-unmixing-1048576x256-k10", 1048576, 256, 10, 10, 2, 300, "f32"),
    "C4": Config("C4-noisy-lowrank-200000x20000-r40", 200000, 20000, 40, 20, 2, 200, "f32"),
    "C5": Config("C5-box-500000x100000-r64", 500000, 100000, 64, 32, 3, 100, "f32"),
}


def c1_matrix(seed: int = 0, m: int = 2000, n: int = 1000, rank: int = 20) -> np.ndarray:
    """X = W0 H0 with W0, H0 = |N(0,1)| (fp64)."""
    rng = np.random.default_rng(seed)
    w0 = np.abs(rng.standard_normal((m, rank)))
    h0 = np.abs(rng.standard_normal((rank, n)))
    return w0 @ h0


def faces_matrix(seed: int = 0, height: int = 192, width: int = 168, n: int = 2410, parts: int = 16,
                 dtype=np.float32) -> np.ndarray:
    """Each column is a nonnegative mixture of `parts` 2-D Gaussian blobs (sigma 5-25 px, weights
    |N(0,1)|) plus |N(0, 0.02)| noise, scaled to [0, 1].  Shape (height*width) x n."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:height, 0:width]
    basis = np.empty((height * width, parts), dtype=np.float64)
    for i in range(parts):
        cy, cx = rng.uniform(0, height), rng.uniform(0, width)
        sig = rng.uniform(5.0, 25.0)
        basis[:, i] = np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * sig * sig)).ravel()
    mix = np.abs(rng.standard_normal((parts, n)))
    x = (basis @ mix).astype(dtype)
    x += np.abs(rng.standard_normal(x.shape, dtype=np.float32) * 0.02).astype(dtype)
    x /= x.max()
    return np.ascontiguousarray(x, dtype=dtype)


def unmixing_matrix(seed: int = 0, m: int = 1048576, n: int = 256, ends: int = 10, dtype=np.float32) -> np.ndarray:
    """X = A E + |N(0, 0.01)|, A (m x ends) Dirichlet(0.5) rows, E (ends x n) smooth spectra: sums of
    3 Gaussians over the band index with amplitudes U(0.1, 1)."""
    rng = np.random.default_rng(seed)
    a = rng.dirichlet(np.full(ends, 0.5), size=m)
    band = np.arange(n)
    e = np.zeros((ends, n))
    for i in range(ends):
        for _ in range(3):
            c = rng.uniform(0, n)
            w = rng.uniform(n / 50, n / 6)
            e[i] += rng.uniform(0.1, 1.0) * np.exp(-((band - c) ** 2) / (2 * w * w))
    x = (a @ e).astype(dtype)
    x += np.abs(rng.standard_normal(x.shape, dtype=np.float32) * 0.01).astype(dtype)
    return np.ascontiguousarray(x)


def noisy_lowrank_matrix(seed: int, m: int, n: int, rank: int, sparsity: float, noise_frac: float,
                         dtype=np.float32) -> np.ndarray:
    """C4/C5 generator on the host (small slices): X = W0 H0 + |N(0, noise_frac*mean)| with W0, H0
    |N(0,1)| and a Bernoulli(sparsity) zero mask."""
    rng = np.random.default_rng(seed)
    w0 = np.abs(rng.standard_normal((m, rank))) * (rng.random((m, rank)) >= sparsity)
    h0 = np.abs(rng.standard_normal((rank, n))) * (rng.random((rank, n)) >= sparsity)
    x = w0 @ h0
    x += np.abs(rng.standard_normal(x.shape) * (noise_frac * x.mean()))
    return np.ascontiguousarray(x.astype(dtype))


GEN_BLOCK_ROWS = 4096


def lowrank_expected_mean(rank: int, sparsity: float) -> float:
    """E[(W0 H0)_ij] for W0, H0 = |N(0,1)| with a Bernoulli(sparsity) zero mask:
    rank * (1 - sparsity)^2 * E|N(0,1)|^2 = rank * (1 - sparsity)^2 * 2 / pi."""
    return rank * (1.0 - sparsity) ** 2 * 2.0 / np.pi


def noisy_lowrank_shard(seed: int, m: int, n: int, rank: int, sparsity: float, noise_frac: float, row0: int,
                        rows: int, device="cuda", block: int = GEN_BLOCK_ROWS):
    """Rows [row0, row0 + rows) of the m x n C4/C5 matrix X = W0 H0 + |N(0, noise_frac * mean)|, generated
    on the device without materialising any other rows (counter-based, keyed by
    (seed, global row block), so every shard count produces the same global X).

    * H0 (rank x n) = |N(0,1)| * Bernoulli mask from a generator keyed by the seed alone
      (replicated on every rank);
    * global row block b (rows [b*block, (b+1)*block)) draws its W0 rows and its noise from a
      generator keyed by (seed, b);
    * the noise scale uses the expected mean of W0 H0 (lowrank_expected_mean), which needs no
      pass over the whole matrix.
    fp32 on `device`; the GEMM W0_rows H0 runs in fp32 (TF32 off)."""
    import torch

    if not (0 <= row0 and rows >= 0 and row0 + rows <= m):
        raise ValueError(f"rows [{row0}, {row0 + rows}) outside 0..{m}")
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed) * 1000003 + 17)
    h0 = torch.randn((rank, n), generator=g, device=dev).abs_()
    h0 *= (torch.rand((rank, n), generator=g, device=dev) >= sparsity)
    sigma = noise_frac * lowrank_expected_mean(rank, sparsity)
    x = torch.empty((rows, n), dtype=torch.float32, device=dev)
    tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for b in range(row0 // block, (row0 + rows + block - 1) // block if rows else row0 // block):
            b0, b1 = b * block, min(m, (b + 1) * block)
            g.manual_seed((int(seed) * 0x9E3779B1 + 0x632BE5AB * (b + 1)) & 0x7FFFFFFFFFFFFFFF)
            w = torch.randn((b1 - b0, rank), generator=g, device=dev).abs_()
            w *= (torch.rand((b1 - b0, rank), generator=g, device=dev) >= sparsity)
            lo, hi = max(b0, row0), min(b1, row0 + rows)
            blk = w[lo - b0:hi - b0] @ h0
            noise = torch.randn((b1 - b0, n), generator=g, device=dev)[lo - b0:hi - b0]
            blk += noise.abs_() * sigma
            x[lo - row0:hi - row0] = blk
    finally:
        torch.backends.cuda.matmul.allow_tf32 = tf32
    return x


def config_shard(cfg_name: str, row0: int, rows: int, device="cuda"):
    """Device rows of a C4 / C5 workload (the seeded per-block generator above)."""
    cfg = CONFIGS[cfg_name]
    if cfg_name == "C4":
        return noisy_lowrank_shard(0, cfg.m, cfg.n, 40, 0.5, 0.1, row0, rows, device)
    if cfg_name == "C5":
        return noisy_lowrank_shard(0, cfg.m, cfg.n, 64, 0.7, 0.05, row0, rows, device)
    raise KeyError(cfg_name)


def injected_inputs(seed: int, m: int, n: int, k: int, l: int, gaussian_omega: bool = True):
    """Host draws injected into both the GPU path and the oracle: Omega (n x l) N(0,1) and unscaled
    init |N(0,1)| for W (m x k) and H (k x n) (BASELINE config wording)."""
    rng = np.random.default_rng(seed + 7919)
    omega = rng.standard_normal((n, l)) if gaussian_omega else rng.random((n, l))
    w0 = np.abs(rng.standard_normal((m, k)))
    h0 = np.abs(rng.standard_normal((k, n)))
    return omega, w0, h0
