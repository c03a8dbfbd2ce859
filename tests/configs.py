"""Test-side generators for BASELINE.json configs 2–4 (test infrastructure).

The reference has no generator for these (problems.hpp:199-232 only knows
Gaussian, sparse, file and stacked sources), so they are
restated here from the config text with numpy, seeded.  Inputs are generated in
the test process and fed to both the oracle and the GPU, so no cross-machine
bit reproducibility is needed.
"""
import numpy as np


def orthonormal(rng, rows, cols):
    q, r = np.linalg.qr(rng.standard_normal((rows, cols)))
    return q * np.sign(np.diag(r))  # unique Haar-distributed factor


def svd_built(rng, rows, cols, sigma_max=1.0, sigma_min=1e-2, rank=None):
    """U·diag(σ)·Vᵀ, σ log-spaced sigma_max..sigma_min; the smallest
    r − rank singular values zeroed (config 2, config 3 rank-deficient)."""
    r = min(rows, cols)
    U = orthonormal(rng, rows, r)
    V = orthonormal(rng, cols, r)
    sig = np.logspace(np.log10(sigma_max), np.log10(sigma_min), r)
    if rank is not None:
        sig[rank:] = 0.0
    return (U * sig) @ V.T


def config2(seed=0, m=2000, p=500, q=400, n=2000):
    """Config 2: A m×p, B q×n, both U·diag(σ)·Vᵀ with σ log-spaced 1..1e-2; X* N(0,1)."""
    rng = np.random.default_rng(seed)
    A = svd_built(rng, m, p)
    B = svd_built(rng, q, n)
    Xs = rng.standard_normal((p, q))
    return A, B, Xs, (A @ Xs) @ B


def config3_rank_deficient(seed=0, m=512, p=128, q=128, n=512, rank=96):
    """Config 3 analogue: Gaussian-spectrum A with rank(A) < p, B full row rank,
    X0 N(0,1); the iteration converges to X⁰_* = A⁺CB⁺ + X0 − A⁺AX0BB⁺
    (analysis.hpp:95-104)."""
    rng = np.random.default_rng(seed)
    U = orthonormal(rng, m, p)
    V = orthonormal(rng, p, p)
    s = np.sort(np.abs(rng.standard_normal(p)) * np.sqrt(m))[::-1]
    s[rank:] = 0.0
    A = (U * s) @ V.T
    B = rng.standard_normal((q, n))
    Xs = rng.standard_normal((p, q))
    X0 = rng.standard_normal((p, q))
    C = (A @ Xs) @ B
    Ap, Bp = np.linalg.pinv(A, rcond=1e-10), np.linalg.pinv(B)
    target = Ap @ C @ Bp + X0 - Ap @ A @ X0 @ B @ Bp
    return A, B, C, X0, target


def gaussian_blur_toeplitz(nn, sigma=3.0, half_band=7):
    """Symmetric banded Toeplitz from a normalised 1-D Gaussian, zero boundary
    (the 1-D analogue of imaging.hpp:93-136)."""
    k = np.arange(-half_band, half_band + 1)
    w = np.exp(-k ** 2 / (2 * sigma ** 2))
    w /= w.sum()
    T = np.zeros((nn, nn))
    for d, v in zip(k, w):
        T += np.diag(np.full(nn - abs(d), v), d)
    return T


def smooth_field(rng, nn, sigma=8.0):
    """Uniform noise filtered by a separable Gaussian (σ px), min–max to [0, 1]."""
    F = gaussian_blur_toeplitz(nn, sigma, int(3 * sigma))
    X = F @ rng.random((nn, nn)) @ F.T
    return (X - X.min()) / (X.max() - X.min())


def config4_channel(seed=0, nn=1024, half_band=7, noise=1e-3):
    """Config 4, one colour channel: A = B = blur Toeplitz, C = A·X*·B + N(0, noise²)."""
    rng = np.random.default_rng(seed)
    A = gaussian_blur_toeplitz(nn, 3.0, half_band)
    Xs = smooth_field(rng, nn)
    C = A @ Xs @ A + noise * rng.standard_normal((nn, nn))
    return A, A.copy(), Xs, C
