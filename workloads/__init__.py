"""Seeded synthetic inputs shaped like the paper's workloads (shared by the
oracle tests, the GPU parity tests and bench.py).

This module holds NONE of the filter's arithmetic: it only draws images and the
per-pixel range-kernel centre theta(i) / width sigma(i) maps.  The paper's own
images are not available, so each config in
BASELINE.json is a synthetic stand-in (recipes and readings in DESIGN.md,
section "Inputs").  All images are integer valued in [0, 255] and stored as
float32, like the paper's 8-bit inputs.

Seeds: image ``1000*cfg + index``; the theta/sigma noise uses ``+500``.
"""
from __future__ import annotations

import dataclasses

import numpy as np

__all__ = [
    "Workload",
    "rectangles",
    "texture",
    "voronoi",
    "config",
    "config5",
    "CONFIG5_RHOS",
    "CONFIG5_NS",
    "random_case",
]

CONFIG5_RHOS = (2, 5, 10, 20, 40)
CONFIG5_NS = (4, 6, 8, 10)


@dataclasses.dataclass
class Workload:
    name: str
    img: np.ndarray    # float32, B x H x W
    theta: np.ndarray  # float32, B x H x W
    sigma: np.ndarray  # float32, B x H x W
    rho: int
    N: int

    @property
    def shape(self):
        return self.img.shape

    @property
    def pixels(self) -> int:
        return int(self.img.size)


def _finish(x: np.ndarray) -> np.ndarray:
    return np.clip(np.rint(x), 0, 255).astype(np.float32)


def rectangles(H: int, W: int, seed: int, n_rect: int = 8, noise_sd: float = 10.0) -> np.ndarray:
    """Config-1 generator: background U[0,255], then ``n_rect`` axis-aligned
    rectangles (side U[W/8, W/2], uniform position, level U[0,255]) painted in
    order, plus N(0, noise_sd^2), rint, clip."""
    rng = np.random.default_rng(seed)
    f = np.full((H, W), rng.uniform(0, 255), np.float64)
    for _ in range(n_rect):
        h = int(rng.uniform(H / 8, H / 2))
        w = int(rng.uniform(W / 8, W / 2))
        y = int(rng.integers(0, max(1, H - h + 1)))
        x = int(rng.integers(0, max(1, W - w + 1)))
        f[y:y + h, x:x + w] = rng.uniform(0, 255)
    f += rng.normal(0.0, noise_sd, (H, W))
    return _finish(f)


def texture(H: int, W: int, seed: int) -> np.ndarray:
    """Config-2 generator: linear gradient along a random direction (span
    80-160 levels, offset 0-40) + amplitude-25 sinusoid with period U[6,12] px at a
    random angle + 6 piecewise-constant rectangles with offsets U[-80,80]."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    ang = rng.uniform(0, 2 * np.pi)
    proj = xx * np.cos(ang) + yy * np.sin(ang)
    proj = (proj - proj.min()) / max(1e-9, proj.max() - proj.min())
    f = rng.uniform(0, 40) + rng.uniform(80, 160) * proj
    period = rng.uniform(6, 12)
    ang2 = rng.uniform(0, np.pi)
    phase = rng.uniform(0, 2 * np.pi)
    f += 25.0 * np.sin(2 * np.pi * (xx * np.cos(ang2) + yy * np.sin(ang2)) / period + phase)
    for _ in range(6):
        h = int(rng.uniform(H / 8, H / 2))
        w = int(rng.uniform(W / 8, W / 2))
        y = int(rng.integers(0, max(1, H - h + 1)))
        x = int(rng.integers(0, max(1, W - w + 1)))
        f[y:y + h, x:x + w] += rng.uniform(-80, 80)
    return _finish(f)


def voronoi(H: int, W: int, seed: int, n_seeds: int = 64, noise_sd: float = 15.0) -> np.ndarray:
    """Config-3/4 generator: piecewise-constant Voronoi cells (seeds uniform in
    the image, nearest seed in Euclidean distance, levels U[0,255]) plus
    N(0, noise_sd^2), rint, clip."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    pts = np.stack([rng.uniform(0, H, n_seeds), rng.uniform(0, W, n_seeds)], axis=1)
    levels = rng.uniform(0, 255, n_seeds)
    yy, xx = np.mgrid[0:H, 0:W]
    q = np.stack([yy.ravel() + 0.5, xx.ravel() + 0.5], axis=1)
    _, nearest = cKDTree(pts).query(q, k=1)
    f = levels[nearest].reshape(H, W)
    f = f + rng.normal(0.0, noise_sd, (H, W))
    return _finish(f)


def _stack(x):
    return np.ascontiguousarray(x[None] if x.ndim == 2 else x, dtype=np.float32)


def config(cfg: int, scale: float = 1.0, frame: int = 0) -> Workload:
    """Configs 1-4 of BASELINE.json (1-based as printed there).

    ``scale`` < 1 shrinks the image (for quick tests) while keeping rho and N.
    ``frame`` > 0 draws another frame of the same recipe (other seeds; frame 0
    is the BASELINE frame) -- the frames a multi-GPU run shards over ranks."""
    if frame:
        w = _config_seeded(cfg, scale, 1000 * cfg + 10007 * frame)
        return Workload(f"{w.name}_frame{frame}", w.img, w.theta, w.sigma, w.rho, w.N)
    return _config_seeded(cfg, scale, 1000 * cfg)


def _config_seeded(cfg: int, scale: float, seed: int) -> Workload:
    from scipy import ndimage

    if cfg == 1:
        H = W = max(16, int(256 * scale))
        f = rectangles(H, W, seed)
        rng = np.random.default_rng(seed + 500)
        sigma = rng.uniform(10, 40, f.shape)
        theta = f + rng.uniform(-10, 10, f.shape)
        return Workload("cfg1_256x256_rects_rho3_N5", _stack(f), _stack(theta), _stack(sigma), 3, 5)
    if cfg == 2:
        H, W = max(16, int(450 * scale)), max(16, int(600 * scale))
        f = texture(H, W, seed)
        rng11 = ndimage.maximum_filter(f, size=11, mode="reflect") - ndimage.minimum_filter(
            f, size=11, mode="reflect")
        sigma = 5.0 + 2.5 * rng11
        theta = f.copy()
        return Workload("cfg2_600x450_texture_rho5_N6", _stack(f), _stack(theta), _stack(sigma), 5, 6)
    if cfg == 3:
        H, W = max(32, int(1080 * scale)), max(32, int(1920 * scale))
        f = voronoi(H, W, seed, n_seeds=64, noise_sd=15.0)
        L = -ndimage.gaussian_laplace(f.astype(np.float64), 2.0, mode="reflect", truncate=4.0)
        tl = np.tanh(L / 10.0)
        theta = f + 20.0 * tl
        sigma = 10.0 + 20.0 * np.abs(tl)
        return Workload("cfg3_1920x1080_voronoi64_rho10_N8", _stack(f), _stack(theta), _stack(sigma), 10, 8)
    if cfg == 4:
        H, W = max(64, int(2160 * scale)), max(64, int(3840 * scale))
        f = voronoi(H, W, seed, n_seeds=256, noise_sd=20.0)
        rng = np.random.default_rng(seed + 500)
        sigma = rng.uniform(5, 60, f.shape)
        theta = f + rng.uniform(-15, 15, f.shape)
        return Workload("cfg4_3840x2160_voronoi256_rho20_N8", _stack(f), _stack(theta), _stack(sigma), 20, 8)
    raise ValueError(f"unknown config {cfg}")


def config5(rho: int, N: int, batch: int = 32, size: int = 1024, generator: str = "texture",
            first: int = 0) -> Workload:
    """Config 5: ``batch`` grey images of size x size (the config-2 'texture'
    generator, 0-based reading of BASELINE.json; 'rectangles' is the secondary
    reading), sigma ~ U[5,60], theta = f."""
    gen = texture if generator == "texture" else rectangles
    imgs, sig = [], []
    for b in range(first, first + batch):
        imgs.append(gen(size, size, 5000 + b))
        rng = np.random.default_rng(5000 + b + 500)
        sig.append(rng.uniform(5, 60, (size, size)))
    f = np.stack(imgs).astype(np.float32)
    return Workload(f"cfg5_{batch}x{size}^2_{generator}_rho{rho}_N{N}", f, f.copy(),
                    np.stack(sig).astype(np.float32), rho, N)


def random_case(B: int, H: int, W: int, seed: int, kind: str = "rect", rho: int = 2, N: int = 4,
                sigma_range=(5.0, 60.0), theta_jitter: float = 15.0) -> Workload:
    """Small seeded cases for parity tests (odd shapes, tails, special values)."""
    rng = np.random.default_rng(seed)
    imgs = []
    for b in range(B):
        if kind == "rect":
            imgs.append(rectangles(H, W, seed * 7919 + b))
        elif kind == "texture":
            imgs.append(texture(H, W, seed * 7919 + b))
        elif kind == "voronoi":
            imgs.append(voronoi(H, W, seed * 7919 + b, n_seeds=max(4, H * W // 400), noise_sd=15.0))
        elif kind == "uniform":
            imgs.append(np.rint(rng.uniform(0, 255, (H, W))).astype(np.float32))
        elif kind == "float":  # non-integer intensities on an arbitrary scale
            imgs.append(rng.uniform(-3.0, 5.0, (H, W)).astype(np.float32))
        elif kind == "flat":  # large constant areas -> identity pixels
            a = np.full((H, W), 100.0, np.float32)
            a[H // 2:, W // 2:] = 180.0
            imgs.append(a)
        else:
            raise ValueError(kind)
    f = np.stack(imgs).astype(np.float32)
    span = float(f.max() - f.min()) or 1.0
    scale = span / 255.0
    sigma = rng.uniform(*sigma_range, f.shape) * scale
    theta = f + rng.uniform(-theta_jitter, theta_jitter, f.shape) * scale
    return Workload(f"rand_{kind}_{B}x{H}x{W}_rho{rho}_N{N}", f, theta.astype(np.float32),
                    sigma.astype(np.float32), rho, N)
