"""Seeded synthetic depth scenes for the BASELINE.json workloads (C1-C5).

There is no public dataset for this path, so every input is
generated here.  Conventions follow the reference sensor model
(``synth.py:137-194``, ``camera.py:29``): each pixel's ray ``(tan_x, tan_y, 1)``
is intersected with the scene, the nearest positive hit wins, depth noise is
``Z += 1.425e-3 * Z**2 * N(0, 1)``, and invalid pixels hold ``Z = 0``.  Depth
is stored as float32 metres (or uint16 millimetres with ``np.round`` half-even
quantisation, ``synth.py:106``).  The parity tests never regenerate inputs
separately for the oracle: both sides read the same stored tensor.

Generator decisions that BASELINE.json leaves open (recorded in DESIGN.md):
plane tilt is capped at 70 degrees from the viewing ray (grazing planes would
leave cells almost empty), and per-config depth ranges are listed in
``CONFIGS``.  Scene parameters come from ``numpy.random.default_rng(seed)``;
per-pixel noise/dropout come from a ``torch.Generator`` on the target device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

NOISE_COEFFICIENT = 1.425e-3  # reference camera.py:29


@dataclass(frozen=True)
class SceneConfig:
    name: str
    frames: int
    width: int
    height: int
    f: float
    windows: tuple
    depth_range: tuple
    cells: int            # Voronoi cells (0: nearest of `planes` whole-image planes)
    planes: int = 0
    spheres: int = 0
    paraboloids: int = 0
    invalid: float = 0.05  # Bernoulli dropout fraction
    rect_holes: float = 0.0  # fraction covered by random rectangles (C3)
    u16: bool = False
    near_corner: bool = False  # C5: near-depth cells in the bottom-right quadrant

    @property
    def cx(self) -> float:
        return (self.width - 1) / 2.0

    @property
    def cy(self) -> float:
        return (self.height - 1) / 2.0


CONFIGS = {
    "C1": SceneConfig("C1", 1, 640, 480, 525.0, (5,), (0.5, 4.0), cells=0, planes=3),
    "C2": SceneConfig("C2", 64, 640, 480, 525.0, (3, 5, 7, 11, 15), (0.5, 4.0), cells=16),
    "C3": SceneConfig("C3", 256, 1280, 720, 920.0, (9,), (0.5, 6.0), cells=32, spheres=4,
                      invalid=0.02, rect_holes=0.08),
    "C4": SceneConfig("C4", 1024, 1920, 1080, 1380.0, (15,), (0.3, 8.0), cells=64, paraboloids=8,
                      invalid=0.08, u16=True),
    "C5": SceneConfig("C5", 128, 4096, 3072, 2900.0, (31,), (0.3, 20.0), cells=128, near_corner=True),
}


def _random_plane(rng, ray, z0, max_tilt_deg=70.0):
    """Unit normal facing the camera (n . ray < 0), tilt <= max_tilt from -ray."""
    view = -ray / np.linalg.norm(ray)
    cmin = math.cos(math.radians(max_tilt_deg))
    while True:
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        if n @ view < 0:
            n = -n
        if n @ view >= cmin:
            break
    p0 = ray * z0
    return n, -float(n @ p0)


def render_frame(cfg: SceneConfig, seed: int, device="cpu") -> torch.Tensor:
    """One frame as float32 metres (or uint16 mm for u16 configs), shape [H, W]."""
    rng = np.random.default_rng(seed)
    W, H, f = cfg.width, cfg.height, cfg.f
    dev = torch.device(device)
    tx = ((torch.arange(W, dtype=torch.float64, device=dev) - cfg.cx) / f)[None, :].expand(H, W)
    ty = ((torch.arange(H, dtype=torch.float64, device=dev) - cfg.cy) / f)[:, None].expand(H, W)
    zlo, zhi = cfg.depth_range
    inf = torch.tensor(float("inf"), dtype=torch.float64, device=dev)

    def plane_depth(n, d):
        den = n[0] * tx + n[1] * ty + n[2]
        z = torch.where(den != 0, -d / den, inf)
        return torch.where(torch.isfinite(z) & (z > 0), z, inf)

    if cfg.cells > 0:
        sx = rng.uniform(0, W, cfg.cells)
        sy = rng.uniform(0, H, cfg.cells)
        xx = torch.arange(W, dtype=torch.float32, device=dev)[None, :]
        yy = torch.arange(H, dtype=torch.float32, device=dev)[:, None]
        best = torch.full((H, W), float("inf"), device=dev)
        label = torch.zeros((H, W), dtype=torch.int64, device=dev)
        for c in range(cfg.cells):
            dist = (xx - float(sx[c])) ** 2 + (yy - float(sy[c])) ** 2
            closer = dist < best
            best = torch.where(closer, dist, best)
            label = torch.where(closer, torch.full_like(label, c), label)
        depth = torch.full((H, W), float("inf"), dtype=torch.float64, device=dev)
        for c in range(cfg.cells):
            ray = np.array([(sx[c] - cfg.cx) / f, (sy[c] - cfg.cy) / f, 1.0])
            if cfg.near_corner and sx[c] > W / 2 and sy[c] > H / 2:
                z0 = rng.uniform(zlo, zlo + 0.2)
            else:
                z0 = rng.uniform(zlo, zhi)
            n, d = _random_plane(rng, ray, z0)
            depth = torch.where(label == c, plane_depth(n, d), depth)
    else:
        depth = torch.full((H, W), float("inf"), dtype=torch.float64, device=dev)
        for _ in range(cfg.planes):
            ray = np.array([(rng.uniform(0, W) - cfg.cx) / f, (rng.uniform(0, H) - cfg.cy) / f, 1.0])
            n, d = _random_plane(rng, ray, rng.uniform(zlo, zhi))
            depth = torch.minimum(depth, plane_depth(n, d))

    # spheres: nearest positive ray hit t*(tx, ty, 1) with |p - c| = R
    for _ in range(cfg.spheres):
        c = np.array([rng.uniform(-0.5, 0.5), rng.uniform(-0.4, 0.4), rng.uniform(1.2, 4.0)])
        R = rng.uniform(0.2, 1.0)
        a = tx * tx + ty * ty + 1.0
        b = -2.0 * (tx * c[0] + ty * c[1] + c[2])
        cc = float(c @ c - R * R)
        disc = b * b - 4 * a * cc
        t = (-b - torch.sqrt(torch.clamp(disc, min=0))) / (2 * a)
        hit = (disc >= 0) & (t > 0)
        depth = torch.where(hit, torch.minimum(depth, t), depth)
    # paraboloid patches z = z0 + k((X-x0)^2 + (Y-y0)^2) inside a disc of radius R
    for _ in range(cfg.paraboloids):
        z0 = rng.uniform(zlo + 0.5, min(zhi, 4.0))
        x0 = rng.uniform(-0.3, 0.3) * z0
        y0 = rng.uniform(-0.2, 0.2) * z0
        k = rng.choice([-1.0, 1.0]) * rng.uniform(0.1, 1.0)
        R = rng.uniform(0.2, 0.6)
        # solve k t^2 (tx^2+ty^2) - t (1 + 2k(x0 tx + y0 ty)) + z0 + k(x0^2+y0^2) = 0
        A = k * (tx * tx + ty * ty)
        Bq = -(1.0 + 2.0 * k * (x0 * tx + y0 * ty))
        Cq = z0 + k * (x0 * x0 + y0 * y0)
        disc = Bq * Bq - 4 * A * Cq
        sq = torch.sqrt(torch.clamp(disc, min=0))
        t1 = (-Bq - sq) / (2 * A)
        t2 = (-Bq + sq) / (2 * A)
        tt = torch.where((t1 > 0) & ((t1 <= t2) | (t2 <= 0)), t1, t2)
        X, Y = tt * tx, tt * ty
        inside = ((X - x0) ** 2 + (Y - y0) ** 2 <= R * R) & (disc >= 0) & (tt > 0)
        depth = torch.where(inside, torch.minimum(depth, tt), depth)

    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed))
    valid = torch.isfinite(depth) & (depth >= zlo) & (depth <= zhi)
    z = torch.where(valid, depth, torch.zeros_like(depth))
    noise = torch.randn((H, W), generator=gen, device=dev, dtype=torch.float64)
    z = z + NOISE_COEFFICIENT * z * z * noise
    drop = torch.rand((H, W), generator=gen, device=dev) < cfg.invalid
    valid = valid & ~drop & (z > 0)
    if cfg.rect_holes > 0:
        hole = torch.zeros((H, W), dtype=torch.bool, device=dev)
        target = cfg.rect_holes * H * W
        covered = 0.0
        while covered < target:
            w_, h_ = int(rng.integers(4, 41)), int(rng.integers(4, 41))
            x_, y_ = int(rng.integers(0, W)), int(rng.integers(0, H))
            hole[y_:y_ + h_, x_:x_ + w_] = True
            covered = float(hole.sum())
        valid = valid & ~hole
    z = torch.where(valid, z, torch.zeros_like(z))
    if cfg.u16:
        mm = torch.round(z * 1000.0)
        mm = torch.where((mm >= 300) & (mm <= 8000), mm, torch.zeros_like(mm))
        return mm.to(torch.int32).to(torch.uint16)
    return z.to(torch.float32)


def render_batch(cfg: SceneConfig, frames: int | None = None, device="cpu", seed_base: int | None = None):
    """[B, H, W] batch; frame k uses seed 1000*config_index + k."""
    frames = cfg.frames if frames is None else frames
    if seed_base is None:
        seed_base = 1000 * int(cfg.name[1:])
    out = torch.empty((frames, cfg.height, cfg.width), dtype=torch.uint16 if cfg.u16 else torch.float32,
                      device=device)
    for k in range(frames):
        out[k] = render_frame(cfg, seed_base + k, device=device)
    return out


def small_config(name: str, width: int, height: int, f: float | None = None) -> SceneConfig:
    """A reduced-size variant of a BASELINE config for parity tests."""
    base = CONFIGS[name]
    scale = width / base.width
    return SceneConfig(
        name=base.name, frames=1, width=width, height=height,
        f=base.f * scale if f is None else f, windows=base.windows, depth_range=base.depth_range,
        cells=max(1, base.cells // 2) if base.cells else 0, planes=base.planes, spheres=base.spheres,
        paraboloids=base.paraboloids, invalid=base.invalid, rect_holes=base.rect_holes, u16=base.u16,
        near_corner=base.near_corner,
    )
