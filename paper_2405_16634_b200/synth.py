"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds ONLY geometry sampling (points on analytic surfaces, their analytic normals,
noise, outliers); it contains none of the method's arithmetic (no kernels, no trees, no
operators).  Recipes follow SURVEY.md §8(d) d.2 and are restated in DESIGN.md §"Inputs":

  C1  unit sphere, N = 2,000, area-uniform, random-sign GT normals (for operator inputs)
  C2  torus R=1 r=0.3 (and superquadric |x|^4+|y|^4+|z|^4 = 1), N = 50,000, 0.5 % noise
  C3  bumpy sphere r(u) = 1 + 0.15 sin(5θ) sin(4φ), N = 500,000, density ∝ 0.1 + 0.9((1+ẑ)/2)^2
  C4  thin plate 1.8×1.8×0.02 + thin torus R=0.6 r=0.01, N = 200,000, 1 % uniform outliers
  C5  8 shapes on a 2×2×2 grid, N = 4,000,000, 0.25 % noise
  T5  level-7 icosphere (163,842 vertices) of PAPER.md:L945-L961 Table 5

Seeds: shape RNG = 1000 + config index, noise = +1, sign flips = +2.
All sampling is done in float64 and returned as float32 points.
"""
from __future__ import annotations

import numpy as np


def _unit(v):
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _uniform_dirs(rng, n):
    return _unit(rng.standard_normal((n, 3)))


def sphere(n, seed=1001, R=1.0, center=(0.0, 0.0, 0.0)):
    """Area-uniform random points on a sphere; outward normals."""
    rng = np.random.default_rng(seed)
    u = _uniform_dirs(rng, n)
    return (u * R + np.asarray(center)).astype(np.float32), u


def fibonacci_sphere(n, R=1.0):
    """Deterministic Fibonacci lattice (near-uniform, symmetric spacing)."""
    i = np.arange(n) + 0.5
    z = 1 - 2 * i / n
    phi = np.pi * (1 + 5 ** 0.5) * i
    rho = np.sqrt(1 - z * z)
    u = np.stack([rho * np.cos(phi), rho * np.sin(phi), z], axis=1)
    return (u * R).astype(np.float32), u


def icosphere(level=7, R=1.0):
    """Icosphere: icosahedron, `level` midpoint subdivisions, vertices re-projected onto the sphere
    after every subdivision (10·4^level + 2 vertices; level 7 → 163,842 = Table 5's count)."""
    t = (1 + 5 ** 0.5) / 2
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t],
                  [0, 1, -t], [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], dtype=np.float64)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4],
                  [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8],
                  [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    v = _unit(v)
    for _ in range(level):
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        e.sort(axis=1)
        ue, inv = np.unique(e, axis=0, return_inverse=True)
        inv = inv.reshape(-1)
        mid = _unit((v[ue[:, 0]] + v[ue[:, 1]]) / 2)
        m = inv.reshape(3, -1).T + len(v)       # midpoint ids of edges (01, 12, 20) per face
        v = np.concatenate([v, mid])
        a, b, c = f[:, 0], f[:, 1], f[:, 2]
        ab, bc, ca = m[:, 0], m[:, 1], m[:, 2]
        f = np.concatenate([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                            np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)])
    return (v * R).astype(np.float32), v, f


def torus(n, seed=1002, R=1.0, r=0.3, center=(0.0, 0.0, 0.0)):
    """Area-uniform torus (accept (φ, ψ) with probability (R + r cos ψ)/(R + r))."""
    rng = np.random.default_rng(seed)
    out_p, out_n, have = [], [], 0
    while have < n:
        m = 2 * (n - have) + 64
        phi = rng.uniform(0, 2 * np.pi, m)
        psi = rng.uniform(0, 2 * np.pi, m)
        keep = rng.uniform(0, 1, m) < (R + r * np.cos(psi)) / (R + r)
        phi, psi = phi[keep], psi[keep]
        nrm = np.stack([np.cos(psi) * np.cos(phi), np.cos(psi) * np.sin(phi), np.sin(psi)], 1)
        p = np.stack([(R + r * np.cos(psi)) * np.cos(phi), (R + r * np.cos(psi)) * np.sin(phi),
                      r * np.sin(psi)], 1)
        out_p.append(p)
        out_n.append(nrm)
        have += len(p)
    p = np.concatenate(out_p)[:n] + np.asarray(center)
    return p.astype(np.float32), np.concatenate(out_n)[:n]


def _star_shaped(n, rng, radius_fn, normal_fn, density_fn=None):
    """x = r(u) u with u uniform on S², accepted with probability ∝ r(u)²/(n̂·u) (area element),
    optionally times a density factor in [0, 1]."""
    out_p, out_n, have = [], [], 0
    bound = None
    while have < n:
        m = 4 * (n - have) + 1024
        u = _uniform_dirs(rng, m)
        r = radius_fn(u)
        p = u * r[:, None]
        nrm = normal_fn(p, u)
        wgt = r ** 2 / np.sum(nrm * u, axis=1)
        if density_fn is not None:
            wgt = wgt * density_fn(p)
        if bound is None:
            bound = 1.05 * wgt.max()
        keep = rng.uniform(0, bound, m) < wgt
        out_p.append(p[keep])
        out_n.append(nrm[keep])
        have += int(keep.sum())
    return np.concatenate(out_p)[:n], np.concatenate(out_n)[:n]


def superquadric(n, seed=1002, p=4.0, scale=1.0, center=(0.0, 0.0, 0.0)):
    """|x|^p + |y|^p + |z|^p = 1 (p = 4)."""
    rng = np.random.default_rng(seed)
    rad = lambda u: np.sum(np.abs(u) ** p, axis=1) ** (-1.0 / p)
    nor = lambda x, u: _unit(np.sign(x) * np.abs(x) ** (p - 1))
    pts, nrm = _star_shaped(n, rng, rad, nor)
    return (pts * scale + np.asarray(center)).astype(np.float32), nrm


def _bumpy_radius(u):
    th = np.arccos(np.clip(u[:, 2], -1, 1))
    ph = np.arctan2(u[:, 1], u[:, 0])
    return 1 + 0.15 * np.sin(5 * th) * np.sin(4 * ph)


def _bumpy_normal(x, u):
    """∇(|x| − r(θ, φ)) = û − (∂r/∂θ)/ρ θ̂ − (∂r/∂φ)/(ρ sin θ) φ̂."""
    rho = np.linalg.norm(x, axis=1)
    th = np.arccos(np.clip(u[:, 2], -1, 1))
    ph = np.arctan2(u[:, 1], u[:, 0])
    dr_dth = 0.15 * 5 * np.cos(5 * th) * np.sin(4 * ph)
    dr_dph = 0.15 * 4 * np.sin(5 * th) * np.cos(4 * ph)
    th_hat = np.stack([np.cos(th) * np.cos(ph), np.cos(th) * np.sin(ph), -np.sin(th)], 1)
    ph_hat = np.stack([-np.sin(ph), np.cos(ph), np.zeros_like(ph)], 1)
    st = np.maximum(np.sin(th), 1e-12)
    g = u - (dr_dth / rho)[:, None] * th_hat - (dr_dph / (rho * st))[:, None] * ph_hat
    return _unit(g)


def bumpy_sphere(n, seed=1003, nonuniform=True, scale=1.0, center=(0.0, 0.0, 0.0)):
    """C3: r(u) = 1 + 0.15 sin(5θ) sin(4φ); density ∝ 0.1 + 0.9((1+ẑ)/2)^2 (10:1 ratio)."""
    rng = np.random.default_rng(seed)
    dens = None
    if nonuniform:
        zmax = 1.15
        dens = lambda x: 0.1 + 0.9 * ((1 + np.clip(x[:, 2] / zmax, -1, 1)) / 2) ** 2
    pts, nrm = _star_shaped(n, rng, _bumpy_radius, _bumpy_normal, dens)
    return (pts * scale + np.asarray(center)).astype(np.float32), nrm


def box_surface(n, seed, ext=(1.8, 1.8, 0.02), center=(0.0, 0.0, 0.0)):
    """Area-uniform samples on the surface of an axis-aligned box; normals ±e_k."""
    rng = np.random.default_rng(seed)
    ex = np.asarray(ext, np.float64)
    areas = np.array([ex[1] * ex[2], ex[1] * ex[2], ex[0] * ex[2], ex[0] * ex[2], ex[0] * ex[1], ex[0] * ex[1]])
    face = rng.choice(6, size=n, p=areas / areas.sum())
    p = (rng.uniform(-0.5, 0.5, (n, 3))) * ex
    nrm = np.zeros((n, 3))
    ax = face // 2
    sg = np.where(face % 2 == 0, -1.0, 1.0)
    p[np.arange(n), ax] = sg * ex[ax] / 2
    nrm[np.arange(n), ax] = sg
    return (p + np.asarray(center)).astype(np.float32), nrm


def add_noise(pts, sigma_frac, seed):
    """Gaussian noise N(0, (σ·bbox-diagonal)^2) per axis."""
    if sigma_frac <= 0:
        return pts
    rng = np.random.default_rng(seed)
    p = pts.astype(np.float64)
    diag = np.linalg.norm(p.max(0) - p.min(0))
    return (p + rng.normal(0, sigma_frac * diag, p.shape)).astype(np.float32)


def random_signs(normals, seed):
    rng = np.random.default_rng(seed)
    s = np.where(rng.uniform(size=len(normals)) < 0.5, -1.0, 1.0)
    return normals * s[:, None]


def config(name: str, n: int | None = None):
    """Named BASELINE.json configs.  Returns dict(points f32 n×3, normals f64 n×3 (analytic, outward),
    inlier bool mask, name)."""
    name = name.upper()
    if name == "C1":
        n = n or 2000
        p, nr = sphere(n, seed=1001)
    elif name in ("C2", "C2T"):
        n = n or 50000
        p, nr = torus(n, seed=1002)
        p = add_noise(p, 0.005, 1003)
    elif name == "C2S":
        n = n or 50000
        p, nr = superquadric(n, seed=1002)
        p = add_noise(p, 0.005, 1003)
    elif name == "C3":
        n = n or 500000
        p, nr = bumpy_sphere(n, seed=1003)
    elif name == "C4":
        n = n or 200000
        n_out = n // 100
        n_in = n - n_out
        n_plate = n_in * 2 // 3
        pa, na = box_surface(n_plate, 1004, ext=(1.8, 1.8, 0.02), center=(0.0, 0.0, -0.3))
        pb_, nb = torus(n_in - n_plate, seed=1014, R=0.6, r=0.01, center=(0.0, 0.0, 0.3))
        p = np.concatenate([pa, pb_]).astype(np.float64)
        nr = np.concatenate([na, nb])
        rng = np.random.default_rng(1006)
        lo, hi = p.min(0), p.max(0)
        c, h = (lo + hi) / 2, (hi - lo) / 2 * 1.05
        po = rng.uniform(c - h, c + h, (n_out, 3))
        p = np.concatenate([p, po]).astype(np.float32)
        nr = np.concatenate([nr, np.zeros((n_out, 3))])
        mask = np.concatenate([np.ones(n_in, bool), np.zeros(n_out, bool)])
        return dict(points=p, normals=nr, inlier=mask, name="C4")
    elif name == "C5":
        n = n or 4000000
        k = n // 8
        parts = []
        gens = [lambda m, s, c: sphere(m, s, 0.4, c), lambda m, s, c: sphere(m, s, 0.4, c),
                lambda m, s, c: torus(m, s, 0.4 / 1.3, 0.12 / 1.3, c),
                lambda m, s, c: torus(m, s, 0.4 / 1.3, 0.12 / 1.3, c),
                lambda m, s, c: superquadric(m, s, 4.0, 0.4, c), lambda m, s, c: superquadric(m, s, 4.0, 0.4, c),
                lambda m, s, c: bumpy_sphere(m, s, False, 0.4 / 1.15, c),
                lambda m, s, c: bumpy_sphere(m, s, False, 0.4 / 1.15, c)]
        for g, gen in enumerate(gens):
            ctr = (((g >> 2) & 1) - 0.5, ((g >> 1) & 1) - 0.5, (g & 1) - 0.5)
            m = k if g < 7 else n - 7 * k
            parts.append(gen(m, 1005 + 10 * g, ctr))
        p = np.concatenate([q[0] for q in parts])
        nr = np.concatenate([q[1] for q in parts])
        p = add_noise(p, 0.0025, 1006)
    elif name == "T5":
        p, nr, _ = icosphere(7)
    else:
        raise ValueError(f"unknown config {name}")
    return dict(points=p, normals=nr, inlier=np.ones(len(p), bool), name=name)
