"""Deterministic synthetic volumes for the BASELINE configs (BASELINE.json configs 1-5).

Everything is analytic (no interpolation), so the same arrays are produced on
any host from the seed alone; the reference CPU oracle and the CUDA engine are
fed identical bytes.  Images are min-max rescaled to [0, 1] like the
reference CLI does (io.hpp:166-178, lddmm_cli.cpp:220-223).
"""
from __future__ import annotations

import numpy as np


def rescale_unit(f):
    lo, hi = float(f.min()), float(f.max())
    return (f - lo) / (hi - lo) if hi > lo else np.zeros_like(f)


def _coords(dims, spacing=(1.0, 1.0, 1.0)):
    return [np.arange(n, dtype=np.float64).reshape([-1 if a == b else 1 for b in range(3)]) * spacing[a]
            for a, n in enumerate(dims)]


def _periodic(d, L):
    return d - L * np.round(d / L)


def tanh_ellipsoid(dims, center, semi, edge=1.5, disp=None, spacing=(1.0, 1.0, 1.0)):
    """0.5 (1 - tanh((r - 1) * s / edge)), r the ellipsoidal radius, periodic distances.
    disp (3, *dims): evaluate at x - disp (analytic pull-back)."""
    X = _coords(dims, spacing)
    L = [n * h for n, h in zip(dims, spacing)]
    r2 = 0.0
    for a in range(3):
        xa = X[a] - (disp[a] if disp is not None else 0.0)
        r2 = r2 + (_periodic(xa - center[a], L[a]) / semi[a]) ** 2
    r = np.sqrt(r2)
    scale = float(np.min(semi))
    return 0.5 * (1.0 - np.tanh((r - 1.0) * scale / edge))


def sphere_ellipsoid_pair(n=64):
    """Config 1: tanh-edged sphere (r=16, edge 1.5, centre n/2) -> ellipsoid (20, 16, 12)."""
    dims = (n, n, n)
    c = (n / 2, n / 2, n / 2)
    s = rescale_unit(tanh_ellipsoid(dims, c, (16.0, 16.0, 16.0)))
    t = rescale_unit(tanh_ellipsoid(dims, c, (20.0, 16.0, 12.0)))
    return s, t


def _cosine_field(dims, rng, nmodes, kmax, disp=None):
    X = _coords(dims)
    out = np.zeros(dims)
    for _ in range(nmodes):
        k = rng.integers(-kmax, kmax + 1, size=3)
        if not k.any():
            k[0] = 1
        ph = rng.uniform(0, 2 * np.pi)
        amp = rng.normal()
        arg = ph
        for a in range(3):
            xa = X[a] - (disp[a] if disp is not None else 0.0)
            arg = arg + 2 * np.pi * k[a] * xa / dims[a]
        out = out + amp * np.cos(arg)
    return out


def smooth_displacement(dims, seed, amplitude=4.0, kmax=3, nmodes=6):
    """Periodic smooth displacement (3, *dims) with max |u| = amplitude voxels."""
    rng = np.random.default_rng(seed)
    u = np.stack([_cosine_field(dims, rng, nmodes, kmax) for _ in range(3)])
    m = np.max(np.abs(u))
    return u * (amplitude / m) if m > 0 else u


def brain_like(dims, seed=2006, disp=None):
    """Brain-like phantom: textured tanh ellipsoid with two dark 'ventricles'."""
    rng = np.random.default_rng(seed)
    c = tuple(n / 2 for n in dims)
    semi = (0.39 * dims[0], 0.405 * dims[1], 0.36 * dims[2])
    head = tanh_ellipsoid(dims, c, semi, 1.5, disp)
    tex = _cosine_field(dims, rng, 12, 6, disp)
    tex = (tex - tex.min()) / max(tex.max() - tex.min(), 1e-12)
    img = head * (0.6 + 0.4 * tex)
    for sgn in (-1, 1):
        vc = (c[0] + sgn * 0.06 * dims[0], c[1] - 0.02 * dims[1], c[2])
        img = img - 0.35 * tanh_ellipsoid(dims, vc, (0.05 * dims[0], 0.12 * dims[1], 0.06 * dims[2]), 1.5, disp)
    return img


def brain_pair(dims=(180, 210, 180), seed=2006, amplitude=4.0):
    """Config 2/3/4 pair: source = brain_like, target = source o (x - u_true) (analytic)."""
    s = brain_like(dims, seed)
    u = smooth_displacement(dims, seed + 1, amplitude)
    t = brain_like(dims, seed, disp=u)
    return rescale_unit(s), rescale_unit(t)


def subject(dims, s, seed_template=2006, amplitude=4.0):
    """Config 5 subject s: template o (x - u_s), u_s seeded 100 + s."""
    u = smooth_displacement(dims, 100 + s, amplitude)
    return rescale_unit(brain_like(dims, seed_template, disp=u))
