"""Seeded synthetic input generators (shared by the oracle tests and the product).

This module builds the linear systems the paper benchmarks on; it holds none of
the method's arithmetic (no strength, aggregation, smoothing, RAP or solve).  It
imports nothing from ``oracle/`` or ``paper_1811_05704_b200/``.  Every input is
synthetic and seeded; the recipes are:

* ``poisson3d``      -- Eq. (2) of the paper, -Lap u = 1 on [0,1]^3 with u = 0 on the
  boundary, 7-point finite differences on a uniform mesh,
  Dirichlet nodes eliminated, scaled by 1/h^2 with h = 1/(n+1) (§8c).  At
  n = 150 this is the paper's 3,375,000 x 3,375,000 system with 23,490,000
  nonzeros.
* ``var_coef_poisson3d`` -- log-normal coefficients k = exp(sigma g), g ~ N(0,1)
  i.i.d. per node (numpy default_rng(5704)), harmonic face means (§8c).
* ``convdiff3d``     -- -Lap u + b.grad u = 1, b = (1,1,1)/h, first-order upwind
  (cell Peclet 1/2): stencil x h^2 = diag 9, -2 at -x/-y/-z, -1 at +x/+y/+z (§8c).
* ``permute_symmetric`` -- A' = Pi A Pi^T, f' = Pi f with a default_rng(1811)
  permutation, to mimic an unstructured ordering (§8c).

Natural ordering: idx = x + nx*(y + ny*z).  CSR: int64 ptr, int32 col (strictly
increasing per row), float64 val.
"""
from __future__ import annotations

import numpy as np

SEED_PERM = 1811
SEED_COEF = 5704
SEED_VEC = 42


def _stencil_csr(nx, ny, nz, offdiag, diag):
    """Assemble a 7-point-pattern CSR from per-direction coefficient arrays.

    ``offdiag`` maps direction name -> array (N,) of the entry a_{i, nbr(i)} (only
    read where the neighbour exists); ``diag`` is the (N,) diagonal.  Entries of a
    row are emitted in ascending column order: -z, -y, -x, diag, +x, +y, +z.
    """
    N = nx * ny * nz
    idx = np.arange(N, dtype=np.int64)
    x = idx % nx
    y = (idx // nx) % ny
    z = idx // (nx * ny)
    plan = [("-z", -nx * ny, z > 0), ("-y", -nx, y > 0), ("-x", -1, x > 0), ("d", 0, None),
            ("+x", 1, x < nx - 1), ("+y", nx, y < ny - 1), ("+z", nx * ny, z < nz - 1)]
    cols = np.empty((N, 7), np.int32)
    vals = np.empty((N, 7), np.float64)
    mask = np.empty((N, 7), bool)
    for k, (name, off, ok) in enumerate(plan):
        cols[:, k] = (idx + off).astype(np.int32) if off else idx.astype(np.int32)
        if name == "d":
            vals[:, k] = diag
            mask[:, k] = True
        else:
            vals[:, k] = offdiag[name]
            mask[:, k] = ok
    del x, y, z
    counts = mask.sum(axis=1)
    ptr = np.zeros(N + 1, np.int64)
    np.cumsum(counts, out=ptr[1:])
    col = cols[mask]
    val = vals[mask]
    return ptr, col, val


def poisson3d(nx, ny=None, nz=None, h=None, scaled=True):
    """7-point Laplacian (Eq. (2)); returns (ptr, col, val, f).

    h defaults to 1/(nx+1); ``scaled=False`` gives the unit stencil (6, -1).
    nnz = 7N - 2(nx ny + ny nz + nx nz).
    """
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    N = nx * ny * nz
    inv_h2 = float((nx + 1) ** 2) if h is None else 1.0 / (h * h)
    if not scaled:
        inv_h2 = 1.0
    off = {d: np.full(N, -inv_h2) for d in ("-z", "-y", "-x", "+x", "+y", "+z")}
    ptr, col, val = _stencil_csr(nx, ny, nz, off, np.full(N, 6.0 * inv_h2))
    return ptr, col, val, np.ones(N)


def var_coef_poisson3d(n, sigma=1.0, seed=SEED_COEF):
    """-div(k grad u) = 1 with log-normal k (§8c); returns (ptr, col, val, f).

    k_i = exp(sigma g_i); the face between i and j (i < j) has coefficient
    2 k_i k_j / (k_i + k_j) (same expression for both rows, so A is bitwise
    symmetric); a Dirichlet face of node i uses k_i; a_ij = -k_f/h^2 and
    a_ii = sum of the six face coefficients / h^2.
    """
    nx = ny = nz = n
    N = n ** 3
    inv_h2 = float((n + 1) ** 2)
    g = np.random.default_rng(seed).standard_normal(N)
    k = np.exp(sigma * g)
    idx = np.arange(N, dtype=np.int64)
    x = idx % nx
    y = (idx // nx) % ny
    z = idx // (nx * ny)
    faces = {}
    for name, off, ok in (("x", 1, x < nx - 1), ("y", nx, y < ny - 1), ("z", nx * ny, z < nz - 1)):
        # face between i and i+off, stored at i (lo index)
        j = np.minimum(idx + off, N - 1)
        kf = (2.0 * k * k[j]) / (k + k[j])
        faces[name] = np.where(ok, kf, k)  # Dirichlet face uses k_i
    # coefficient of each of the 6 faces of node i
    fpx, fpy, fpz = faces["x"], faces["y"], faces["z"]
    fmx = np.where(x > 0, np.roll(faces["x"], 1), k)
    fmy = np.where(y > 0, np.roll(faces["y"], nx), k)
    fmz = np.where(z > 0, np.roll(faces["z"], nx * ny), k)
    diag = (((((fmz + fmy) + fmx) + fpx) + fpy) + fpz) * inv_h2
    off = {"-z": -fmz * inv_h2, "-y": -fmy * inv_h2, "-x": -fmx * inv_h2,
           "+x": -fpx * inv_h2, "+y": -fpy * inv_h2, "+z": -fpz * inv_h2}
    ptr, col, val = _stencil_csr(nx, ny, nz, off, diag)
    return ptr, col, val, np.ones(N)


def convdiff3d(n):
    """Upwind convection-diffusion, b = (1,1,1)/h (§8c); returns (ptr, col, val, f)."""
    N = n ** 3
    inv_h2 = float((n + 1) ** 2)
    off = {d: np.full(N, -2.0 * inv_h2) for d in ("-z", "-y", "-x")}
    off.update({d: np.full(N, -1.0 * inv_h2) for d in ("+x", "+y", "+z")})
    ptr, col, val = _stencil_csr(n, n, n, off, np.full(N, 9.0 * inv_h2))
    return ptr, col, val, np.ones(N)


def poisson2d(nx, ny=None):
    """Unit 5-point Laplacian (4, -1) on an nx x ny grid, idx = x + nx y."""
    ny = nx if ny is None else ny
    ptr, col, val, f = poisson3d(nx, ny, 1, scaled=False)
    # drop the z part: in a single plane there are no z neighbours; diagonal 6 -> 4
    d = np.repeat(np.arange(nx * ny), np.diff(ptr)) == col
    val = val.copy()
    val[d] = 4.0
    return ptr, col, val, f


def poisson1d(n):
    """Unit 1D Laplacian [-1, 2, -1]."""
    ptr, col, val, f = poisson3d(n, 1, 1, scaled=False)
    d = np.repeat(np.arange(n), np.diff(ptr)) == col
    val = val.copy()
    val[d] = 2.0
    return ptr, col, val, f


def permute_symmetric(ptr, col, val, f, seed=SEED_PERM):
    """A' = Pi A Pi^T, f' = Pi f (§8c); new row k is old row perm[k]."""
    N = len(ptr) - 1
    perm = np.random.default_rng(seed).permutation(N)
    inv = np.empty(N, np.int64)
    inv[perm] = np.arange(N)
    lens = np.diff(ptr)[perm]
    nptr = np.zeros(N + 1, np.int64)
    np.cumsum(lens, out=nptr[1:])
    rows = np.repeat(np.arange(N, dtype=np.int64), lens)
    src = np.repeat(ptr[:-1][perm], lens) + (np.arange(nptr[-1], dtype=np.int64) - nptr[:-1][rows])
    ncol = inv[col[src]]
    order = np.lexsort((ncol, rows))
    return nptr, ncol[order].astype(np.int32), val[src][order], f[perm]


def problem(name, n):
    """Named configurations of BASELINE.json."""
    if name == "poisson":
        return poisson3d(n)
    if name == "poisson_perm":
        return permute_symmetric(*poisson3d(n))
    if name == "varcoef":
        return var_coef_poisson3d(n)
    if name == "convdiff":
        return convdiff3d(n)
    raise ValueError(name)


def problem_rows(name, n):
    """Rows of problem(name, n) without building it (every generator is n^3)."""
    if name not in ("poisson", "poisson_perm", "varcoef", "convdiff"):
        raise ValueError(name)
    return n ** 3


def rhs_slice(name, n, r0, r1):
    """Rows r0..r1-1 of problem(name, n)'s right-hand side without building the
    matrix (f = 1 for every configuration; a permutation of ones
    is ones) -- what a rank > 0 of the scattered multi-GPU setup needs."""
    problem_rows(name, n)
    return np.ones(r1 - r0)


def weak_poisson(nranks, n=256):
    """Weak-scaling configuration (BASELINE.json configs[4], §8c): Poisson
    on the global box n x n x (n nranks), h = 1/(n+1) in every direction, so
    each rank's z-slab is one n^3 block.  Returns (ptr, col, val, f)."""
    return poisson3d(n, n, n * nranks)  # 1/h^2 = (n+1)^2 exactly (the default of poisson3d)


def random_vector(n, seed=SEED_VEC):
    return np.random.default_rng(seed).standard_normal(n)
