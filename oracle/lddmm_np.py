"""CPU oracle: a plain numpy restatement of the reference's band-limited SL
LDDMM path (fp64 throughout).

TEST INFRASTRUCTURE ONLY.  This module is the checker the CUDA engine is
compared against; only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import it.  The product package never does.

Every function cites the reference file:line it restates
(/root/reference/proj/include/lddmm/...).  FFTW (an unpinned third-party
dependency of the reference, CMakeLists.txt:15) is replaced by numpy's
pocketfft; the FFT sign/normalisation contract is fft.hpp:1-9 (forward
unscaled, backward / N).  The restatement is pinned against the reference
itself (oracle/_ref, built from /root/reference by oracle/Makefile) through
the committed fixtures in tests/golden (see tests/test_oracle.py).

Layouts: grid scalar [*dims]; grid vector [d, *dims]; band scalar complex
[*band]; band vector complex [d, *band]; velocity (stationary) = one band
vector, (nonstationary) = list of nt+1 band vectors.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# grids and bands (core.hpp:42-122, spectral.hpp:22-83)


@dataclass(frozen=True)
class Grid:
    dims: tuple
    spacing: tuple

    @property
    def d(self):
        return len(self.dims)

    @property
    def size(self):
        return int(np.prod(self.dims))

    def cell_volume(self):  # core.hpp:89-93
        return float(np.prod(self.spacing))

    def min_spacing(self):  # core.hpp:95-99
        return float(min(self.spacing))


@dataclass(frozen=True)
class Band:
    grid: Grid
    bounds: tuple

    @property
    def d(self):
        return self.grid.d

    def signed_freq(self, a):  # spectral.hpp:70
        K = self.bounds[a]
        f = np.arange(K)
        return np.where(f < K // 2, f, f - K)

    def omega(self, a):  # spectral.hpp:77-79
        return 2.0 * np.pi * self.signed_freq(a) / (self.grid.dims[a] * self.grid.spacing[a])

    def parent_index(self, a):  # spectral.hpp:72-75
        k = self.signed_freq(a)
        return np.where(k >= 0, k, k + self.grid.dims[a])

    def nyquist_mask(self):  # spectral.hpp:71 (band Nyquist planes)
        m = np.zeros(self.bounds, dtype=bool)
        for a in range(self.d):
            sl = [slice(None)] * self.d
            sl[a] = self.bounds[a] // 2
            m[tuple(sl)] = True
        return m

    def omega_grids(self):
        return np.meshgrid(*[self.omega(a) for a in range(self.d)], indexing="ij")


def identity_map(g: Grid):  # core.hpp:261-269
    axes = [np.arange(n) * h for n, h in zip(g.dims, g.spacing)]
    return np.stack(np.meshgrid(*axes, indexing="ij"))


def l2_inner(x, y, g: Grid):  # core.hpp:218-231
    return float(np.sum(x * y)) * g.cell_volume()


# ---------------------------------------------------------------------------
# projection / embedding (spectral.hpp:194-285, fft.hpp:69-101)


def project(f, b: Band):
    """spectral.hpp:242-260 — full forward DFT, gather retained modes, zero band Nyquist."""
    F = np.fft.fftn(f, axes=tuple(range(-b.d, 0)))
    ix = np.ix_(*[b.parent_index(a) for a in range(b.d)])
    out = F[(Ellipsis,) + ix].copy()
    out[..., b.nyquist_mask()] = 0.0
    return out


def embed(c, b: Band):
    """spectral.hpp:262-285 — scatter into a zero spectrum, backward DFT / N, real part."""
    c = np.asarray(c)
    full = np.zeros(c.shape[:-b.d] + b.grid.dims, dtype=np.complex128)
    cc = c.copy()
    cc[..., b.nyquist_mask()] = 0.0  # scatter skips Nyquist entries (spectral.hpp:220-226)
    ix = np.ix_(*[b.parent_index(a) for a in range(b.d)])
    full[(Ellipsis,) + ix] = cc
    out = np.fft.ifftn(full, axes=tuple(range(-b.d, 0)))
    return out.real.copy()


def spectral_gradient(f, g: Grid):
    """spectral.hpp:326-334,356-370 — full-grid derivative, grid Nyquist zeroed."""
    F = np.fft.fftn(f)
    out = []
    for a in range(g.d):
        n = g.dims[a]
        j = np.arange(n)
        k = np.where(j < n // 2, j, j - n)
        w = np.where(j == n // 2, 0.0, 2 * np.pi * k / (n * g.spacing[a]))
        shape = [1] * g.d
        shape[a] = n
        out.append(np.fft.ifftn(F * (1j * w.reshape(shape))).real)
    return np.stack(out)


def spectral_derivative(f, g: Grid, axis):  # spectral.hpp:347-354
    F = np.fft.fftn(f)
    n = g.dims[axis]
    j = np.arange(n)
    k = np.where(j < n // 2, j, j - n)
    w = np.where(j == n // 2, 0.0, 2 * np.pi * k / (n * g.spacing[axis]))
    shape = [1] * g.d
    shape[axis] = n
    return np.fft.ifftn(F * (1j * w.reshape(shape))).real


# band-diagonal operators (spectral.hpp:419-451)

def band_derivative(c, b: Band, axis):
    shape = [1] * b.d
    shape[axis] = b.bounds[axis]
    return c * (1j * b.omega(axis).reshape(shape))


def band_gradient(c, b: Band):
    return np.stack([band_derivative(c, b, a) for a in range(b.d)])


def band_divergence(v, b: Band):
    return sum(band_derivative(v[a], b, a) for a in range(b.d))


def band_inner(x, y, b: Band):  # spectral.hpp:170-185 (Parseval, h^d / N)
    s = float(np.sum(x.real * y.real + x.imag * y.imag))
    return s * b.grid.cell_volume() / b.grid.size


def linf_norm_band(x):  # spectral.hpp:141-152
    return float(np.max(np.abs(x))) if x.size else 0.0


# truncated products through the parent grid (spectral.hpp:460-510)

def star(a, bf, b: Band):
    """star(scalar, scalar) / star(scalar, vector)."""
    fa = embed(a, b)
    fb = embed(bf, b)
    return project(fa * fb, b)


def star_dot(a, bf, b: Band):
    return project(np.sum(embed(a, b) * embed(bf, b), axis=0), b)


def band_jac_mul(u, w, b: Band):  # spectral.hpp:480-494
    we = embed(w, b)
    acc = np.zeros((b.d,) + b.grid.dims)
    for a in range(b.d):
        for bb in range(b.d):
            acc[a] += embed(band_derivative(u[a], b, bb), b) * we[bb]
    return project(acc, b)


def band_jacT_mul(u, w, b: Band):  # spectral.hpp:496-510
    we = embed(w, b)
    acc = np.zeros((b.d,) + b.grid.dims)
    for a in range(b.d):
        for bb in range(b.d):
            acc[bb] += embed(band_derivative(u[a], b, bb), b) * we[a]
    return project(acc, b)


@dataclass
class Sobolev:  # spectral.hpp:518-544
    alpha: float = 0.0025
    s: int = 2

    def symbol(self, b: Band):
        w2 = sum(w * w for w in b.omega_grids())
        return (1.0 + self.alpha * w2) ** self.s

    def apply(self, v, b: Band, inverse=False):
        m = self.symbol(b)
        return v * (1.0 / m if inverse else m)


def conj_symmetrize(c, b: Band):  # spectral.hpp:289-317
    c = c.copy()
    nyq = b.nyquist_mask()
    flat = c.reshape(-1)
    K = b.bounds
    for i in range(flat.size):
        idx = np.unravel_index(i, K)
        if nyq[idx]:
            flat[i] = 0
            continue
        mir = tuple((K[a] - idx[a]) % K[a] for a in range(b.d))
        j = np.ravel_multi_index(mir, K)
        if j < i:
            continue
        avg = 0.5 * (flat[i] + np.conj(flat[j]))
        flat[i] = avg
        flat[j] = np.conj(avg)
    return c


# ---------------------------------------------------------------------------
# interpolation (interp.hpp)

K_POLE = -0.26794919243112270647  # interp.hpp:18


def prefilter_axis(v, axis):
    """interp.hpp:23-63 — exact periodic cubic B-spline prefilter along one axis
    (vectorised over all lines)."""
    x = np.moveaxis(v, axis, -1).copy()
    n = x.shape[-1]
    z = K_POLE
    zn = z ** n
    denom = 1.0 - zn
    init = np.zeros(x.shape[:-1])
    zp = 1.0
    for m in range(n):
        init += zp * x[..., (n - m) % n]
        zp *= z
    cplus = np.empty_like(x)
    cplus[..., 0] = init / denom
    for k in range(1, n):
        cplus[..., k] = x[..., k] + z * cplus[..., k - 1]
    tail = np.zeros(x.shape[:-1])
    zp = 1.0
    for m in range(n):
        tail += zp * cplus[..., (n - 1 + m) % n]
        zp *= z
    cm = -z * tail / denom
    out = np.empty_like(x)
    out[..., n - 1] = 6.0 * cm
    for k in range(n - 2, -1, -1):
        cm = z * (cm - cplus[..., k])
        out[..., k] = 6.0 * cm
    return np.moveaxis(out, -1, axis)


def spline_coefficients(f):  # interp.hpp:80-84
    out = np.array(f, dtype=np.float64, copy=True)
    for a in range(out.ndim):
        out = prefilter_axis(out, a)
    return out


def cubic_weights(t):  # interp.hpp:65-71
    t2 = t * t
    t3 = t2 * t
    return [(1.0 - 3.0 * t + 3.0 * t2 - t3) / 6.0,
            (4.0 - 6.0 * t2 + 3.0 * t3) / 6.0,
            (1.0 + 3.0 * t + 3.0 * t2 - 3.0 * t3) / 6.0,
            t3 / 6.0]


def sample_cubic(coef, pts, g: Grid):
    """interp.hpp:119-159 — 4^d-tap periodic stencil at physical points.
    coef: spline coefficients [*dims]; pts [d, *dims] (physical)."""
    d = g.d
    idx, wts = [], []
    for a in range(d):
        u = pts[a] / g.spacing[a]
        fl = np.floor(u)
        t = u - fl
        i0 = fl.astype(np.int64)
        wts.append(cubic_weights(t))
        idx.append([np.mod(i0 - 1 + j, g.dims[a]) for j in range(4)])
    out = np.zeros(pts.shape[1:])
    if d == 2:
        for j0 in range(4):
            partial = np.zeros_like(out)
            for j1 in range(4):
                partial += wts[1][j1] * coef[idx[0][j0], idx[1][j1]]
            out += wts[0][j0] * partial
    else:
        for j0 in range(4):
            for j1 in range(4):
                w01 = wts[0][j0] * wts[1][j1]
                partial = np.zeros_like(out)
                for j2 in range(4):
                    partial += wts[2][j2] * coef[idx[0][j0], idx[1][j1], idx[2][j2]]
                out += w01 * partial
    return out


def sample_linear(f, pts, g: Grid):  # interp.hpp:103-117
    d = g.d
    idx, wts = [], []
    for a in range(d):
        u = pts[a] / g.spacing[a]
        fl = np.floor(u)
        t = u - fl
        i0 = fl.astype(np.int64)
        idx.append([np.mod(i0, g.dims[a]), np.mod(i0 + 1, g.dims[a])])
        wts.append([1.0 - t, t])
    out = np.zeros(pts.shape[1:])
    import itertools
    for js in itertools.product(range(2), repeat=d):
        w = np.ones_like(out)
        for a in range(d):
            w = w * wts[a][js[a]]
        out += w * f[tuple(idx[a][js[a]] for a in range(d))]
    return out


def warp(f, pts, g: Grid, kind="cubic"):
    """interp.hpp:178-210 — pull-back out(x) = f(points(x)); f scalar or vector."""
    f = np.asarray(f)
    if f.ndim == g.d + 1:
        return np.stack([warp(f[c], pts, g, kind) for c in range(f.shape[0])])
    if kind == "cubic":
        return sample_cubic(spline_coefficients(f), pts, g)
    if kind == "linear":
        return sample_linear(f, pts, g)
    raise ValueError(kind)


def warp_nearest(f, pts, g: Grid):  # interp.hpp:213-225 (llround: half away from zero)
    idx = []
    for a in range(g.d):
        u = pts[a] / g.spacing[a]
        r = np.where(u >= 0, np.floor(u + 0.5), np.ceil(u - 0.5)).astype(np.int64)
        idx.append(np.mod(r, g.dims[a]))
    return f[tuple(idx)]


# ---------------------------------------------------------------------------
# transport (transport.hpp)


def advect_band(q, pts, b: Band):
    """transport.hpp:67-73 — project(warp(embed(q), X, cubic))."""
    return project(warp(embed(q, b), pts, b.grid, "cubic"), b)


def sl_departure(v_grid, v_traced_coef, dt, direction, g: Grid):
    """transport.hpp:83-102.  v_traced_coef = spline coefficients of the traced velocity."""
    sgn = -1.0 if direction == "forward" else 1.0
    x = identity_map(g)
    xs = x + sgn * dt * v_grid
    vm = np.stack([sample_cubic(v_traced_coef[a], xs, g) for a in range(g.d)])
    return x + sgn * 0.5 * dt * (vm + v_grid)


class Provider:
    """VelocityProvider<BandVectorField> (transport.hpp:109-218); memoised slots."""

    def __init__(self, v, nt, b: Band, stationary=True):
        self.v, self.nt, self.b, self.stationary = v, nt, b, stationary
        self.dt = 1.0 / nt
        self._spatial, self._coef, self._div, self._dep = {}, {}, {}, {}

    def slot(self, i):
        return 0 if self.stationary else i

    def node(self, i):
        return self.v if self.stationary else self.v[i]

    def spatial_node(self, i):
        s = self.slot(i)
        if s not in self._spatial:
            self._spatial[s] = embed(self.node(i), self.b)
        return self._spatial[s]

    def sampler_node(self, i):
        s = self.slot(i)
        if s not in self._coef:
            self._coef[s] = np.stack([spline_coefficients(c) for c in self.spatial_node(i)])
        return self._coef[s]

    def div_node(self, i):
        s = self.slot(i)
        if s not in self._div:
            self._div[s] = band_divergence(self.node(i), self.b)
        return self._div[s]

    def at(self, t):  # transport.hpp:141
        return tv_sample(self.v, t, self.stationary)

    def div_at(self, t):  # transport.hpp:164-172
        if self.stationary:
            return self.div_node(0)
        return _lerp_nodes([self.div_node(i) for i in range(self.nt + 1)], min(max(t, 0.0), 1.0) * self.nt, self.nt)

    def departure(self, step, direction):  # transport.hpp:176-187
        key = (0 if self.stationary else step, direction)
        if key not in self._dep:
            if direction == "forward":
                self._dep[key] = sl_departure(self.spatial_node(step + 1), self.sampler_node(step), self.dt,
                                              direction, self.b.grid)
            else:
                self._dep[key] = sl_departure(self.spatial_node(step), self.sampler_node(step + 1), self.dt,
                                              direction, self.b.grid)
        return self._dep[key]

    def cfl(self):  # transport.hpp:189-194
        last = 0 if self.stationary else self.nt
        vmax = max(float(np.max(np.abs(self.spatial_node(i)))) for i in range(last + 1))
        return vmax * self.dt / self.b.grid.min_spacing()


class Divergence(RuntimeError):
    def __init__(self, step):
        super().__init__(f"transport produced non-finite values (step {step})")
        self.step = step


def sl_integrate(q_init, nt, direction, prov: Provider, src=None):
    """transport.hpp:264-298 — SL-RK2 with trapezoidal source injection."""
    nodes = [None] * (nt + 1)
    dt = 1.0 / nt
    fwd = direction == "forward"
    nodes[0 if fwd else nt] = q_init
    for s in range(nt):
        frm = s if fwd else nt - s
        to = s + 1 if fwd else nt - s - 1
        step = s if fwd else nt - s - 1
        X = prov.departure(step, direction)
        q_from = nodes[frm]
        A = advect_band(q_from, X, prov.b)
        if src is None:
            nxt = A
        else:
            sdt = dt if fwd else -dt
            f_from = advect_band(src(q_from, frm), X, prov.b)
            q_star = sdt * f_from + A
            f_to = src(q_star, to)
            nxt = 0.5 * sdt * f_from + (0.5 * sdt * f_to + A)
        if not np.all(np.isfinite(nxt)):
            raise Divergence(s)
        nodes[to] = nxt
    return nodes


def rk4_integrate(q_init, nt, direction, rhs):
    """transport.hpp:234-258 — classic RK4 on dq/dt = rhs(q, t) (Eulerian right-hand side)."""
    if nt < 2:
        raise ValueError("rk4 requires nt >= 2")
    nodes = [None] * (nt + 1)
    fwd = direction == "forward"
    dt = 1.0 / nt if fwd else -1.0 / nt
    at = 0 if fwd else nt
    nodes[at] = q_init
    for s in range(nt):
        q = nodes[at]
        t = at / nt
        k1 = rhs(q, t)
        k2 = rhs(0.5 * dt * k1 + q, t + 0.5 * dt)
        k3 = rhs(0.5 * dt * k2 + q, t + 0.5 * dt)
        k4 = rhs(dt * k3 + q, t + dt)
        nxt = dt / 6.0 * k1 + (dt / 3.0 * k2 + (dt / 3.0 * k3 + (dt / 6.0 * k4 + q)))
        if not np.all(np.isfinite(nxt)):
            raise Divergence(s)
        at += 1 if fwd else -1
        nodes[at] = nxt
    return nodes


def _lerp_nodes(nodes, u, n):  # shared by sample (core.hpp:303-315) and sample_nodes (transport.hpp:44-54)
    i = min(int(np.floor(u)), n - 1)
    i = max(i, 0)
    w = u - i
    if w < 1e-14:
        return nodes[i]
    if w > 1.0 - 1e-14:
        return nodes[i + 1]
    return (1.0 - w) * nodes[i] + w * nodes[i + 1]


def sample_nodes(nodes, t):  # transport.hpp:44-54 (t clamped to [0, 1])
    n = len(nodes) - 1
    return _lerp_nodes(nodes, min(max(t, 0.0), 1.0) * n, n)


def tv_sample(v, t, stationary):  # TimeVaryingVelocity::sample (core.hpp:303-315)
    if t < -1e-12 or t > 1.0 + 1e-12:
        raise ValueError("sample: t outside [0,1]")
    if stationary:
        return v
    return _lerp_nodes(v, t * (len(v) - 1), len(v) - 1)


# ---------------------------------------------------------------------------
# model (variants.hpp)


def trapezoid_weights(nt):  # variants.hpp:40-46
    w = np.full(nt + 1, 1.0 / nt)
    w[0] *= 0.5
    w[-1] *= 0.5
    return w


def points_from_displacement(disp, g: Grid):  # variants.hpp:49-51
    return identity_map(g) - disp


@dataclass
class Cache:  # variants.hpp:188-224 (the fields the BL SL path uses)
    provider: Provider
    with_adjoint: bool = False
    cfl: float = 0.0
    energy: float = 0.0
    energy_reg: float = 0.0
    energy_data: float = 0.0
    m1: np.ndarray = None
    residual: np.ndarray = None
    m: list = None
    gm: list = None
    lam: list = None
    u: list = None
    phi1_pts: np.ndarray = None
    nu: list = None
    big_u: list = None
    jac_factor: list = None
    psi_pts: list = None
    lam_nodes: list = None
    grad_src_warped: np.ndarray = None
    rho: list = None


@dataclass
class Model:
    """Model<BandAlgebra> with the SL integrator (variants.hpp:229-548)."""
    band: Band
    source: np.ndarray
    target: np.ndarray
    variant: str = "original"
    nt: int = 5
    sigma2: float = 1.0
    lop: Sobolev = field(default_factory=Sobolev)
    stationary: bool = True
    integrator: str = "sl"  # Model::integrator (variants.hpp:35,241): "sl" | "rk4"

    @property
    def grid(self):
        return self.band.grid

    # tv helpers (variants.hpp:65-117)
    def nodes(self, v):
        return [v] if self.stationary else list(v)

    def tv_inner(self, a, b):
        if self.stationary:
            return band_inner(a, b, self.band)
        w = trapezoid_weights(self.nt)
        return sum(w[i] * band_inner(a[i], b[i], self.band) for i in range(self.nt + 1))

    def tv_axpy(self, a, x, y):
        return a * x + y if self.stationary else [a * xi + yi for xi, yi in zip(x, y)]

    def tv_scaled(self, x, a):
        return a * x if self.stationary else [a * xi for xi in x]

    def tv_linf(self, x):
        return max(linf_norm_band(n) for n in self.nodes(x))

    def tv_node(self, dv, i):
        return dv if self.stationary else dv[i]

    def zero_velocity(self):
        z = np.zeros((self.grid.d,) + self.band.bounds, dtype=np.complex128)
        return z if self.stationary else [z.copy() for _ in range(self.nt + 1)]

    # forward (variants.hpp:262-276)
    def forward(self, v, with_adjoint):
        c = Cache(Provider(v, self.nt, self.band, self.stationary))
        c.with_adjoint = with_adjoint
        c.cfl = c.provider.cfl()
        {"original": self._forward_original, "state_equation": self._forward_state,
         "deformation_state_equation": self._forward_deformation}[self.variant](c)
        c.energy_reg = self.reg_energy(v)
        c.energy_data = l2_inner(c.residual, c.residual, self.grid) / self.sigma2
        c.energy = c.energy_reg + c.energy_data
        return c

    def energy(self, v):
        return self.forward(v, False).energy

    def reg_energy(self, v):  # variants.hpp:280-287
        b = self.band
        if self.stationary:
            return 0.5 * band_inner(self.lop.apply(v, b), v, b)
        w = trapezoid_weights(self.nt)
        return 0.5 * sum(w[i] * band_inner(self.lop.apply(v[i], b), v[i], b) for i in range(self.nt + 1))

    def gradient(self, c: Cache):  # variants.hpp:291-309
        b = self.band
        terms = []
        for i in range(self.nt + 1):
            if self.variant == "original":
                terms.append(star(c.lam[i], c.gm[i], b))
            elif self.variant == "state_equation":
                terms.append(star(c.lam_nodes[i], c.gm[i], b))
            else:
                terms.append(-1.0 * band_jacT_mul(c.u[i], c.rho[i], b) + c.rho[i])
        return self._assemble(c.provider.v, terms)

    def hessvec(self, c: Cache, dv):  # variants.hpp:313-344
        b, g = self.band, self.grid
        terms = []
        if self.variant == "original":
            dm = self.solve_incremental_image(c.provider, c.gm, dv)
            dlam1 = dm[-1] * (-2.0 / self.sigma2)
            dlam = self.solve_scalar_continuity_backward(c.provider, dlam1)
            terms = [star(dlam[i], c.gm[i], b) for i in range(self.nt + 1)]
        else:
            du = self.solve_incremental_displacement(c.provider, c.u, dv)
            du1 = embed(du[-1], b)
            dm1 = -1.0 * np.sum(c.grad_src_warped * du1, axis=0)
            dlam1 = dm1 * (-2.0 / self.sigma2)
            if self.variant == "state_equation":
                coef = spline_coefficients(dlam1)
                for i in range(self.nt + 1):
                    dli = c.jac_factor[i] * sample_cubic(coef, c.psi_pts[i], g)
                    terms.append(star(project(dli, b), c.gm[i], b))
            else:
                dr1 = dlam1 * c.grad_src_warped
                drho = self.solve_vector_continuity_backward(c.provider, project(dr1, b))
                terms = [-1.0 * band_jacT_mul(c.u[i], drho[i], b) + drho[i] for i in range(self.nt + 1)]
        return self._assemble(dv, terms)

    def precondition(self, g):  # variants.hpp:347-353
        if self.stationary:
            return self.lop.apply(g, self.band, True)
        return [self.lop.apply(x, self.band, True) for x in g]

    def _assemble(self, like, terms):  # variants.hpp:357-369
        b = self.band
        if self.stationary:
            w = trapezoid_weights(self.nt)
            acc = np.zeros((self.grid.d,) + b.bounds, dtype=np.complex128)
            for i in range(self.nt + 1):
                acc = w[i] * terms[i] + acc
            return 1.0 * self.lop.apply(like, b) + acc
        return [1.0 * self.lop.apply(like[i], b) + terms[i] for i in range(self.nt + 1)]

    # per-variant forward passes (variants.hpp:373-433)
    def _forward_original(self, c):
        b = self.band
        m0 = project(self.source, b)
        c.m = self.solve_image_forward(c.provider, m0)
        c.m1 = embed(c.m[-1], b)
        c.residual = -1.0 * self.target + c.m1
        if not c.with_adjoint:
            return
        c.gm = [band_gradient(m, b) for m in c.m]
        lam1 = project(c.residual * (-2.0 / self.sigma2), b)
        c.lam = self.solve_scalar_continuity_backward(c.provider, lam1)

    def _forward_state(self, c):
        b, g = self.band, self.grid
        c.u = self.solve_displacement(c.provider, "forward")
        c.phi1_pts = points_from_displacement(embed(c.u[-1], b), g)
        src_coef = spline_coefficients(self.source)
        c.m1 = sample_cubic(src_coef, c.phi1_pts, g)
        c.residual = -1.0 * self.target + c.m1
        if not c.with_adjoint:
            return
        c.gm = []
        for i in range(self.nt + 1):
            pts = points_from_displacement(embed(c.u[i], b), g)
            mi = project(sample_cubic(src_coef, pts, g), b)
            c.gm.append(band_gradient(mi, b))
        c.nu = self.solve_displacement(c.provider, "backward")
        c.big_u = self.solve_jacobian_factor(c.provider)
        c.jac_factor = [-1.0 * embed(c.big_u[i], b) + 1.0 for i in range(self.nt + 1)]
        c.psi_pts = [points_from_displacement(embed(c.nu[i], b), g) for i in range(self.nt + 1)]
        lam1 = c.residual * (-2.0 / self.sigma2)
        lcoef = spline_coefficients(lam1)
        c.lam_nodes = [project(c.jac_factor[i] * sample_cubic(lcoef, c.psi_pts[i], g), b)
                       for i in range(self.nt + 1)]
        fg = embed(band_gradient(project(self.source, b), b), b)  # variants.hpp:176-178
        c.grad_src_warped = warp(fg, c.phi1_pts, g, "cubic")

    def _forward_deformation(self, c):
        b, g = self.band, self.grid
        c.u = self.solve_displacement(c.provider, "forward")
        c.phi1_pts = points_from_displacement(embed(c.u[-1], b), g)
        c.m1 = warp(self.source, c.phi1_pts, g, "cubic")
        c.residual = -1.0 * self.target + c.m1
        if not c.with_adjoint:
            return
        c.grad_src_warped = warp(spectral_gradient(self.source, g), c.phi1_pts, g, "cubic")
        r1 = (c.residual * (-2.0 / self.sigma2)) * c.grad_src_warped
        c.rho = self.solve_vector_continuity_backward(c.provider, project(r1, b))

    # equation solvers (variants.hpp:444-547): SL gets the material source at nodes,
    # RK4 the Eulerian right-hand side
    def solve_image_forward(self, pv, m0):
        if self.integrator == "sl":
            return sl_integrate(m0, self.nt, "forward", pv, None)
        b = self.band
        return rk4_integrate(m0, self.nt, "forward",
                             lambda q, t: -1.0 * star_dot(band_gradient(q, b), pv.at(t), b))

    def solve_scalar_continuity_backward(self, pv, q1):
        b = self.band
        if self.integrator == "sl":
            return sl_integrate(q1, self.nt, "backward", pv, lambda q, i: -1.0 * star(q, pv.div_node(i), b))
        return rk4_integrate(q1, self.nt, "backward", lambda q, t: -1.0 * (
            1.0 * star(q, pv.div_at(t), b) + star_dot(band_gradient(q, b), pv.at(t), b)))

    def solve_displacement(self, pv, direction):
        b = self.band
        z = np.zeros((self.grid.d,) + self.band.bounds, dtype=np.complex128)
        if self.integrator == "sl":
            return sl_integrate(z, self.nt, direction, pv, lambda q, i: pv.node(i).copy())

        def rhs(q, t):
            vt = pv.at(t)
            return -1.0 * band_jac_mul(q, vt, b) + vt
        return rk4_integrate(z, self.nt, direction, rhs)

    def solve_jacobian_factor(self, pv):
        b = self.band
        z = np.zeros(self.band.bounds, dtype=np.complex128)
        if self.integrator == "sl":
            def src(q, i):
                dvv = pv.div_node(i)
                return -1.0 * star(q, dvv, b) + dvv
            return sl_integrate(z, self.nt, "backward", pv, src)

        def rhs(q, t):
            dvv = pv.div_at(t)
            return -1.0 * star_dot(band_gradient(q, b), pv.at(t), b) + (-1.0 * star(q, dvv, b) + dvv)
        return rk4_integrate(z, self.nt, "backward", rhs)

    def solve_vector_continuity_backward(self, pv, q1):
        b = self.band
        if self.integrator == "sl":
            return sl_integrate(q1, self.nt, "backward", pv, lambda q, i: -1.0 * star(pv.div_node(i), q, b))
        return rk4_integrate(q1, self.nt, "backward", lambda q, t: -1.0 * (
            1.0 * star(pv.div_at(t), q, b) + band_jac_mul(q, pv.at(t), b)))

    def solve_incremental_image(self, pv, gm, dv):
        b = self.band
        z = np.zeros(self.band.bounds, dtype=np.complex128)
        if self.integrator == "sl":
            return sl_integrate(z, self.nt, "forward", pv,
                                lambda q, i: -1.0 * star_dot(gm[i], self.tv_node(dv, i), b))

        def rhs(q, t):
            gmt = sample_nodes(gm, t)
            return -1.0 * (1.0 * star_dot(gmt, tv_sample(dv, t, self.stationary), b)
                           + star_dot(band_gradient(q, b), pv.at(t), b))
        return rk4_integrate(z, self.nt, "forward", rhs)

    def solve_incremental_displacement(self, pv, u, dv):
        b = self.band
        z = np.zeros((self.grid.d,) + self.band.bounds, dtype=np.complex128)
        if self.integrator == "sl":
            def src(q, i):
                dvi = self.tv_node(dv, i)
                return -1.0 * band_jac_mul(u[i], dvi, b) + dvi
            return sl_integrate(z, self.nt, "forward", pv, src)

        def rhs(q, t):
            dvt = tv_sample(dv, t, self.stationary)
            ut = sample_nodes(u, t)
            return -1.0 * band_jac_mul(q, pv.at(t), b) + (-1.0 * band_jac_mul(ut, dvt, b) + dvt)
        return rk4_integrate(z, self.nt, "forward", rhs)


# ---------------------------------------------------------------------------
# optimizer (optimizer.hpp)

STOP = ["gradient", "energy_change", "step_size", "zero_gradient", "max_iterations", "line_search_failure"]


@dataclass
class Options:  # optimizer.hpp:18-27
    max_iter: int = 50
    pcg_max_iter: int = 5
    pcg_tol: float = 0.1
    grad_tol: float = 1e-2
    energy_tol: float = 1e-4
    step_tol: float = 1e-4
    armijo_c: float = 1e-4
    armijo_max_trials: int = 10


def pcg_solve(model: Model, cache, rhs, max_iter, tol):
    """optimizer.hpp:86-120."""
    info = dict(iters=0, negative_curvature=False, residuals=[])
    x = model.tv_scaled(rhs, 0.0)
    r = rhs
    z = model.precondition(r)
    rz = model.tv_inner(r, z)
    if not (rz > 0.0):
        return x, info
    res0 = math.sqrt(rz)
    p = z
    for k in range(max_iter):
        hp = model.hessvec(cache, p)
        php = model.tv_inner(p, hp)
        if not (php > 0.0):
            info["negative_curvature"] = True
            break
        alpha = rz / php
        x = model.tv_axpy(alpha, p, x)
        r = model.tv_axpy(-alpha, hp, r)
        z = model.precondition(r)
        rz_next = max(model.tv_inner(r, z), 0.0)
        rel = math.sqrt(rz_next) / res0
        info["residuals"].append(rel)
        info["iters"] = k + 1
        if rel <= tol:
            break
        p = model.tv_axpy(rz_next / rz, p, z)
        rz = rz_next
    return x, info


def trial_energy(model, v):  # optimizer.hpp:127-134
    try:
        e = model.energy(v)
        return e if math.isfinite(e) else math.inf
    except Divergence:
        return math.inf


def optimize(model: Model, v0, opt: Options = Options()):
    """optimizer.hpp:143-262; returns dict(v, history, stop, converged, iterations, ...)."""
    g_ = model.grid
    dd = model.source - model.target
    mse_denom = l2_inner(dd, dd, g_)

    def mse_rel(res):
        return l2_inner(res, res, g_) / mse_denom if mse_denom > 0 else 0.0

    out = dict(v=v0, history=[], stop="max_iterations", converged=False, iterations=0)
    cache = model.forward(v0, True)
    g = model.gradient(cache)
    g0 = model.tv_linf(g)
    out["history"].append(dict(iter=0, energy=cache.energy, energy_data=cache.energy_data,
                               energy_reg=cache.energy_reg, mse_rel=mse_rel(cache.residual),
                               rel_grad=1.0 if g0 > 0 else 0.0, pcg_iters=0, pcg_fallback=False,
                               epsilon=0.0, cfl=cache.cfl, pcg_residuals=[]))
    out["m1"], out["residual"], out["final_energy"] = cache.m1, cache.residual, cache.energy
    if g0 == 0.0:
        out.update(stop="zero_gradient", converged=True, rel_grad=0.0)
        return out
    e_prev = cache.energy
    v = v0
    for it in range(1, opt.max_iter + 1):
        rhs = model.tv_scaled(g, -1.0)
        dv, pcg = pcg_solve(model, cache, rhs, opt.pcg_max_iter, opt.pcg_tol)
        gd = model.tv_inner(g, dv)
        fallback = False
        if not (gd < 0.0):
            dv = model.precondition(rhs)
            gd = model.tv_inner(g, dv)
            fallback = True
        eps = 1.0
        accepted = False
        for _ in range(opt.armijo_max_trials):
            e_trial = trial_energy(model, model.tv_axpy(eps, dv, v))
            if e_trial <= e_prev + opt.armijo_c * eps * gd:
                accepted = True
                break
            eps *= 0.5
        if not accepted:
            out.update(stop="line_search_failure", converged=False, v=v)
            return out
        v = model.tv_axpy(eps, dv, v)
        cache = model.forward(v, True)
        g = model.gradient(cache)
        relg = model.tv_linf(g) / g0
        out.update(v=v, iterations=it, m1=cache.m1, residual=cache.residual, final_energy=cache.energy,
                   rel_grad=relg)
        out["history"].append(dict(iter=it, energy=cache.energy, energy_data=cache.energy_data,
                                   energy_reg=cache.energy_reg, mse_rel=mse_rel(cache.residual),
                                   rel_grad=relg, pcg_iters=pcg["iters"], pcg_fallback=fallback,
                                   epsilon=eps, cfl=cache.cfl, pcg_residuals=list(pcg["residuals"])))
        step_norm = eps * model.tv_linf(dv)
        de = abs(e_prev - cache.energy) / max(abs(e_prev), 1e-30)
        e_prev = cache.energy
        if relg <= opt.grad_tol:
            out.update(stop="gradient", converged=True)
            return out
        if de <= opt.energy_tol:
            out.update(stop="energy_change", converged=True)
            return out
        if step_norm <= opt.step_tol:
            out.update(stop="step_size", converged=True)
            return out
    out.update(stop="max_iterations", converged=False)
    return out


# ---------------------------------------------------------------------------
# metrics (metrics.hpp)


def compute_maps(model: Model, v):  # metrics.hpp:24-36
    pv = Provider(v, model.nt, model.band, model.stationary)
    u = model.solve_displacement(pv, "forward")
    nu = model.solve_displacement(pv, "backward")
    fwd = embed(u[-1], model.band)
    inv = embed(nu[0], model.band)
    return fwd, inv


def map_jacobian_determinant(disp, g: Grid):  # metrics.hpp:40-65
    du = [[spectral_derivative(disp[a], g, b) for b in range(g.d)] for a in range(g.d)]
    m = [[(1.0 if a == b else 0.0) - du[a][b] for b in range(g.d)] for a in range(g.d)]
    if g.d == 2:
        return m[0][0] * m[1][1] - m[0][1] * m[1][0]
    return (m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1])
            - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0])
            + m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]))


def mse_rel(warped, target, source, g: Grid):  # metrics.hpp:82-89
    num = warped - target
    den = source - target
    d = l2_inner(den, den, g)
    return 0.0 if d <= 0 else l2_inner(num, num, g) / d


def dice(a, b, label):  # metrics.hpp:97-112 -> (dsc, both_empty)
    ia, ib = (a == label), (b == label)
    na, nb, nab = int(ia.sum()), int(ib.sum()), int((ia & ib).sum())
    if na + nb == 0:
        return 1.0, True
    return 2.0 * nab / (na + nb), False


def mean_dice(warped_labels, target_labels):  # metrics.hpp:114-131 (labels ascending, std::set)
    labels = sorted(set(np.unique(target_labels[target_labels != 0]).tolist()))
    if not labels:
        return dice(warped_labels, target_labels, 1.0)[0]
    s = 0.0
    for lab in labels:
        s += dice(warped_labels, target_labels, lab)[0]
    return s / len(labels)


def rescale_unit(f):  # io.hpp:166-178
    lo, hi = float(np.min(f)), float(np.max(f))
    if hi > lo:
        return (f - lo) * (1.0 / (hi - lo))
    return np.zeros_like(f)
