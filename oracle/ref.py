"""ctypes binding of oracle/_ref/libref_lddmm.so — the UNMODIFIED reference
(/root/reference/proj/include, header-only C++) compiled in place by
oracle/Makefile together with our FFTW3-API shim.

TEST INFRASTRUCTURE ONLY: imported by tests/, tests/golden/make_golden.py and
bench.py's reference / cpu_baseline legs.  The product package never imports
this module.

Layouts follow the reference:
  grid field   float64[ncomp, *dims]   (core.hpp:8-9, axis 0 slowest)
  band field   complex128[ncomp, *band] (spectral.hpp:8-12, DFT order)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libref_lddmm.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle ref)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_model_create.restype = C.c_void_p
        _lib.ref_model_destroy.argtypes = [C.c_void_p]
        for name in ("ref_band_inner", "ref_cfl", "ref_model_energy"):
            getattr(_lib, name).restype = C.c_double
    return _lib


def set_threads(n: int) -> None:
    lib().ref_set_threads(int(n))


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def _i(seq):
    arr = (C.c_int * 3)(*([int(x) for x in seq] + [1] * (3 - len(seq))))
    return arr


def _check(rc, what):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == 2:
        raise RefDivergence(msg)
    raise RefError(f"{what}: {msg}")


class RefError(RuntimeError):
    pass


class RefDivergence(RefError):
    pass


def _cplx_view(buf, shape):
    return buf.view(np.complex128).reshape(shape)


def _grid_args(dims, spacing):
    d = len(dims)
    return d, _i(dims), (C.c_double * 3)(*(list(map(float, spacing)) + [1.0] * (3 - d)))


# ---- spectral.hpp -------------------------------------------------------------

def embed(coeffs, dims, spacing, band):
    coeffs = np.asarray(coeffs, dtype=np.complex128)
    nc = coeffs.shape[0]
    d, di, hi = _grid_args(dims, spacing)
    cb, cp = _d(coeffs.view(np.float64))
    out = np.zeros((nc,) + tuple(dims))
    ob, op = _d(out)
    _check(lib().ref_embed(d, di, hi, _i(band), nc, cp, op), "embed")
    return ob


def project(field, dims, spacing, band):
    field = np.asarray(field, dtype=np.float64)
    nc = field.shape[0]
    d, di, hi = _grid_args(dims, spacing)
    fb, fp = _d(field)
    out = np.zeros(nc * int(np.prod(band)) * 2)
    ob, op = _d(out)
    _check(lib().ref_project(d, di, hi, _i(band), nc, fp, op), "project")
    return _cplx_view(ob, (nc,) + tuple(band))


BAND_OPS = {"star_ss": (0, 1), "star_sv": (1, None), "star_dot": (2, 1), "jac": (3, None),
            "jacT": (4, None), "grad": (5, None), "div": (6, 1), "sobolev": (7, None),
            "sobolev_inv": (8, None)}


def band_op(name, a, b, dims, spacing, band, alpha=0.0025, s=2):
    op, outc = BAND_OPS[name]
    d = len(dims)
    outc = outc or d
    d_, di, hi = _grid_args(dims, spacing)
    ab, ap = _d(np.asarray(a, dtype=np.complex128).view(np.float64))
    if b is None:
        b = np.zeros(1, dtype=np.complex128)
    bb, bp = _d(np.asarray(b, dtype=np.complex128).view(np.float64))
    out = np.zeros(outc * int(np.prod(band)) * 2)
    ob, op_ = _d(out)
    _check(lib().ref_band_op(op, d_, di, hi, _i(band), ap, bp, op_, C.c_double(alpha), int(s)), name)
    return _cplx_view(ob, (outc,) + tuple(band))


def band_inner(x, y, dims, spacing, band):
    x = np.asarray(x, dtype=np.complex128)
    d, di, hi = _grid_args(dims, spacing)
    xb, xp = _d(x.view(np.float64))
    yb, yp = _d(np.asarray(y, dtype=np.complex128).view(np.float64))
    return lib().ref_band_inner(d, di, hi, _i(band), x.shape[0], xp, yp)


def spectral_gradient(f, dims, spacing):
    d, di, hi = _grid_args(dims, spacing)
    fb, fp = _d(f)
    out = np.zeros((d,) + tuple(dims))
    ob, op = _d(out)
    _check(lib().ref_spectral_gradient(d, di, hi, fp, op), "spectral_gradient")
    return ob


# ---- interp.hpp ---------------------------------------------------------------

def spline_coefficients(f, dims, spacing):
    d, di, hi = _grid_args(dims, spacing)
    fb, fp = _d(f)
    out = np.zeros(tuple(dims))
    ob, op = _d(out)
    _check(lib().ref_spline_coefficients(d, di, hi, fp, op), "spline_coefficients")
    return ob


def warp(f, pts, dims, spacing, kind="cubic"):
    f = np.asarray(f, dtype=np.float64)
    if f.ndim == len(dims):
        f = f[None]
    nc = f.shape[0]
    d, di, hi = _grid_args(dims, spacing)
    fb, fp = _d(f)
    pb, pp = _d(pts)
    out = np.zeros((nc,) + tuple(dims))
    ob, op = _d(out)
    k = {"linear": 0, "cubic": 1, "nearest": 2}[kind]
    _check(lib().ref_warp(d, di, hi, nc, fp, pp, k, op), "warp")
    return ob


# ---- transport.hpp --------------------------------------------------------------

def departure(v, dims, spacing, band, nt, direction="forward"):
    d, di, hi = _grid_args(dims, spacing)
    vb, vp = _d(np.asarray(v, dtype=np.complex128).view(np.float64))
    out = np.zeros((d,) + tuple(dims))
    ob, op = _d(out)
    _check(lib().ref_departure(d, di, hi, _i(band), nt, vp, 0 if direction == "forward" else 1, op),
           "departure")
    return ob


def advect_band(q, pts, dims, spacing, band):
    q = np.asarray(q, dtype=np.complex128)
    nc = q.shape[0]
    d, di, hi = _grid_args(dims, spacing)
    qb, qp = _d(q.view(np.float64))
    pb, pp = _d(pts)
    out = np.zeros(nc * int(np.prod(band)) * 2)
    ob, op = _d(out)
    _check(lib().ref_advect_band(d, di, hi, _i(band), nc, qp, pp, op), "advect")
    return _cplx_view(ob, (nc,) + tuple(band))


def cfl(v, dims, spacing, band, nt):
    d, di, hi = _grid_args(dims, spacing)
    vb, vp = _d(np.asarray(v, dtype=np.complex128).view(np.float64))
    return lib().ref_cfl(d, di, hi, _i(band), nt, vp)


# ---- variants.hpp / optimizer.hpp ---------------------------------------------

VARIANTS = {"original": 0, "state_equation": 1, "deformation_state_equation": 2}
STOP_REASONS = ["gradient", "energy_change", "step_size", "zero_gradient", "max_iterations",
                "line_search_failure"]


@dataclass
class IterationRecord:
    iter: int
    energy: float
    energy_data: float
    energy_reg: float
    mse_rel: float
    rel_grad: float
    pcg_iters: int
    pcg_fallback: bool
    epsilon: float
    cfl: float
    pcg_residuals: list


class RefModel:
    """Model<BandAlgebra> of the reference (variants.hpp:229-548), SL integrator."""

    def __init__(self, I0, I1, dims, spacing, band, variant="deformation_state_equation", nt=5,
                 sigma2=1.0, alpha=0.0025, s=2, param="stationary", integrator="sl"):
        self.dims, self.spacing, self.band = tuple(dims), tuple(spacing), tuple(band)
        self.d = len(dims)
        self.nt = nt
        self.param = param
        d, di, hi = _grid_args(dims, spacing)
        self._i0, ip0 = _d(I0)
        self._i1, ip1 = _d(I1)
        h = lib().ref_model_create(d, di, hi, _i(band), ip0, ip1, VARIANTS[variant], nt,
                                   C.c_double(sigma2), C.c_double(alpha), int(s),
                                   0 if param == "stationary" else 1)
        if not h:
            raise RefError(lib().ref_last_error().decode())
        self.h = C.c_void_p(h)
        if integrator != "sl":
            _check(lib().ref_model_set_integrator(self.h, 1 if integrator == "rk4" else 0), "set_integrator")

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_model_destroy(self.h)
            self.h = None

    @property
    def nodes(self):
        return 1 if self.param == "stationary" else self.nt + 1

    def _vshape(self):
        return (self.nodes, self.d) + self.band

    def _vin(self, v):
        v = np.asarray(v, dtype=np.complex128).reshape(self._vshape())
        return _d(v.view(np.float64))

    def _vout(self):
        return np.zeros(int(np.prod(self._vshape())) * 2)

    def forward(self, v, with_adjoint=True):
        vb, vp = self._vin(v)
        e = np.zeros(4)
        eb, ep = _d(e)
        step = C.c_int(-1)
        _check(lib().ref_model_forward(self.h, vp, int(with_adjoint), ep, C.byref(step)), "forward")
        return dict(energy=eb[0], energy_reg=eb[1], energy_data=eb[2], cfl=eb[3])

    def fields(self):
        n = int(np.prod(self.dims))
        m1 = np.zeros(n)
        r = np.zeros(n)
        mb, mp = _d(m1)
        rb, rp = _d(r)
        _check(lib().ref_model_fields(self.h, mp, rp), "fields")
        return mb.reshape(self.dims), rb.reshape(self.dims)

    def series(self, which="u"):
        out = np.zeros((self.nt + 1) * self.d * int(np.prod(self.band)) * 2)
        ob, op = _d(out)
        _check(lib().ref_model_series(self.h, 0 if which == "u" else 1, op), "series")
        return _cplx_view(ob, (self.nt + 1, self.d) + self.band)

    def _vop(self, fn, v):
        vb, vp = self._vin(v)
        ob, op = _d(self._vout())
        _check(fn(self.h, vp, op), fn.__name__)
        return _cplx_view(ob, self._vshape())

    def gradient(self):
        ob, op = _d(self._vout())
        _check(lib().ref_model_gradient(self.h, op), "gradient")
        return _cplx_view(ob, self._vshape())

    def hessvec(self, dv):
        return self._vop(lib().ref_model_hessvec, dv)

    def precondition(self, g):
        return self._vop(lib().ref_model_precondition, g)

    def energy(self, v):
        vb, vp = self._vin(v)
        return lib().ref_model_energy(self.h, vp)

    def optimize(self, v0=None, max_iter=50, pcg_max_iter=5, pcg_tol=0.1, grad_tol=1e-2,
                 energy_tol=1e-4, step_tol=1e-4):
        if v0 is None:
            v0 = np.zeros(self._vshape(), dtype=np.complex128)
        vb, vp = self._vin(v0)
        cap = max_iter + 2
        rec = np.zeros(cap * 10)
        pres = np.zeros(cap * 8)
        info = (C.c_int * 4)()
        wall = C.c_double(0)
        rb, rp = _d(rec)
        pb, pp = _d(pres)
        _check(lib().ref_optimize(self.h, vp, max_iter, pcg_max_iter, C.c_double(pcg_tol),
                                  C.c_double(grad_tol), C.c_double(energy_tol), C.c_double(step_tol),
                                  cap, rp, pp, info, C.byref(wall)), "optimize")
        n = info[0]
        hist = []
        for k in range(min(n, cap)):
            o = rb[k * 10:(k + 1) * 10]
            pr = [x for x in pb[k * 8:(k + 1) * 8] if x >= 0]
            hist.append(IterationRecord(int(o[0]), o[1], o[2], o[3], o[4], o[5], int(o[6]), bool(o[7]),
                                        o[8], o[9], pr))
        return dict(v=_cplx_view(vb, self._vshape()).copy(), history=hist, stop=STOP_REASONS[info[1]],
                    converged=bool(info[2]), iterations=info[3], wall_ms=wall.value)

    def maps(self, v):
        vb, vp = self._vin(v)
        n = self.d * int(np.prod(self.dims))
        f = np.zeros(n)
        i = np.zeros(n)
        j = np.zeros(4)
        fb, fp = _d(f)
        ib, ip = _d(i)
        jb, jp = _d(j)
        _check(lib().ref_maps(self.h, vp, fp, ip, jp), "maps")
        return fb.reshape((self.d,) + self.dims), ib.reshape((self.d,) + self.dims), jb


def jacobian_determinant(disp, dims, spacing):
    d, di, hi = _grid_args(dims, spacing)
    db, dp = _d(disp)
    out = np.zeros(tuple(dims))
    ob, op = _d(out)
    _check(lib().ref_jacobian_determinant(d, di, hi, dp, op), "jacobian")
    return ob


# ---- timing of the reference's own primitives (bench cpu_baseline) -------------------

def time_ops(dims, spacing, band, mask=0b0111):
    """Milliseconds of one reference FFT / prefilter / cubic gather / vector advect at `dims`."""
    d, di, hi = _grid_args(dims, spacing)
    t = np.full(4, np.nan)
    tb, tp = _d(t)
    _check(lib().ref_time_ops(d, di, hi, _i(band), int(mask), tp), "time_ops")
    return dict(fft=tb[0], prefilter=tb[1], gather=tb[2], advect=tb[3])


def defstate_op_counts_measured(nt, forwards, hessvecs, trials):
    """As defstate_op_counts, for a run that did `forwards` adjoint forwards (+ gradients),
    `hessvecs` Hessian-vector products and `trials` energy-only line-search trials."""
    nt_ = nt
    fwd_adj = dict(fft=38 * nt_ + 13, warp=12 * nt_ + 4, pre=3, gath=6)
    energy = dict(fft=12 * nt_ + 6, warp=6 * nt_ + 1, pre=3, gath=3)
    grad = dict(fft=15 * (nt_ + 1), warp=0, pre=0, gath=0)
    hv = dict(fft=83 * nt_ + 21, warp=12 * nt_, pre=0, gath=0)
    return {k: forwards * (fwd_adj[k] + grad[k]) + hessvecs * hv[k] + trials * energy[k] for k in fwd_adj}


def defstate_op_counts(nt, gn_iters, pcg_per_iter, trials_per_iter=1):
    """Full-grid transform / warp counts of one reference registration (deformation-state
    variant, SL, stationary, band-limited), read off the reference code paths:
      forward+adjoint 38nt+13 FFTs (variants.hpp:424-433, transport.hpp:264-298),
      energy-only 12nt+6, gradient 15(nt+1) (band_jacT_mul: 3+9 embeds, 3 projects),
      hessvec 83nt+21 (variants.hpp:313-344); scalar cubic warps (prefilter + gather):
      forward+adjoint 12nt+4, energy 6nt+1, hessvec 12nt; plus the provider's sampler
      prefilters (3) and departure gathers (3 per direction)."""
    fwd_adj = dict(fft=38 * nt + 13, warp=12 * nt + 4, pre=3, gath=6)
    energy = dict(fft=12 * nt + 6, warp=6 * nt + 1, pre=3, gath=3)
    grad = dict(fft=15 * (nt + 1), warp=0, pre=0, gath=0)
    hv = dict(fft=83 * nt + 21, warp=12 * nt, pre=0, gath=0)
    tot = {k: fwd_adj[k] + grad[k] for k in fwd_adj}
    for _ in range(gn_iters):
        for k in tot:
            tot[k] += pcg_per_iter * hv[k] + trials_per_iter * energy[k] + fwd_adj[k] + grad[k]
    return tot


def registration_cost_ms(times, counts):
    return (counts["fft"] * times["fft"] + counts["warp"] * (times["prefilter"] + times["gather"])
            + counts["pre"] * times["prefilter"] + counts["gath"] * times["gather"])


# ---- synth.hpp / io.hpp -------------------------------------------------------------

def blob_pair(dims, spacing, seed):
    d, di, hi = _grid_args(dims, spacing)
    s = np.zeros(tuple(dims))
    t = np.zeros(tuple(dims))
    sb, sp = _d(s)
    tb, tp = _d(t)
    _check(lib().ref_blob_pair(d, di, hi, C.c_ulonglong(seed), sp, tp), "blob_pair")
    return sb, tb


def two_disc_case(dims, spacing, seed):
    d, di, hi = _grid_args(dims, spacing)
    bufs = [np.zeros(tuple(dims)) for _ in range(4)]
    ptrs = [_d(b) for b in bufs]
    _check(lib().ref_two_disc_case(d, di, hi, C.c_ulonglong(seed), *[p for _, p in ptrs]), "two_disc")
    return tuple(b for b, _ in ptrs)


def evaluate(dims, spacing, warped=None, target=None, source=None, warped_labels=None, target_labels=None,
             disp=None):
    """mse_rel / mean_dice / map_jacobian_determinant + value_range (metrics.hpp:40-131)."""
    d, di, hi = _grid_args(dims, spacing)
    keep = []

    def arg(x):
        if x is None:
            return None
        b, p = _d(np.asarray(x, dtype=np.float64))
        keep.append(b)
        return p
    mse, dice = C.c_double(-1.0), C.c_double(-1.0)
    jac = np.zeros(2)
    det = np.zeros(tuple(dims))
    jb, jp = _d(jac)
    db, dp = _d(det)
    _check(lib().ref_evaluate(d, di, hi, arg(warped), arg(target), arg(source), arg(warped_labels),
                              arg(target_labels), arg(disp), C.byref(mse), C.byref(dice), jp, dp), "evaluate")
    return dict(mse_rel=mse.value, dice_mean=dice.value, jac=jb.copy(), det=db.copy())


def random_band_field(dims, spacing, band, seed, amplitude, k0):
    d, di, hi = _grid_args(dims, spacing)
    out = np.zeros(d * int(np.prod(band)) * 2)
    ob, op = _d(out)
    _check(lib().ref_random_band_field(d, di, hi, _i(band), C.c_ulonglong(seed), C.c_double(amplitude),
                                       C.c_double(k0), op), "random_band_field")
    return _cplx_view(ob, (d,) + tuple(band))


def random_smooth_image(dims, spacing, seed, k0):
    d, di, hi = _grid_args(dims, spacing)
    out = np.zeros(tuple(dims))
    ob, op = _d(out)
    _check(lib().ref_random_smooth_image(d, di, hi, C.c_ulonglong(seed), C.c_double(k0), op), "img")
    return ob


def random_smooth_field(dims, spacing, seed, amplitude, k0):
    d, di, hi = _grid_args(dims, spacing)
    out = np.zeros((d,) + tuple(dims))
    ob, op = _d(out)
    _check(lib().ref_random_smooth_field(d, di, hi, C.c_ulonglong(seed), C.c_double(amplitude),
                                         C.c_double(k0), op), "field")
    return ob


def rescale_unit(f, dims, spacing):
    d, di, hi = _grid_args(dims, spacing)
    fb, fp = _d(f)
    out = np.zeros(tuple(dims))
    ob, op = _d(out)
    _check(lib().ref_rescale_unit(d, di, hi, fp, op), "rescale")
    return ob
