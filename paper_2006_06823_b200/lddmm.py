"""Python mirror of the reference's registration API over the CUDA engine.

The reference (arxiv 2006.06823, proj/include/lddmm) is a header-only C++
library; its operator surface for the band-limited SL path is
``Model<BandAlgebra>`` + ``optimize`` (variants.hpp:229-548,
optimizer.hpp:18-262).  This module keeps those names and argument meanings
(GridSpec, BandSpec, SobolevOperator, Model.forward/energy/gradient/hessvec/
precondition, OptimizeOptions, IterationRecord, StopReason, optimize,
compute_maps) and calls liblddmm_cuda.so through its C ABI
(include/lddmm_cuda.h).  Device memory is allocated with torch (plumbing
only); every computation runs in the library's sm_100a kernels.  There is
no CPU fallback: a missing library or GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LDDMM_LIB: an alternative in-tree build of the same library (tools/lab variant builds)
LIB_PATH = os.environ.get("LDDMM_LIB") or os.path.join(_HERE, "liblddmm_cuda.so")

_lib = None


class ShapeError(ValueError):
    """core.hpp:27-30."""


class DivergenceError(RuntimeError):
    """core.hpp:33-38 — carries the failing step index."""

    def __init__(self, msg, step=-1):
        super().__init__(msg)
        self.step = step


class CudaError(RuntimeError):
    pass


class _Problem(C.Structure):
    _fields_ = [("d", C.c_int), ("dims", C.c_int * 3), ("spacing", C.c_double * 3), ("band", C.c_int * 3),
                ("nt", C.c_int), ("variant", C.c_int), ("parameterization", C.c_int), ("alpha", C.c_double),
                ("s", C.c_int), ("sigma2", C.c_double), ("integrator", C.c_int)]


INTEGRATORS = {"sl": 0, "rk4": 1}  # include/lddmm_cuda.h LDDMM_SL / LDDMM_RK4


class _Energies(C.Structure):
    _fields_ = [("energy", C.c_double), ("energy_reg", C.c_double), ("energy_data", C.c_double),
                ("cfl", C.c_double)]


class _Options(C.Structure):
    _fields_ = [("max_iter", C.c_int), ("pcg_max_iter", C.c_int), ("pcg_tol", C.c_double),
                ("grad_tol", C.c_double), ("energy_tol", C.c_double), ("step_tol", C.c_double),
                ("armijo_c", C.c_double), ("armijo_max_trials", C.c_int)]


class _Record(C.Structure):
    _fields_ = [("iter", C.c_int), ("energy", C.c_double), ("energy_data", C.c_double),
                ("energy_reg", C.c_double), ("mse_rel", C.c_double), ("rel_grad", C.c_double),
                ("pcg_iters", C.c_int), ("pcg_fallback", C.c_int), ("epsilon", C.c_double), ("cfl", C.c_double),
                ("wall_ms", C.c_double), ("n_pcg_residuals", C.c_int), ("pcg_residuals", C.c_double * 16)]


class _Result(C.Structure):
    _fields_ = [("stop_reason", C.c_int), ("converged", C.c_int), ("iterations", C.c_int),
                ("n_history", C.c_int), ("final_energy", C.c_double), ("rel_grad", C.c_double),
                ("hessvecs", C.c_int), ("trials", C.c_int), ("forwards", C.c_int)]


def lib():
    """Load liblddmm_cuda.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                              "(make -C paper_2006_06823_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.lddmm_last_error.restype = C.c_char_p
        L.lddmm_last_error.argtypes = [vp]
        L.lddmm_create.argtypes = [C.POINTER(_Problem), C.c_int, C.POINTER(vp)]
        L.lddmm_destroy.argtypes = [vp]
        L.lddmm_launch_count.restype = C.c_longlong
        L.lddmm_velocity_doubles.restype = C.c_longlong
        L.lddmm_velocity_doubles.argtypes = [vp]
        for name, args in {
            "lddmm_sync": [vp],
            "lddmm_set_images": [vp, vp, vp],
            "lddmm_set_images_dev_f32": [vp, vp, vp],
            "lddmm_vel_axpy": [vp, C.c_double, vp, vp, vp],
            "lddmm_vel_scale": [vp, vp, C.c_double, vp],
            "lddmm_vel_inner": [vp, vp, vp, C.POINTER(C.c_double)],
            "lddmm_vel_upload": [vp, vp, vp],
            "lddmm_vel_download": [vp, vp, vp],
            "lddmm_vel_linf": [vp, vp, C.POINTER(C.c_double)],
            "lddmm_vel_all_finite": [vp, vp, C.POINTER(C.c_int)],
            "lddmm_forward": [vp, vp, C.c_int, C.POINTER(_Energies), C.POINTER(C.c_int)],
            "lddmm_energy": [vp, vp, C.POINTER(C.c_double), C.POINTER(C.c_int)],
            "lddmm_gradient": [vp, vp],
            "lddmm_hessvec": [vp, vp, vp, C.POINTER(C.c_int)],
            "lddmm_precondition": [vp, vp, vp],
            "lddmm_get_fields": [vp, vp, vp],
            "lddmm_get_series": [vp, C.c_int, vp],
            "lddmm_get_grid": [vp, C.c_int, vp],
            "lddmm_optimize": [vp, vp, C.POINTER(_Options), C.POINTER(_Record), C.c_int, C.POINTER(_Result)],
            "lddmm_register": [vp, vp, vp, C.POINTER(_Options), vp, C.POINTER(_Record), C.c_int,
                               C.POINTER(_Result)],
            "lddmm_maps": [vp, vp, vp, vp, C.POINTER(C.c_double)],
            "lddmm_op_embed": [vp, vp, C.c_int, vp, C.c_int],
            "lddmm_op_project": [vp, vp, C.c_int, vp],
            "lddmm_op_advect": [vp, vp, C.c_int, vp, vp],
            "lddmm_op_departure": [vp, vp, vp, vp, C.POINTER(C.c_double)],
            "lddmm_op_band": [vp, C.c_int, vp, vp, vp],
            "lddmm_op_warp": [vp, vp, C.c_int, vp, vp],
            "lddmm_op_gather": [vp, C.c_int, vp, C.c_int, vp, vp],
            "lddmm_op_warp_nearest": [vp, vp, C.c_int, vp, vp],
            "lddmm_op_jacobian": [vp, vp, vp, C.POINTER(C.c_double)],
            "lddmm_op_mean_dice": [vp, vp, vp, C.POINTER(C.c_double)],
            "lddmm_warp": [vp, C.c_int, vp, C.c_int, vp, vp],
            "lddmm_jacobian": [vp, vp, vp, C.POINTER(C.c_double)],
            "lddmm_mean_dice": [vp, vp, vp, C.POINTER(C.c_double)],
            "lddmm_vel_from_spatial": [vp, vp, vp],
            "lddmm_vel_to_spatial": [vp, vp, C.c_int, vp],
        }.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = C.c_int
        L.lddmm_default_options.argtypes = [C.POINTER(_Options)]
        L.lddmm_stream.restype = C.c_void_p
        L.lddmm_stream.argtypes = [vp]
        L.lddmm_gather_timing.argtypes = [vp, C.c_int]
        L.lddmm_gather_stats.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_longlong),
                                         C.POINTER(C.c_double)]
        L.lddmm_dft_stats.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_longlong), C.POINTER(C.c_double)]
        _lib = L
    return _lib


def launch_count() -> int:
    return int(lib().lddmm_launch_count())


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise CudaError("the CUDA engine needs a GPU (torch.cuda.is_available() is False)")
    return torch


# ---------------------------------------------------------------------------
# reference value types


@dataclass(frozen=True)
class GridSpec:  # core.hpp:42-122
    dims: tuple
    spacing: tuple = (1.0, 1.0, 1.0)

    @property
    def d(self):
        return len(self.dims)

    def size(self):
        return int(np.prod(self.dims))


@dataclass(frozen=True)
class BandSpec:  # spectral.hpp:22-83
    parent: GridSpec
    bounds: tuple

    @staticmethod
    def uniform(g: GridSpec, k: int):
        return BandSpec(g, tuple(min(k, n) for n in g.dims))

    def size(self):
        return int(np.prod(self.bounds))


@dataclass
class SobolevOperator:  # spectral.hpp:518-525
    alpha: float = 0.0025
    s: int = 2


@dataclass
class OptimizeOptions:  # optimizer.hpp:18-27
    max_iter: int = 50
    pcg_max_iter: int = 5
    pcg_tol: float = 0.1
    grad_tol: float = 1e-2
    energy_tol: float = 1e-4
    step_tol: float = 1e-4
    armijo_c: float = 1e-4
    armijo_max_trials: int = 10

    def _c(self):
        return _Options(self.max_iter, self.pcg_max_iter, self.pcg_tol, self.grad_tol, self.energy_tol,
                        self.step_tol, self.armijo_c, self.armijo_max_trials)


STOP_REASONS = ["gradient", "energy_change", "step_size", "zero_gradient", "max_iterations",
                "line_search_failure"]  # optimizer.hpp:29-36
VARIANTS = {"original": 0, "state_equation": 1, "deformation_state_equation": 2}


@dataclass
class IterationRecord:  # optimizer.hpp:50-61
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
    wall_ms: float
    pcg_residuals: list = field(default_factory=list)


@dataclass
class OptimizeResult:  # optimizer.hpp:63-74
    v: "Velocity"
    history: list
    stop: str
    converged: bool
    iterations: int
    final_energy: float
    rel_grad: float
    hessvecs: int = 0
    trials: int = 0
    forwards: int = 0


def _records(buf, n):
    out = []
    for k in range(n):
        r = buf[k]
        out.append(IterationRecord(r.iter, r.energy, r.energy_data, r.energy_reg, r.mse_rel, r.rel_grad,
                                   r.pcg_iters, bool(r.pcg_fallback), r.epsilon, r.cfl, r.wall_ms,
                                   [r.pcg_residuals[j] for j in range(r.n_pcg_residuals)]))
    return out


# ---------------------------------------------------------------------------
# context


class Context:
    """One engine context (device memory + stream) for one registration problem."""

    def __init__(self, band: BandSpec, variant="deformation_state_equation", nt=5, sigma2=1.0,
                 lop: SobolevOperator = None, parameterization="stationary", device=0, integrator="sl"):
        lop = lop or SobolevOperator()
        g = band.parent
        if g.d not in (2, 3):
            raise ShapeError("grid dimension must be 2 or 3 (core.hpp:49-52)")
        p = _Problem()
        p.d = g.d
        for a in range(3):
            p.dims[a] = g.dims[a] if a < g.d else 1
            p.spacing[a] = float(g.spacing[a]) if a < g.d else 1.0
            p.band[a] = band.bounds[a] if a < g.d else 1
        p.nt = nt
        p.variant = VARIANTS[variant]
        p.parameterization = 0 if parameterization == "stationary" else 1
        p.alpha = lop.alpha
        p.s = lop.s
        p.sigma2 = sigma2
        if integrator not in INTEGRATORS:
            raise ShapeError(f"unknown integrator: {integrator} (expected sl or rk4)")
        p.integrator = INTEGRATORS[integrator]
        h = C.c_void_p()
        rc = lib().lddmm_create(C.byref(p), int(device), C.byref(h))
        if rc != 0:
            self.h = None
            _raise(rc, lib().lddmm_last_error(None).decode())
        self.h = h
        self.band, self.grid, self.nt, self.device = band, g, nt, device
        self.nodes = 1 if parameterization == "stationary" else nt + 1

    def __del__(self):
        h = getattr(self, "h", None)
        self.h = None
        if h and _lib is not None:
            try:
                _lib.lddmm_destroy(h)
            except Exception:  # interpreter shutdown
                pass

    def check(self, rc, step=None):
        if rc != 0:
            msg = lib().lddmm_last_error(self.h).decode()
            _raise(rc, msg, step.value if step is not None else -1)

    @property
    def vel_shape(self):
        """Host layout of a velocity (the reference's BandVectorField per node)."""
        return (self.nodes, self.grid.d) + tuple(self.band.bounds)

    @property
    def dev_vel_shape(self):
        """Device layout: 3-D; a 2-D problem runs with its z axis replicated (Problem::zrep),
        only the kz = 0 plane of the x, y components non-zero, scaled by the replica count."""
        if self.grid.d == 3:
            return self.vel_shape
        return (self.nodes, 3) + tuple(self.band.bounds) + (4,)

    def stream_ptr(self):
        return int(lib().lddmm_stream(self.h))

    def sync(self):
        self.check(lib().lddmm_sync(self.h))

    def gather_timing(self, on=True, dft=False):
        """CUDA events around every SL gather (and, with dft=True, every full-grid DFT call)."""
        self.check(lib().lddmm_gather_timing(self.h, (1 if on else 0) | (2 if dft else 0)))

    def gather_stats(self):
        ms, n, b = C.c_double(), C.c_longlong(), C.c_double()
        self.check(lib().lddmm_gather_stats(self.h, C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value

    def dft_stats(self):
        ms, n, f = C.c_double(), C.c_longlong(), C.c_double()
        self.check(lib().lddmm_dft_stats(self.h, C.byref(ms), C.byref(n), C.byref(f)))
        return ms.value, n.value, f.value


def _raise(rc, msg, step=-1):
    if rc == 1:
        raise ShapeError(msg)
    if rc == 2:
        raise DivergenceError(msg, step)
    raise CudaError(msg)


class Velocity:
    """TimeVaryingVelocity<BandVectorField> (core.hpp:275-317) resident on the device.

    Storage: torch float64 CUDA tensor [nodes, 3, Kx, Ky, Kz, 2] (interleaved re/im); a 2-D
    problem keeps the engine's internal 3-D layout on the device (Context.dev_vel_shape) and
    converts through lddmm_vel_upload / lddmm_vel_download."""

    def __init__(self, ctx: Context, data=None):
        torch = _torch()
        self.ctx = ctx
        self.t = torch.zeros(ctx.dev_vel_shape + (2,), dtype=torch.float64, device=f"cuda:{ctx.device}")
        if data is not None:
            self.set(data)

    def ptr(self):
        return C.c_void_p(self.t.data_ptr())

    def set(self, data):
        torch = _torch()
        if self.ctx.grid.d == 2:
            if isinstance(data, torch.Tensor):
                data = data.detach().cpu().numpy()
                if not np.iscomplexobj(data):
                    data = data.view(np.complex128)
            a = np.ascontiguousarray(np.asarray(data, dtype=np.complex128).reshape(self.ctx.vel_shape))
            torch.cuda.synchronize(self.ctx.device)
            self.ctx.check(lib().lddmm_vel_upload(self.ctx.h, self.ptr(), a.ctypes.data_as(C.c_void_p)))
            return self
        if isinstance(data, torch.Tensor):
            if data.is_complex():
                data = torch.view_as_real(data)
            self.t.copy_(data.reshape(self.t.shape))
        else:
            a = np.asarray(data, dtype=np.complex128).reshape(self.ctx.vel_shape)
            self.t.copy_(torch.from_numpy(a.view(np.float64).reshape(self.t.shape)))
        return self

    def numpy(self):
        torch = _torch()
        torch.cuda.synchronize(self.ctx.device)
        if self.ctx.grid.d == 2:
            out = np.zeros(self.ctx.vel_shape, dtype=np.complex128)
            self.ctx.check(lib().lddmm_vel_download(self.ctx.h, self.ptr(), out.ctypes.data_as(C.c_void_p)))
            return out
        return self.t.cpu().numpy().view(np.complex128).reshape(self.ctx.vel_shape)

    def copy(self):
        v = Velocity(self.ctx)
        v.t.copy_(self.t)
        return v


class Model:
    """Model<BandAlgebra> (variants.hpp:229-548) on one B200; integrator "sl" (SL-RK2,
    the default) or "rk4" (transport.hpp:234-258)."""

    def __init__(self, band: BandSpec, source, target, variant="deformation_state_equation", nt=5, sigma2=1.0,
                 lop: SobolevOperator = None, parameterization="stationary", device=0, integrator="sl"):
        self.ctx = Context(band, variant, nt, sigma2, lop, parameterization, device, integrator)
        self.integrator = integrator
        self.band, self.variant, self.nt, self.sigma2 = band, variant, nt, sigma2
        self.lop = lop or SobolevOperator()
        self.set_images(source, target)

    @property
    def grid(self):
        return self.band.parent

    def set_images(self, source, target):
        torch = _torch()
        if isinstance(source, torch.Tensor) and source.is_cuda:
            for x in (source, target):
                if not (isinstance(x, torch.Tensor) and x.is_cuda):
                    raise ShapeError("model images: both source and target must be CUDA tensors (or both host)")
                if tuple(x.shape) != tuple(self.grid.dims):
                    raise ShapeError("model images must live on the domain grid")
                if x.device.index != self.ctx.device:
                    raise ShapeError(f"model images live on cuda:{x.device.index}, the context on cuda:{self.ctx.device}")
            s = source.to(torch.float32).contiguous()
            t = target.to(torch.float32).contiguous()
            self.ctx.check(lib().lddmm_set_images_dev_f32(self.ctx.h, C.c_void_p(s.data_ptr()),
                                                          C.c_void_p(t.data_ptr())))
        else:
            s = np.ascontiguousarray(source, dtype=np.float64)
            t = np.ascontiguousarray(target, dtype=np.float64)
            if s.shape != tuple(self.grid.dims) or t.shape != tuple(self.grid.dims):
                raise ShapeError("model images must live on the domain grid")
            self.ctx.check(lib().lddmm_set_images(self.ctx.h, s.ctypes.data_as(C.c_void_p),
                                                  t.ctypes.data_as(C.c_void_p)))

    def zero_velocity(self):
        return Velocity(self.ctx)

    def velocity(self, data):
        return Velocity(self.ctx, data)

    def forward(self, v: Velocity, with_adjoint=True):
        e = _Energies()
        step = C.c_int(-1)
        self.ctx.check(lib().lddmm_forward(self.ctx.h, v.ptr(), int(with_adjoint), C.byref(e), C.byref(step)), step)
        return dict(energy=e.energy, energy_reg=e.energy_reg, energy_data=e.energy_data, cfl=e.cfl)

    def energy(self, v: Velocity):
        x = C.c_double()
        step = C.c_int(-1)
        self.ctx.check(lib().lddmm_energy(self.ctx.h, v.ptr(), C.byref(x), C.byref(step)), step)
        return x.value

    def gradient(self):
        out = Velocity(self.ctx)
        self.ctx.check(lib().lddmm_gradient(self.ctx.h, out.ptr()))
        return out

    def hessvec(self, dv: Velocity):
        out = Velocity(self.ctx)
        step = C.c_int(-1)
        self.ctx.check(lib().lddmm_hessvec(self.ctx.h, dv.ptr(), out.ptr(), C.byref(step)), step)
        return out

    def precondition(self, g: Velocity):
        out = Velocity(self.ctx)
        self.ctx.check(lib().lddmm_precondition(self.ctx.h, g.ptr(), out.ptr()))
        return out

    def fields(self):
        n = self.grid.size()
        m1 = np.zeros(n)
        r = np.zeros(n)
        self.ctx.check(lib().lddmm_get_fields(self.ctx.h, m1.ctypes.data_as(C.c_void_p),
                                              r.ctypes.data_as(C.c_void_p)))
        return m1.reshape(self.grid.dims), r.reshape(self.grid.dims)

    GRID_FIELDS = {"m1": 0, "residual": 1, "gsw0": 2, "gsw1": 3, "gsw2": 4, "I0coef": 5, "gI0coef0": 6,
                   "gI0coef1": 7, "gI0coef2": 8, "I1": 9}

    def grid_field(self, name):
        out = np.zeros(self.grid.size())
        self.ctx.check(lib().lddmm_get_grid(self.ctx.h, self.GRID_FIELDS[name], out.ctypes.data_as(C.c_void_p)))
        return out.reshape(self.grid.dims)

    def series(self, which="u"):
        shape = (self.nt + 1, self.grid.d) + tuple(self.band.bounds)
        out = np.zeros(int(np.prod(shape)) * 2)
        self.ctx.check(lib().lddmm_get_series(self.ctx.h, 0 if which == "u" else 1, out.ctypes.data_as(C.c_void_p)))
        return out.view(np.complex128).reshape(shape)

    # TV algebra (variants.hpp:70-117)
    def tv_inner(self, a: Velocity, b: Velocity):
        x = C.c_double()
        self.ctx.check(lib().lddmm_vel_inner(self.ctx.h, a.ptr(), b.ptr(), C.byref(x)))
        return x.value

    def tv_linf(self, a: Velocity):
        x = C.c_double()
        self.ctx.check(lib().lddmm_vel_linf(self.ctx.h, a.ptr(), C.byref(x)))
        return x.value

    def tv_axpy(self, a, x: Velocity, y: Velocity):
        out = Velocity(self.ctx)
        self.ctx.check(lib().lddmm_vel_axpy(self.ctx.h, float(a), x.ptr(), y.ptr(), out.ptr()))
        return out


def optimize(model: Model, v0: Velocity = None, opt: OptimizeOptions = None) -> OptimizeResult:
    """optimize(model, v0, opt) (optimizer.hpp:143-262) — the GN-Krylov loop runs in C++ on the host,
    every operator on the device."""
    opt = opt or OptimizeOptions()
    v = (v0.copy() if v0 is not None else model.zero_velocity())
    cap = opt.max_iter + 2
    recs = (_Record * cap)()
    res = _Result()
    o = opt._c()
    model.ctx.check(lib().lddmm_optimize(model.ctx.h, v.ptr(), C.byref(o), recs, cap, C.byref(res)))
    hist = _records(recs, min(res.n_history, cap))
    return OptimizeResult(v, hist, STOP_REASONS[res.stop_reason], bool(res.converged), res.iterations,
                          res.final_energy, res.rel_grad, res.hessvecs, res.trials, res.forwards)


def register_host(ctx: Context, I0, I1, opt: OptimizeOptions = None, v_out=None):
    """End-to-end registration from host buffers (lddmm_cli.cpp:101-125): returns (v, result).
    Host arrays may live in pinned memory (e.g. numpy views of pinned torch tensors);
    v_out, when given, is a complex128 array of ctx.vel_shape that receives the velocity."""
    opt = opt or OptimizeOptions()
    I0 = np.ascontiguousarray(I0, dtype=np.float64)
    I1 = np.ascontiguousarray(I1, dtype=np.float64)
    if I0.shape != tuple(ctx.grid.dims) or I1.shape != tuple(ctx.grid.dims):
        raise ShapeError(f"register_host: images must have the grid shape {tuple(ctx.grid.dims)}")
    v = v_out if v_out is not None else np.zeros(ctx.vel_shape, dtype=np.complex128)
    if v.shape != tuple(ctx.vel_shape) or v.dtype != np.complex128 or not v.flags.c_contiguous:
        raise ShapeError("register_host: v_out must be C-contiguous complex128 of ctx.vel_shape")
    cap = opt.max_iter + 2
    recs = (_Record * cap)()
    res = _Result()
    o = opt._c()
    ctx.check(lib().lddmm_register(ctx.h, I0.ctypes.data_as(C.c_void_p), I1.ctypes.data_as(C.c_void_p),
                                   C.byref(o), v.ctypes.data_as(C.c_void_p), recs, cap, C.byref(res)))
    hist = _records(recs, min(res.n_history, cap))
    return v, OptimizeResult(None, hist, STOP_REASONS[res.stop_reason], bool(res.converged), res.iterations,
                             res.final_energy, res.rel_grad, res.hessvecs, res.trials, res.forwards)


def maps_jacobian(ctx: Context, v_host):
    """Jacobian determinant ranges of the maps of a host band velocity (metrics.hpp:24-79):
    [fwd min, fwd max, inv min, inv max]; no displacement fields are copied back."""
    v = Velocity(ctx, v_host)
    jac = (C.c_double * 4)()
    ctx.check(lib().lddmm_maps(ctx.h, v.ptr(), None, None, jac))
    return np.array(list(jac))


def compute_maps(model: Model, v: Velocity):
    """compute_maps + map_jacobian_determinant ranges (metrics.hpp:24-79).
    Returns (forward_disp, inverse_disp, jac) with jac = [fmin, fmax, imin, imax]."""
    n = model.grid.d * model.grid.size()
    f = np.zeros(n)
    i = np.zeros(n)
    jac = (C.c_double * 4)()
    model.ctx.check(lib().lddmm_maps(model.ctx.h, v.ptr(), f.ctypes.data_as(C.c_void_p),
                                     i.ctypes.data_as(C.c_void_p), jac))
    shape = (model.grid.d,) + tuple(model.grid.dims)
    return f.reshape(shape), i.reshape(shape), np.array(list(jac))


# ---------------------------------------------------------------------------
# evaluation path on host arrays (metrics.hpp:24-131, interp.hpp:178-225)

INTERP = {"linear": 0, "cubic": 1, "nearest": 2}


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def warp(ctx: Context, field, disp, kind="cubic"):
    """warp(f, x - disp, cubic) / warp_nearest(f, x - disp) (interp.hpp:178-225); field
    [N...] or [C, N...], disp [d, N...] in physical units; fp32 on the device."""
    f = _f64(field)
    nc = 1 if f.ndim == ctx.grid.d else f.shape[0]
    out = np.zeros_like(f)
    d = _f64(disp)
    ctx.check(lib().lddmm_warp(ctx.h, INTERP[kind], f.ctypes.data_as(C.c_void_p), nc, d.ctypes.data_as(C.c_void_p),
                               out.ctypes.data_as(C.c_void_p)))
    return out


def jacobian(ctx: Context, disp, want_field=False):
    """map_jacobian_determinant + value_range (metrics.hpp:40-79) of a grid displacement."""
    d = _f64(disp)
    det = np.zeros(d.shape[1:]) if want_field else None
    mm = (C.c_double * 2)()
    ctx.check(lib().lddmm_jacobian(ctx.h, d.ctypes.data_as(C.c_void_p),
                                   det.ctypes.data_as(C.c_void_p) if want_field else None, mm))
    return (mm[0], mm[1], det) if want_field else (mm[0], mm[1])


def mean_dice(ctx: Context, warped_labels, target_labels):
    """mean_dice (metrics.hpp:92-131), exact counts on the device."""
    a, b = _f64(warped_labels), _f64(target_labels)
    out = C.c_double()
    ctx.check(lib().lddmm_mean_dice(ctx.h, a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                    C.byref(out)))
    return out.value


def mse_rel(warped, target, source):
    """|warped - target|^2 / |source - target|^2 (metrics.hpp:82-89), fp64 on the host
    (the reference's scalar loop order)."""
    w, t, s = (np.ravel(_f64(x)) for x in (warped, target, source))
    num, den = w - t, s - t
    d = float(np.dot(den, den))
    return 0.0 if d <= 0.0 else float(np.dot(num, num)) / d


def velocity_from_spatial(model: "Model", field) -> "Velocity":
    """Alg::from_spatial (project) of a grid vector field into every node (--v0)."""
    v = model.zero_velocity()
    f = _f64(field)
    model.ctx.check(lib().lddmm_vel_from_spatial(model.ctx.h, f.ctypes.data_as(C.c_void_p), v.ptr()))
    return v


def velocity_to_spatial(model: "Model", v: "Velocity", node=0):
    """Alg::to_spatial (embed) of one velocity node -> [d, N...] grid field."""
    out = np.zeros((model.grid.d,) + tuple(model.grid.dims))
    model.ctx.check(lib().lddmm_vel_to_spatial(model.ctx.h, v.ptr(), int(node), out.ctypes.data_as(C.c_void_p)))
    return out


# ---------------------------------------------------------------------------
# primitives on device tensors (parity tests)


class Ops:
    """Direct access to the engine's primitives on torch CUDA tensors."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        self.torch = _torch()

    def _band(self, x, ncomp=None):
        t = self.torch
        if isinstance(x, np.ndarray):
            x = t.from_numpy(np.ascontiguousarray(x, dtype=np.complex128).view(np.float64)).cuda(self.ctx.device)
        return x.contiguous()

    def band_out(self, ncomp):
        return self.torch.zeros((ncomp,) + tuple(self.ctx.band.bounds) + (2,), dtype=self.torch.float64,
                                device=f"cuda:{self.ctx.device}")

    def grid_out(self, ncomp):
        return self.torch.zeros((ncomp,) + tuple(self.ctx.grid.dims), dtype=self.torch.float32,
                                device=f"cuda:{self.ctx.device}")

    @staticmethod
    def to_complex(t):
        return t.cpu().numpy().view(np.complex128)[..., 0]

    def embed(self, c, ncomp, prefilter=False):
        c = self._band(c)
        out = self.grid_out(ncomp)
        self.ctx.check(lib().lddmm_op_embed(self.ctx.h, C.c_void_p(c.data_ptr()), ncomp,
                                            C.c_void_p(out.data_ptr()), int(prefilter)))
        return out

    def project(self, f):
        f = f.to(self.torch.float32).contiguous()
        nc = f.shape[0]
        out = self.band_out(nc)
        self.ctx.check(lib().lddmm_op_project(self.ctx.h, C.c_void_p(f.data_ptr()), nc, C.c_void_p(out.data_ptr())))
        return out

    def advect(self, q, ncomp, dep):
        q = self._band(q)
        dep = dep.to(self.torch.float32).contiguous()
        out = self.band_out(ncomp)
        self.ctx.check(lib().lddmm_op_advect(self.ctx.h, C.c_void_p(q.data_ptr()), ncomp,
                                             C.c_void_p(dep.data_ptr()), C.c_void_p(out.data_ptr())))
        return out

    def departure(self, v):
        v = self._band(v)
        df = self.grid_out(3)
        db = self.grid_out(3)
        cfl = C.c_double()
        self.ctx.check(lib().lddmm_op_departure(self.ctx.h, C.c_void_p(v.data_ptr()), C.c_void_p(df.data_ptr()),
                                                C.c_void_p(db.data_ptr()), C.byref(cfl)))
        return df, db, cfl.value

    def band(self, op, a, b, ncomp_out):
        a = self._band(a)
        b = self._band(b) if b is not None else a
        out = self.band_out(ncomp_out)
        self.ctx.check(lib().lddmm_op_band(self.ctx.h, int(op), C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                           C.c_void_p(out.data_ptr())))
        return out

    def gather(self, coef, dep, impl=0):
        coef = coef.to(self.torch.float32).contiguous()
        dep = dep.to(self.torch.float32).contiguous()
        nc = coef.shape[0]
        out = self.grid_out(nc)
        self.ctx.check(lib().lddmm_op_gather(self.ctx.h, int(impl), C.c_void_p(coef.data_ptr()), nc,
                                             C.c_void_p(dep.data_ptr()), C.c_void_p(out.data_ptr())))
        return out

    def warp_nearest(self, f, disp):
        f = f.to(self.torch.float32).contiguous()
        disp = disp.to(self.torch.float32).contiguous()
        out = self.grid_out(f.shape[0])
        self.ctx.check(lib().lddmm_op_warp_nearest(self.ctx.h, C.c_void_p(f.data_ptr()), f.shape[0],
                                                   C.c_void_p(disp.data_ptr()), C.c_void_p(out.data_ptr())))
        return out

    def jacobian(self, disp):
        disp = disp.to(self.torch.float32).contiguous()
        det = self.grid_out(1)
        mm = (C.c_double * 2)()
        self.ctx.check(lib().lddmm_op_jacobian(self.ctx.h, C.c_void_p(disp.data_ptr()), C.c_void_p(det.data_ptr()),
                                               mm))
        return det[0], (mm[0], mm[1])

    def mean_dice(self, a, b):
        a = a.to(self.torch.float32).contiguous()
        b = b.to(self.torch.float32).contiguous()
        out = C.c_double()
        self.ctx.check(lib().lddmm_op_mean_dice(self.ctx.h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                                C.byref(out)))
        return out.value

    def warp(self, f, disp):
        f = f.to(self.torch.float32).contiguous()
        disp = disp.to(self.torch.float32).contiguous()
        nc = f.shape[0]
        out = self.grid_out(nc)
        self.ctx.check(lib().lddmm_op_warp(self.ctx.h, C.c_void_p(f.data_ptr()), nc, C.c_void_p(disp.data_ptr()),
                                           C.c_void_p(out.data_ptr())))
        return out
