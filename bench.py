#!/usr/bin/env python
"""Benchmark: seconds per registration of the band-limited SL-RK2 GN-Krylov
deformation-state LDDMM path (BASELINE.json metric) on B200.

A step is one full registration with the reference's OptimizeOptions defaults and
max_iter = 10, pcg_max_iter = 5 (the paper's budget), images
resident in HBM when the step starts.  The per-registration image constants (I0
spline coefficients, spectral gradient) are inside the step.  L2 is flushed (512 MiB
write) between steps.

  N = 1: BASELINE.json configs[1] — the synthetic 180x210x180 brain-like pair (band
         32^3, nt=10, deformation-state, stationary, sigma2 = 0.01).
  N > 1: BASELINE.json configs[4] — the config-5 all-pairs sweep of 16 subjects:
         step s on rank r registers pair (s * N + r) of the 240 ordered pairs (one
         process per GPU, no collective on the data path; the per-rank times are
         gathered with one NCCL all_gather at the end and the max over ranks is used).
         Launched under torchrun by the driver, or re-executed under torchrun by this
         script when --gpus N > 1 and WORLD_SIZE is unset.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Extra keys: `roofline` (the SL gather, HBM), `roofline_dft` (the full-grid truncated
DFT pipelines, FP32), `fixed_work` (the reference's iteration-cap mode, every
tolerance 0: 10 GN x 5 PCG, test_optimizer.cpp:197-207), `e2e` (through the C ABI
lddmm_register from pinned host fp64 buffers), `cpu_baseline`.

--impl reference times the reference CPU implementation (oracle/_ref: the unmodified
reference headers compiled with our FFTW3-API shim) on this host, 1 thread (the
reference is single-threaded by construction): per step, one real reference
advect_state (transport.hpp:67-73) of one component at config 2 plus one full-grid
FFT / prefilter / cubic gather, extrapolated to a registration with the reference's
own operation counts for its config-2 run.  The full config-2 reference solve,
measured once offline (5965 s on 8 host threads, tests/golden/config2_ref.npz), is
reported beside it.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "s per registration (180x210x180, BL SL-RK2); SL-gather GB/s vs HBM peak"
DIMS = (180, 210, 180)
BAND = (32, 32, 32)
NT = 10
SIGMA2 = 0.01
GN, PCG = 10, 5


def workload(dims=DIMS, band=BAND, nt=NT):
    return {"workload": f"config2: {dims[0]}x{dims[1]}x{dims[2]} synthetic brain-like pair, BL band "
                        f"{band[0]}^3, deformation-state, SL-RK2 nt={nt}, stationary, sigma2={SIGMA2}, "
                        f"reference OptimizeOptions defaults with max_iter={GN}, pcg_max_iter={PCG}",
            "dims": list(dims), "band": list(band), "nt": nt, "variant": "deformation_state_equation",
            "mode": "parity (reference defaults, max_iter 10)", "l2": "flushed (512 MiB write) between steps", "parallelism": "pairs/rank"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


_ADVECT_MS = {}


def cpu_reference_cost(threads=1, dims=DIMS, band=BAND, nt=NT, measured=None, source="our run"):
    """Reference CPU s/registration for the same workload (see module doc).  measured =
    (forwards, hessvecs, trials) of a run gives the identical operation sequence;
    without it the nominal budget GN x PCG x 1 trial is used."""
    from oracle import ref
    ref.set_threads(threads)
    t0 = time.time()
    times = ref.time_ops(dims, (1.0, 1.0, 1.0), band, mask=0b0111)
    # once per process: one real reference advect_state (embed -> prefilter -> cubic warp
    # -> project) of a scalar band field along a sub-voxel departure field, the composed
    # hot-path op, as a check of the primitive model
    key = (dims, band, threads)
    if key not in _ADVECT_MS:
        rng = np.random.default_rng(0)
        q = ref.random_band_field(dims, (1.0, 1.0, 1.0), band, 7, 1.0, 3.0)[:1]
        x = np.stack(np.meshgrid(*[np.arange(n, dtype=np.float64) for n in dims], indexing="ij"))
        pts = x + 0.25 * np.sin(x / 7.0 + rng.uniform(0, 6, size=(3, 1, 1, 1)))
        t1 = time.time()
        ref.advect_band(q, pts, dims, (1.0, 1.0, 1.0), band)
        _ADVECT_MS[key] = (time.time() - t1) * 1000.0
    t_adv = _ADVECT_MS[key]
    sample_s = time.time() - t0
    if measured is not None:
        counts = ref.defstate_op_counts_measured(nt, *measured)
        how = (f"the op sequence of {source} ({measured[0]} forwards+gradients, {measured[1]} hessvecs, "
               f"{measured[2]} trials)")
    else:
        counts = ref.defstate_op_counts(nt, GN, PCG, 1)
        how = f"the nominal budget {GN} GN x {PCG} PCG x 1 trial"
    ms = ref.registration_cost_ms(times, counts)
    model_adv = 2 * times["fft"] + times["prefilter"] + times["gather"]
    sample = (f"reference code timed at {dims[0]}x{dims[1]}x{dims[2]} on {threads} thread(s): 1 full-grid complex "
              f"FFT {times['fft']:.0f} ms, 1 spline prefilter {times['prefilter']:.0f} ms, 1 cubic gather "
              f"{times['gather']:.0f} ms, 1 scalar advect_state {t_adv:.0f} ms (the model 2 FFT + prefilter + "
              f"gather predicts {model_adv:.0f} ms); {sample_s:.1f} s of CPU work. Extrapolated with the reference "
              f"op counts of {how} at nt={nt}: {counts['fft']} FFTs, {counts['warp']} warps, {counts['pre']} "
              f"prefilters, {counts['gath']} gathers (band-space ops not counted). FFT = FFTW3-API shim "
              f"(libfftw3 absent)")
    return ms / 1000.0, sample, {"fft_ms": times["fft"], "prefilter_ms": times["prefilter"],
                                 "gather_ms": times["gather"], "advect_state_1comp_ms": t_adv, "counts": counts}


def measured_reference_solve():
    """The reference's own full config-2 solve, run once offline (tools/ref_config2_golden.py)."""
    path = os.path.join(ROOT, "tests", "golden", "config2_ref.npz")
    if not os.path.exists(path):
        return None
    d = np.load(path)
    return {"value": float(d["wall_s"]), "unit": "s/registration", "threads": int(d["threads"]),
            "source": "tests/golden/config2_ref.npz (reference optimize on this workload, run offline)"}


def reference_op_sequence():
    """(forwards, hessvecs, trials) of the reference's own config-2 registration, read
    from its GN history (tests/golden/config2_ref.npz: 3 GN iterations, PCG 2+3+4,
    epsilon 1 each): forward+gradient per history row, one hessvec per PCG iteration,
    log2(1/epsilon) + 1 Armijo trials per iteration.  None if the fixture is absent."""
    path = os.path.join(ROOT, "tests", "golden", "config2_ref.npz")
    if not os.path.exists(path):
        return None
    h = np.load(path)["history"]
    forwards = int(h.shape[0])
    hessvecs = int(np.sum(h[1:, 6]))
    trials = int(sum(1 + round(np.log2(1.0 / e)) for e in h[1:, 8] if e > 0))
    return forwards, hessvecs, trials


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref_lddmm.so not built"}))
        return
    threads = 1  # the reference is single-threaded by construction
    measured = reference_op_sequence()
    src = "the reference's own config-2 run (tests/golden/config2_ref.npz)"
    for _ in range(max(0, args.warmup)):
        cpu_reference_cost(threads, measured=measured, source=src)
    vals = []
    sample, parts = "", {}
    for _ in range(max(1, args.steps)):
        v, sample, parts = cpu_reference_cost(threads, measured=measured, source=src)
        vals.append(v)
    value = float(np.mean(vals))
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s/registration", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1000.0, "higher_is_better": False,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload(),
           "cpu_baseline": {"value": value, "unit": "s/registration", "cores": threads, "kind": "reference",
                            "extrapolated": True, "sample": sample, "parts": parts,
                            "measured_full_solve": measured_reference_solve()},
           "e2e": {"value": value, "unit": "s/registration", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def ncu_traffic():
    """DRAM bytes of one captured gather launch (profiles/r2s2_ncu_traffic.json, from
    `ncu --set full`), next to that launch's algorithmic bytes N (12 + 8 F)."""
    path = os.path.join(ROOT, "profiles", "r2s2_ncu_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return {"traffic": t["dram_bytes"], "traffic_launch_algorithmic_bytes": t["algorithmic_bytes"],
                "traffic_source": "profiles/r2s2_ncu_traffic.json (" + t["kernel"] + ", one launch)"}
    except (OSError, KeyError, ValueError):
        return {"traffic": None}


def dft_flops_per_field(dims=DIMS, band=BAND):
    """Algorithmic flops of one full-grid truncated transform, half band along z (SURVEY.md
    §8d): 8 x complex MACs of the y stage (Kx H Ky Ny) and x stage (Ny H Kx Nx) + 4 x
    real-complex MACs of the z stage (Nx Ny Nz H); 617.8 MFLOP at config 2 (the engine
    counts the same per field, Engine::dft_flops_per_field)."""
    Nx, Ny, Nz = dims
    Kx, Ky, H = band[0], band[1], band[2] // 2
    return 8.0 * (Kx * H * Ky * Ny + Ny * H * Kx * Nx) + 4.0 * Nx * Ny * Nz * H


def fp32_peak():
    """FP32 FFMA peak of one B200: 148 SMs x 128 FMA/clk x 2 flop x 1.965 GHz = 74.4 TFLOP/s
    nominal; tools/lab/fma_pipe.cu measured 126.6 FMA/clk/SM with packed FFMA2 (73.6
    TFLOP/s), which is the denominator used (MEASURED_PEAKS.json has no FP32 entry)."""
    return 73.6, "measured (tools/lab/fma_pipe.cu, FFMA2 at 1965 MHz)"


def spawn_torchrun(n):
    """--gpus N > 1 without a torchrun environment: re-execute under torchrun (one rank per GPU)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def sweep_workload(n, steps, warmup):
    return {"workload": f"config5: all-pairs sweep of 16 synthetic {DIMS[0]}x{DIMS[1]}x{DIMS[2]} brain-like subjects "
                        f"(240 ordered pairs), BL band {BAND[0]}^3, deformation-state, SL-RK2 nt={NT}, stationary, "
                        f"sigma2={SIGMA2}, reference OptimizeOptions defaults with max_iter={GN}, pcg_max_iter={PCG}; "
                        f"step s on rank r registers pair s*N+r (after {warmup} warm-up pairs per rank)",
            "dims": list(DIMS), "band": list(BAND), "nt": NT, "variant": "deformation_state_equation",
            "mode": "parity (reference defaults, max_iter 10)", "l2": "flushed (512 MiB write) between steps",
            "parallelism": f"pairs sharded over {n} ranks, no collective on the data path"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fixed-work", action="store_true")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_torchrun(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # nranks / transport in the log for the driver
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2006_06823_b200 import lddmm as L
    from paper_2006_06823_b200 import phantoms
    from paper_2006_06823_b200 import sweep

    dev = f"cuda:{local}"
    band = L.BandSpec(L.GridSpec(DIMS), BAND)
    # the pairs this rank registers: [warm-up pairs] + [timed pairs]
    if world == 1:
        I0, I1 = phantoms.brain_pair(DIMS, seed=2006)
        pair_imgs = [(I0, I1)] * (args.warmup + args.steps)
        config = workload()
    else:
        pl = sweep.pair_list(16)
        idx = [(len(pl) - 1 - (w * world + rank)) % len(pl) for w in range(args.warmup)] + \
              [(s * world + rank) % len(pl) for s in range(args.steps)]
        subj = {}

        def S(k):
            if k not in subj:
                subj[k] = phantoms.subject(DIMS, k)
            return subj[k]
        pair_imgs = [(S(pl[i][0]), S(pl[i][1])) for i in idx]
        config = sweep_workload(world, args.steps, args.warmup)
    dimgs = [(torch.from_numpy(a).to(device=dev, dtype=torch.float32),
              torch.from_numpy(b).to(device=dev, dtype=torch.float32)) for a, b in pair_imgs]
    model = L.Model(band, dimgs[0][0], dimgs[0][1], "deformation_state_equation", NT, SIGMA2, device=local)
    ctx = model.ctx
    opt = L.OptimizeOptions(max_iter=GN, pcg_max_iter=PCG)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def one_registration(k, o=opt):
        model.set_images(*dimgs[k])
        return L.optimize(model, None, o)

    for w in range(args.warmup):
        res = one_registration(w)
    torch.cuda.synchronize()

    step_ms = []
    results = []
    launches0 = L.launch_count()
    ctx.gather_timing(True)
    with Clocks(local) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        for s in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = one_registration(args.warmup + s)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            results.append(res)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    g_ms, g_n, g_bytes = ctx.gather_stats()
    ctx.gather_timing(False)
    launches = L.launch_count() - launches0
    # the DFT roofline from one more registration of the same pair with events around every
    # full-grid DFT call (kept out of the timed steps: ~2 us of event overhead per call)
    ctx.gather_timing(False, dft=True)
    flush.fill_(1.0)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    one_registration(args.warmup)
    e1.record(stream)
    e1.synchronize()
    dft_step_ms = e0.elapsed_time(e1)
    d_ms, d_n, d_flops = ctx.dft_stats()
    ctx.gather_timing(False)

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        return max(float(a.item()) for a in allt)

    total_ms = max_over_ranks(float(np.sum(step_ms)))
    value = total_ms / 1000.0 / (world * args.steps)
    hbm, peak_kind = peaks()
    achieved = (g_bytes / g_n) / (g_ms / g_n * 1e-3) / 1e9 if g_n else 0.0
    # the same gathers against the FP32 pipe: component-samples sum C N over the launches
    # (bytes = N (12 + 8 C) per launch), 84 FMA per sample for the exact separable 4-tap
    # stencil (64 z-dots + 16 + 4) and 150 for the 5 x 5-row / 5-tap window form the
    # kernel executes (DESIGN 4.1); 2 flop per FMA
    npts = float(np.prod(DIMS))
    g_samples = (g_bytes - 12.0 * npts * g_n) / 8.0 if g_n else 0.0
    g_s = g_ms * 1e-3 if g_n else 1.0
    fp32, fp32_kind = fp32_peak()
    dft_tflops = d_flops / (d_ms * 1e-3) / 1e12 if d_n else 0.0

    # fixed-work mode: every tolerance 0 -> exactly max_iter GN x pcg_max_iter PCG
    fixed = None
    if not args.no_fixed_work:
        fopt = L.OptimizeOptions(max_iter=GN, pcg_max_iter=PCG, grad_tol=0.0, energy_tol=0.0, step_tol=0.0,
                                 pcg_tol=0.0)
        one_registration(args.warmup, fopt)
        f_ms = []
        for _ in range(2):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fres = one_registration(args.warmup, fopt)
            e1.record(stream)
            e1.synchronize()
            f_ms.append(e0.elapsed_time(e1))
        fixed = {"value": max_over_ranks(float(np.mean(f_ms))) / 1000.0, "unit": "s/registration",
                 "mode": "fixed work: grad_tol = energy_tol = step_tol = pcg_tol = 0, max_iter 10, pcg 5 "
                         "(test_optimizer.cpp:197-207)", "steps": len(f_ms),
                 "gn_iterations": fres.iterations, "hessvecs": fres.hessvecs, "trials": fres.trials,
                 "stop": fres.stop,
                 # with every tolerance 0 the solve runs until the Armijo search fails at the
                 # fp noise floor, a point that moves with rounding: the per-iteration figure
                 # is the comparable one
                 "s_per_gn_iteration": max_over_ranks(float(np.mean(f_ms))) / 1000.0 / max(1, fres.iterations)}

    e2e = None
    if not args.no_e2e:
        ectx = L.Context(band, "deformation_state_equation", NT, SIGMA2, device=local)
        # inputs and the result velocity in pinned host memory (the reference's fp64
        # ScalarField / BandVectorField layouts): the same fp32-representable images the
        # device arm registers (so both arms do the same GN work); W untimed warm-up calls
        hosts = [(torch.from_numpy(a.astype(np.float32).astype(np.float64)).pin_memory().numpy(),
                  torch.from_numpy(b.astype(np.float32).astype(np.float64)).pin_memory().numpy())
                 for a, b in pair_imgs]
        v_host = torch.zeros(ectx.vel_shape + (2,), dtype=torch.float64).pin_memory().numpy().view(np.complex128)
        v_host = v_host.reshape(ectx.vel_shape)
        for w in range(max(1, args.warmup)):
            L.register_host(ectx, *hosts[min(w, len(hosts) - 1)], opt, v_out=v_host)
        e_ms = []
        for s in range(max(1, args.steps)):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            v_host, r2 = L.register_host(ectx, *hosts[args.warmup + s], opt, v_out=v_host)
            e_ms.append((time.perf_counter() - t0) * 1000.0)
        e2e_ms = max_over_ranks(float(np.sum(e_ms)))
        e2e = {"value": e2e_ms / 1000.0 / (world * len(e_ms)), "unit": "s/registration",
               "h2d_bytes_per_step": int(2 * pair_imgs[0][0].size * 8), "d2h_bytes_per_step": int(v_host.nbytes),
               "path": "lddmm_register (C ABI): pinned host fp64 images in, pinned host fp64 velocity out",
               "result": {"iterations": r2.iterations, "hessvecs": r2.hessvecs, "trials": r2.trials,
                          "forwards": r2.forwards, "final_energy": r2.final_energy}}
        del ectx

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            if ref.available():
                v, sample, parts = cpu_reference_cost(1, measured=(res.forwards, res.hessvecs, res.trials))
                cpu = {"value": v, "unit": "s/registration", "cores": 1, "kind": "reference", "extrapolated": True,
                       "sample": sample, "measured_full_solve": measured_reference_solve()}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unavailable": str(exc)}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "s/registration", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": False,
               "scaling": "weak", "vs_baseline": None, "dtype": "f32 grid / f64 band", "data": "synthetic",
               "config": config,
               "roofline": {"kernel": "gather_pipe_kernel (SL cubic gather, TMA-staged)", "bound": "hbm",
                            "achieved": achieved, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                            "frac": achieved / hbm, **ncu_traffic(),
                            "algorithmic_bytes_per_launch": g_bytes / g_n if g_n else 0,
                            "launches_timed": g_n, "gather_share_of_step": g_ms / total_ms if total_ms else 0},
               "roofline_gather_fp32": {"kernel": "gather_pipe_kernel", "bound": "fp32", "unit": "TFLOP/s",
                                        "achieved_minimal": 2 * 84 * g_samples / g_s / 1e12,
                                        "achieved_executed": 2 * 150 * g_samples / g_s / 1e12,
                                        "peak": fp32, "peak_kind": fp32_kind,
                                        "frac_minimal": 2 * 84 * g_samples / g_s / 1e12 / fp32,
                                        "frac_executed": 2 * 150 * g_samples / g_s / 1e12 / fp32,
                                        "fma_per_sample": {"minimal": 84, "executed": 150},
                                        "component_samples": g_samples},
               "roofline_dft": {"kernel": "full-grid truncated DFT pipelines (y FFMA GEMMs + tcgen05 x / z stages)",
                                "bound": "fp32", "achieved": dft_tflops, "peak": fp32, "peak_kind": fp32_kind,
                                "unit": "TFLOP/s", "frac": dft_tflops / fp32, "traffic": None,
                                "flops_per_field": dft_flops_per_field(),
                                "calls_timed": d_n, "dft_share_of_step": d_ms / dft_step_ms if dft_step_ms else 0,
                                "measured_in": "one extra instrumented registration after the timed steps"},
               "fixed_work": fixed, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
               "clocks": clk.summary(),
               "result": {"stop": res.stop, "iterations": res.iterations, "final_energy": res.final_energy,
                          "hessvecs": res.hessvecs, "trials": res.trials, "forwards": res.forwards,
                          "mse_rel_final": res.history[-1].mse_rel if res.history else None,
                          "gn_per_step": [r.iterations for r in results]}}
        print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
