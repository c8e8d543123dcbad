#!/usr/bin/env python
"""Benchmark: seconds per registration of the band-limited SL-RK2 GN-Krylov
deformation-state LDDMM path (BASELINE.json metric) on B200.

A step is one full registration of a synthetic 180x210x180 brain-like pair
(BASELINE.json configs[1]: band 32^3, nt=10, deformation-state variant,
stationary velocity, sigma2 = 0.01) with the reference's OptimizeOptions defaults
and max_iter = 10, pcg_max_iter = 5 (the paper's budget),
images resident in HBM when the step starts.
The per-registration image constants (I0 spline coefficients, spectral
gradient) are inside the step.  L2 is flushed (512 MiB write) between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): every rank registers its own pair (config 5
style sharding, no collective in the data path); the per-rank step times are
gathered with one NCCL all_gather at the end and the max over ranks is used.

--impl reference times the reference CPU implementation (oracle/_ref, the
unmodified reference headers compiled with our FFTW3-API shim) on this host:
one full-grid FFT, one prefilter and one cubic gather at the same grid,
extrapolated with the reference's own op counts for the same fixed-work
registration (oracle/ref.py:defstate_op_counts).
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


def cpu_reference_cost(threads=1, dims=DIMS, band=BAND, nt=NT, measured=None, source="our run"):
    """Reference CPU s/registration for the same workload (see module doc).  measured =
    (forwards, hessvecs, trials) of our run gives the identical operation sequence;
    without it the nominal budget GN x PCG x 1 trial is used."""
    from oracle import ref
    ref.set_threads(threads)
    t0 = time.time()
    times = ref.time_ops(dims, (1.0, 1.0, 1.0), band, mask=0b0111)
    sample_s = time.time() - t0
    if measured is not None:
        counts = ref.defstate_op_counts_measured(nt, *measured)
        how = (f"the measured op sequence of {source} ({measured[0]} forwards+gradients, {measured[1]} hessvecs, "
               f"{measured[2]} trials)")
    else:
        counts = ref.defstate_op_counts(nt, GN, PCG, 1)
        how = f"the nominal budget {GN} GN x {PCG} PCG x 1 trial"
    ms = ref.registration_cost_ms(times, counts)
    sample = (f"reference primitives timed at {dims[0]}x{dims[1]}x{dims[2]}: 1 full-grid complex FFT "
              f"{times['fft']:.0f} ms, 1 spline prefilter {times['prefilter']:.0f} ms, 1 cubic gather "
              f"{times['gather']:.0f} ms ({sample_s:.1f} s of CPU work); extrapolated with the reference op "
              f"counts of {how} at nt={nt}: {counts['fft']} FFTs, {counts['warp']} "
              f"warps, {counts['pre']} prefilters, {counts['gath']} gathers (band-space ops not counted). "
              f"FFT = FFTW3-API shim (libfftw3 absent), {threads} thread(s)")
    return ms / 1000.0, sample


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
    threads = os.cpu_count() or 1
    measured = reference_op_sequence()
    vals = []
    sample = ""
    for _ in range(max(1, args.steps)):
        v, sample = cpu_reference_cost(threads, measured=measured,
                                       source="the reference's own config-2 run (tests/golden/config2_ref.npz)")
        vals.append(v)
    value = float(np.mean(vals))
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s/registration", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1000.0, "higher_is_better": False,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload(),
           "cpu_baseline": {"value": value, "unit": "s/registration", "cores": threads, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": value, "unit": "s/registration", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def ncu_traffic():
    """DRAM bytes of one captured gather launch (profiles/r1_ncu_traffic.json, from
    `ncu --set full`), next to that launch's algorithmic bytes N (12 + 8 F)."""
    path = os.path.join(ROOT, "profiles", "r1_ncu_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return {"traffic": t["dram_bytes"], "traffic_launch_algorithmic_bytes": t["algorithmic_bytes"],
                "traffic_source": "profiles/r1_ncu_traffic.json (" + t["kernel"] + ", one launch)"}
    except (OSError, KeyError, ValueError):
        return {"traffic": None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

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
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2006_06823_b200 import lddmm as L
    from paper_2006_06823_b200 import phantoms

    seed = 2006 + rank
    I0, I1 = phantoms.brain_pair(DIMS, seed=seed)
    d0 = torch.from_numpy(I0).to(device=f"cuda:{local}", dtype=torch.float32)
    d1 = torch.from_numpy(I1).to(device=f"cuda:{local}", dtype=torch.float32)
    band = L.BandSpec(L.GridSpec(DIMS), BAND)
    model = L.Model(band, d0, d1, "deformation_state_equation", NT, SIGMA2, device=local)
    ctx = model.ctx
    opt = L.OptimizeOptions(max_iter=GN, pcg_max_iter=PCG)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=f"cuda:{local}")
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def one_registration():
        model.set_images(d0, d1)
        return L.optimize(model, None, opt)

    for _ in range(args.warmup):
        res = one_registration()
    torch.cuda.synchronize()

    step_ms = []
    launches0 = L.launch_count()
    ctx.gather_timing(True)
    with Clocks(local) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = one_registration()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    g_ms, g_n, g_bytes = ctx.gather_stats()
    ctx.gather_timing(False)
    launches = L.launch_count() - launches0

    total_ms = float(np.sum(step_ms))
    if dist is not None:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        total_ms = max(float(x.item()) for x in allt)
    value = total_ms / 1000.0 / (world * args.steps)
    hbm, peak_kind = peaks()
    achieved = (g_bytes / g_n) / (g_ms / g_n * 1e-3) / 1e9 if g_n else 0.0

    e2e = None
    if not args.no_e2e:
        ectx = L.Context(band, "deformation_state_equation", NT, SIGMA2, device=local)
        # inputs and the result velocity in pinned host memory (the reference's fp64
        # ScalarField / BandVectorField layouts); W untimed warm-up calls first
        # the same fp32-representable images the device arm registers (so both arms do
        # the same GN work), held as the reference's fp64 host fields
        h0 = torch.from_numpy(I0.astype(np.float32).astype(np.float64)).pin_memory().numpy()
        h1 = torch.from_numpy(I1.astype(np.float32).astype(np.float64)).pin_memory().numpy()
        v_host = torch.zeros(ectx.vel_shape + (2,), dtype=torch.float64).pin_memory().numpy().view(np.complex128)
        v_host = v_host.reshape(ectx.vel_shape)
        for _ in range(max(1, args.warmup)):
            L.register_host(ectx, h0, h1, opt, v_out=v_host)
        e_ms = []
        for k in range(max(1, args.steps)):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            v_host, r2 = L.register_host(ectx, h0, h1, opt, v_out=v_host)
            e_ms.append((time.perf_counter() - t0) * 1000.0)
        e2e_ms = float(np.sum(e_ms))
        if dist is not None:
            t = torch.tensor([e2e_ms], device=f"cuda:{local}", dtype=torch.float64)
            allt = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(allt, t)
            e2e_ms = max(float(x.item()) for x in allt)
        e2e = {"value": e2e_ms / 1000.0 / (world * len(e_ms)), "unit": "s/registration",
               "h2d_bytes_per_step": int(2 * I0.size * 8), "d2h_bytes_per_step": int(v_host.nbytes),
               "path": "lddmm_register (C ABI): pinned host fp64 images in, pinned host fp64 velocity out",
               "result": {"iterations": r2.iterations, "hessvecs": r2.hessvecs, "trials": r2.trials,
                          "forwards": r2.forwards, "final_energy": r2.final_energy}}
        del ectx

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            if ref.available():
                v, sample = cpu_reference_cost(1, measured=(res.forwards, res.hessvecs, res.trials))
                cpu = {"value": v, "unit": "s/registration", "cores": 1, "kind": "reference", "sample": sample}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unavailable": str(exc)}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "s/registration", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": False,
               "scaling": "weak", "vs_baseline": None, "dtype": "f32 grid / f64 band", "data": "synthetic",
               "config": workload(),
               "roofline": {"kernel": "gather_march_kernel (SL cubic gather)", "bound": "hbm",
                            "achieved": achieved, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                            "frac": achieved / hbm, **ncu_traffic(),
                            "algorithmic_bytes_per_launch": g_bytes / g_n if g_n else 0,
                            "launches_timed": g_n, "gather_share_of_step": g_ms / total_ms if total_ms else 0},
               "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
               "result": {"stop": res.stop, "iterations": res.iterations, "final_energy": res.final_energy,
                          "hessvecs": res.hessvecs, "trials": res.trials, "forwards": res.forwards,
                          "mse_rel_final": res.history[-1].mse_rel if res.history else None}}
        print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
