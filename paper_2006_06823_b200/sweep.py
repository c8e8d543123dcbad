"""Batched pairwise registration sweeps sharded over the GPUs of one node (config 5).

SURVEY.md §8e: a single registration stays on one GPU; a sweep over registration
pairs (all ordered pairs of S subjects) is embarrassingly parallel.  One process
per GPU (torchrun); each rank takes pairs from a work queue — a file-backed
atomic counter shared by the ranks of the node (dynamic balancing of pairs that
stop early), or static round-robin — and registers them with no communication
during the solves.  At the end the result records are gathered with two
collectives: the per-pair metadata (GN history, stop reason, Jacobian ranges;
all_gather_object) and the band velocities as one fixed-size tensor per rank
(all_gather; NCCL on the GPU box, gloo in the CPU tests) — the outputs the
reference CLI writes per registration (lddmm_cli.cpp:136-160: velocity, history,
Jacobian statistics).

--contexts-per-gpu C runs C engine contexts per GPU, each on its own CUDA stream
driven by its own host thread (the C ABI releases the GIL), pulling pairs from the
same queue: small registrations under-fill a B200, several in flight fill it.

    torchrun --nproc-per-node 8 -m paper_2006_06823_b200.sweep --subjects 16
"""
from __future__ import annotations

import argparse
import fcntl
import json
import os
import threading
import time
from dataclasses import asdict, dataclass, field


def pair_list(n_subjects):
    """All ordered pairs (source, target), source != target."""
    return [(i, j) for i in range(n_subjects) for j in range(n_subjects) if i != j]


def shard_round_robin(pairs, rank, world):
    return pairs[rank::world]


class WorkQueue:
    """Node-local atomic counter in a file (flock): next() hands out indices 0, 1, ...
    across processes until `total` is reached."""

    def __init__(self, path, total):
        self.path, self.total = path, total

    def reset(self):
        with open(self.path, "w") as f:
            f.write("0")

    def next(self):
        with open(self.path, "r+") as f:
            fcntl.flock(f, fcntl.LOCK_EX)
            try:
                f.seek(0)
                i = int(f.read().strip() or "0")
                if i >= self.total:
                    return None
                f.seek(0)
                f.truncate()
                f.write(str(i + 1))
                f.flush()
                return i
            finally:
                fcntl.flock(f, fcntl.LOCK_UN)


@dataclass
class PairResult:
    source: int
    target: int
    rank: int
    stop: str = ""
    iterations: int = 0
    hessvecs: int = 0
    final_energy: float = 0.0
    mse_rel_initial: float = 0.0
    mse_rel_final: float = 0.0
    vmax: float = 0.0
    seconds: float = 0.0
    context: int = 0
    # per GN iteration: iter, energy, energy_data, energy_reg, mse_rel, rel_grad, pcg_iters,
    # pcg_fallback, epsilon, cfl (IterationRecord, optimizer.hpp:50-61)
    history: list = field(default_factory=list)
    # compute_maps Jacobian determinant ranges: fwd min, fwd max, inv min, inv max
    jac: list = field(default_factory=list)


def run_pairs(next_pair, register, rank, context=0, velocities=None):
    """Drive `register(source, target) -> dict` over the pairs handed out by next_pair().
    A returned "velocity" entry (band coefficients) goes to `velocities[(s, t)]`."""
    out = []
    while True:
        p = next_pair()
        if p is None:
            break
        s, t = p
        t0 = time.perf_counter()
        info = dict(register(s, t))
        v = info.pop("velocity", None)
        if velocities is not None and v is not None:
            velocities[(s, t)] = v
        r = PairResult(s, t, rank, seconds=time.perf_counter() - t0, context=context, **info)
        out.append(r)
    return out


def run_pairs_threaded(next_pair, registers, rank, velocities=None):
    """Several engine contexts on one GPU: one host thread per context, all pulling from
    the same next_pair (serialised by a lock)."""
    lock = threading.Lock()

    def locked_next():
        with lock:
            return next_pair()

    results = [None] * len(registers)
    errors = []

    def work(k):
        try:
            results[k] = run_pairs(locked_next, registers[k], rank, context=k, velocities=velocities)
        except BaseException as exc:  # pragma: no cover - surfaced below
            errors.append(exc)

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(registers))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    return [r for lst in results for r in lst]


def gather_results(results, dist=None, velocities=None, device=None):
    """End of sweep, every rank gets every record.  Metadata: one all_gather_object.
    Velocities (fixed-size band vectors, complex128): one all_gather of a
    [max_pairs_per_rank, 2 * V] float64 tensor per rank (on `device` — CUDA for NCCL).
    Returns (records sorted by (source, target), velocities dict or None)."""
    import numpy as np
    recs = [asdict(r) if isinstance(r, PairResult) else r for r in results]
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        recs.sort(key=lambda r: (r["source"], r["target"]))
        return recs, (dict(velocities) if velocities is not None else None)
    allr = [None] * dist.get_world_size()
    dist.all_gather_object(allr, recs)
    merged = [r for lst in allr for r in lst]
    merged.sort(key=lambda r: (r["source"], r["target"]))
    if velocities is None:
        return merged, None
    import torch
    keys = [(r["source"], r["target"]) for r in recs]
    shape = next(iter(velocities.values())).shape if velocities else None
    shapes = [None] * dist.get_world_size()
    dist.all_gather_object(shapes, shape)
    shape = next(x for x in shapes if x is not None)
    V = int(np.prod(shape)) * 2
    counts = [len(lst) for lst in allr]
    cap = max(counts)
    buf = torch.zeros((cap, V), dtype=torch.float64)
    for k, key in enumerate(keys):
        buf[k] = torch.from_numpy(np.ascontiguousarray(velocities[key]).view(np.float64).ravel())
    buf = buf.to(device) if device is not None else buf
    outs = [torch.zeros_like(buf) for _ in range(dist.get_world_size())]
    dist.all_gather(outs, buf)
    vel = {}
    for rk, lst in enumerate(allr):
        o = outs[rk].cpu().numpy()
        for k, r in enumerate(lst):
            vel[(r["source"], r["target"])] = o[k].view(np.complex128).reshape(shape)
    return merged, vel


def make_register(dims, band, nt, sigma2, variant, opt_kwargs, device, with_maps=True, cache=None):
    """Registration callable on this rank's GPU: subjects generated on the host (phantoms),
    registered through the C ABI (lddmm_register, host buffers in / velocity out), then
    compute_maps for the Jacobian ranges (lddmm_maps)."""
    import numpy as np

    from . import lddmm as L
    from . import phantoms

    ctx = L.Context(L.BandSpec(L.GridSpec(dims), band), variant, nt, sigma2, device=device)
    cache = {} if cache is None else cache  # subjects, shareable between contexts

    def subject(k):
        if k not in cache:
            cache[k] = phantoms.subject(dims, k)
        return cache[k]

    opt = L.OptimizeOptions(**opt_kwargs)

    def prepare(ids):  # host-side subject synthesis, outside the timed sweep
        for k in ids:
            subject(k)

    def register(s, t):
        v, res = L.register_host(ctx, subject(s), subject(t), opt)
        jac = L.maps_jacobian(ctx, v) if with_maps else []
        hist = [[h.iter, h.energy, h.energy_data, h.energy_reg, h.mse_rel, h.rel_grad, h.pcg_iters,
                 int(h.pcg_fallback), h.epsilon, h.cfl] for h in res.history]
        return dict(stop=res.stop, iterations=res.iterations, hessvecs=res.hessvecs,
                    final_energy=res.final_energy, mse_rel_initial=res.history[0].mse_rel,
                    mse_rel_final=res.history[-1].mse_rel, vmax=float(np.abs(v).max()),
                    history=hist, jac=[float(x) for x in jac], velocity=v.copy())

    register.prepare = prepare
    return register


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--subjects", type=int, default=16)
    ap.add_argument("--pairs", type=int, default=0, help="limit the number of pairs (0 = all)")
    ap.add_argument("--dims", default="180,210,180")
    ap.add_argument("--band", type=int, default=32)
    ap.add_argument("--nt", type=int, default=10)
    ap.add_argument("--sigma2", type=float, default=0.01)
    ap.add_argument("--variant", default="deformation_state_equation")
    ap.add_argument("--max-iter", type=int, default=10)
    ap.add_argument("--queue", default="", help="work-queue file (dynamic balancing); empty = round robin")
    ap.add_argument("--contexts-per-gpu", type=int, default=1)
    ap.add_argument("--no-maps", action="store_true", help="skip compute_maps (Jacobian ranges)")
    ap.add_argument("--out", default="", help="JSON summary + per-pair records")
    ap.add_argument("--velocities", default="", help=".npz of the gathered band velocities (rank 0)")
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    if args.queue and local_world != world:
        raise SystemExit("--queue is a node-local file: use it with one node (WORLD_SIZE == LOCAL_WORLD_SIZE)")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the driver reads nranks / NVLS from the log
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dims = tuple(int(x) for x in args.dims.split(","))
    pairs = pair_list(args.subjects)
    if args.pairs:
        pairs = pairs[: args.pairs]
    subjects = {}
    registers = [make_register(dims, (args.band,) * 3, args.nt, args.sigma2, args.variant,
                               dict(max_iter=args.max_iter), local, with_maps=not args.no_maps, cache=subjects)
                 for _ in range(max(1, args.contexts_per_gpu))]
    if args.queue:
        q = WorkQueue(args.queue, len(pairs))
        if rank == 0:
            q.reset()
        if world > 1:
            dist.barrier()

        def next_pair():
            i = q.next()
            return None if i is None else pairs[i]
    else:
        mine = iter(shard_round_robin(pairs, rank, world))

        def next_pair():
            return next(mine, None)
    registers[0].prepare(sorted({k for p in pairs for k in p}))
    if world > 1:
        dist.barrier()
    vel = {}
    t0 = time.perf_counter()
    if len(registers) == 1:
        res = run_pairs(next_pair, registers[0], rank, velocities=vel)
    else:
        res = run_pairs_threaded(next_pair, registers, rank, velocities=vel)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    recs, vel = gather_results(res, dist if world > 1 else None, vel, device=torch.device("cuda", local))
    if world > 1:
        t = torch.tensor([wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    if rank == 0:
        summary = {"pairs": len(recs), "n_gpus": world, "contexts_per_gpu": len(registers), "wall_s": wall,
                   "registrations_per_hour": len(recs) / wall * 3600.0 if wall > 0 else 0.0}
        print(json.dumps(summary))
        if args.out:
            with open(args.out, "w") as f:
                json.dump({"summary": summary, "results": recs}, f)
        if args.velocities:
            np.savez_compressed(args.velocities, **{f"v_{s}_{t}": v for (s, t), v in sorted(vel.items())})
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
