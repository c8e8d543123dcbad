"""Batched pairwise registration sweeps sharded over the GPUs of one node (config 5).

SURVEY.md §8e: a single registration stays on one GPU; a sweep over registration
pairs (all ordered pairs of S subjects) is embarrassingly parallel.  One process
per GPU (torchrun); each rank takes pairs from a work queue — a file-backed
atomic counter shared by the ranks of the node (dynamic balancing of pairs that
stop early), or static round-robin — and registers them with no communication
during the solves.  At the end the fixed-size result records are gathered on
rank 0 with one collective (torch.distributed all_gather_object: NCCL on the
GPU box, gloo in the CPU tests).

    torchrun --nproc-per-node 8 -m paper_2006_06823_b200.sweep --subjects 16
"""
from __future__ import annotations

import argparse
import fcntl
import json
import os
import time
from dataclasses import asdict, dataclass


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


def run_pairs(next_pair, register, rank):
    """Drive `register(source, target) -> dict` over the pairs handed out by next_pair()."""
    out = []
    while True:
        p = next_pair()
        if p is None:
            break
        s, t = p
        t0 = time.perf_counter()
        info = register(s, t)
        r = PairResult(s, t, rank, seconds=time.perf_counter() - t0, **info)
        out.append(r)
    return out


def gather_results(results, dist=None):
    """One collective at the end: every rank's list of PairResult dicts -> rank 0 (all ranks get it)."""
    recs = [asdict(r) if isinstance(r, PairResult) else r for r in results]
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return recs
    allr = [None] * dist.get_world_size()
    dist.all_gather_object(allr, recs)
    merged = [r for lst in allr for r in lst]
    merged.sort(key=lambda r: (r["source"], r["target"]))
    return merged


def make_register(dims, band, nt, sigma2, variant, opt_kwargs, device):
    """Registration callable on this rank's GPU: subjects generated on the host (phantoms),
    registered through the C ABI (lddmm_register, host buffers in / velocity out)."""
    import numpy as np

    from . import lddmm as L
    from . import phantoms

    ctx = L.Context(L.BandSpec(L.GridSpec(dims), band), variant, nt, sigma2, device=device)
    cache = {}

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
        return dict(stop=res.stop, iterations=res.iterations, hessvecs=res.hessvecs,
                    final_energy=res.final_energy, mse_rel_initial=res.history[0].mse_rel,
                    mse_rel_final=res.history[-1].mse_rel, vmax=float(np.abs(v).max()))

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
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dims = tuple(int(x) for x in args.dims.split(","))
    pairs = pair_list(args.subjects)
    if args.pairs:
        pairs = pairs[: args.pairs]
    register = make_register(dims, (args.band,) * 3, args.nt, args.sigma2, args.variant,
                             dict(max_iter=args.max_iter), local)
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
    register.prepare(sorted({k for p in pairs for k in p}))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    res = run_pairs(next_pair, register, rank)
    wall = time.perf_counter() - t0
    recs = gather_results(res, dist if world > 1 else None)
    if world > 1:
        t = torch.tensor([wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    if rank == 0:
        summary = {"pairs": len(recs), "n_gpus": world, "wall_s": wall,
                   "registrations_per_hour": len(recs) / wall * 3600.0 if wall > 0 else 0.0}
        print(json.dumps(summary))
        if args.out:
            with open(args.out, "w") as f:
                json.dump({"summary": summary, "results": recs}, f)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
