"""Host-side logic of the multi-GPU pair sweep (config 5) on CPU:
sharding, the node-local work queue, and the single end-of-sweep gather over a
world_size-2 gloo process group (the GPU box uses NCCL for the same call)."""
import multiprocessing as mp
import os
import socket
import tempfile

import pytest

from paper_2006_06823_b200 import sweep


def test_pair_list_and_round_robin():
    pairs = sweep.pair_list(16)
    assert len(pairs) == 240 and len(set(pairs)) == 240 and all(s != t for s, t in pairs)
    for world in (1, 2, 4, 8):
        shards = [sweep.shard_round_robin(pairs, r, world) for r in range(world)]
        flat = [p for sh in shards for p in sh]
        assert sorted(flat) == sorted(pairs)
        assert max(map(len, shards)) - min(map(len, shards)) <= 1


def _drain(path, total, out):
    q = sweep.WorkQueue(path, total)
    got = []
    while True:
        i = q.next()
        if i is None:
            break
        got.append(i)
    out.put(got)


def test_work_queue_hands_out_each_index_once():
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "q")
        q = sweep.WorkQueue(path, 200)
        q.reset()
        ctx = mp.get_context("fork")
        out = ctx.Queue()
        procs = [ctx.Process(target=_drain, args=(path, 200, out)) for _ in range(4)]
        for p in procs:
            p.start()
        got = [out.get(timeout=60) for _ in procs]
        for p in procs:
            p.join(timeout=60)
        flat = sorted(i for g in got for i in g)
        assert flat == list(range(200))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, qpath, result_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pairs = sweep.pair_list(5)
    q = sweep.WorkQueue(qpath, len(pairs))
    if rank == 0:
        q.reset()
    dist.barrier()

    def next_pair():
        i = q.next()
        return None if i is None else pairs[i]

    def register(s, t):  # stand-in for the GPU registration: deterministic per pair
        return dict(stop="gradient", iterations=(s + t) % 4 + 1, hessvecs=0, final_energy=float(s * 10 + t),
                    mse_rel_initial=1.0, mse_rel_final=0.5, vmax=0.0)

    res = sweep.run_pairs(next_pair, register, rank)
    recs, _ = sweep.gather_results(res, dist)
    dist.destroy_process_group()
    result_q.put((rank, len(res), recs))


def test_gloo_two_ranks_gather_every_pair_once():
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        qpath = os.path.join(d, "queue")
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, qpath, result_q)) for r in range(2)]
        for p in procs:
            p.start()
        outs = [result_q.get(timeout=120) for _ in procs]
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    outs.sort()
    pairs = sweep.pair_list(5)
    assert outs[0][1] + outs[1][1] == len(pairs)  # the queue split the work
    for _, _, recs in outs:  # every rank holds the full gathered list
        assert [(r["source"], r["target"]) for r in recs] == sorted(pairs)
        assert all(r["final_energy"] == r["source"] * 10 + r["target"] for r in recs)
        assert {r["rank"] for r in recs} <= {0, 1}


def _velocity(s, t, shape=(1, 3, 6, 6, 4)):
    """Deterministic stand-in band velocity of pair (s, t) (complex128, reference layout)."""
    import numpy as np
    rng = np.random.default_rng(1000 * s + t)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _register_stub(s, t):
    return dict(stop="gradient", iterations=(s + t) % 3 + 1, hessvecs=2, final_energy=float(s * 10 + t),
                mse_rel_initial=1.0, mse_rel_final=0.5, vmax=0.0,
                history=[[0, 1.0, 1.0, 0.0, 1.0, 0.0, 0, 0, 0.0, 0.0], [1, 0.5, 0.4, 0.1, 0.5, 0.1, 2, 0, 1.0, 0.2]],
                jac=[0.5 + 0.01 * s, 1.5, 0.6, 1.4], velocity=_velocity(s, t))


def _worker4(rank, world, port, qpath, contexts, result_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pairs = sweep.pair_list(6)
    q = sweep.WorkQueue(qpath, len(pairs))
    if rank == 0:
        q.reset()
    dist.barrier()

    def next_pair():
        i = q.next()
        return None if i is None else pairs[i]

    vel = {}
    if contexts == 1:
        res = sweep.run_pairs(next_pair, _register_stub, rank, velocities=vel)
    else:
        res = sweep.run_pairs_threaded(next_pair, [_register_stub] * contexts, rank, velocities=vel)
    recs, allv = sweep.gather_results(res, dist, vel)
    dist.destroy_process_group()
    result_q.put((rank, len(res), recs, {k: v for k, v in allv.items()}))


@pytest.mark.parametrize("contexts", [1, 3])
def test_gloo_four_ranks_gather_velocities_bitwise(contexts):
    """World size 4 (CPU gloo): the end-of-sweep gather hands every rank every pair's
    record and its band velocity, bit for bit what the single-pair registration returned
    (here a deterministic stand-in for the GPU registration); with several contexts per
    rank the threads split the queue without duplicates."""
    import numpy as np
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    world = 4
    with tempfile.TemporaryDirectory() as d:
        qpath = os.path.join(d, "queue")
        port = _free_port()
        procs = [ctx.Process(target=_worker4, args=(r, world, port, qpath, contexts, result_q)) for r in range(world)]
        for p in procs:
            p.start()
        outs = [result_q.get(timeout=180) for _ in procs]
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    pairs = sweep.pair_list(6)
    assert sum(o[1] for o in outs) == len(pairs)
    for _, _, recs, allv in outs:
        assert [(r["source"], r["target"]) for r in recs] == sorted(pairs)
        assert sorted(allv) == sorted(pairs)
        for (s, t), v in allv.items():
            assert np.array_equal(v, _velocity(s, t))
        for r in recs:
            assert r["jac"][0] == 0.5 + 0.01 * r["source"] and len(r["history"]) == 2
            if contexts > 1:
                assert 0 <= r["context"] < contexts
