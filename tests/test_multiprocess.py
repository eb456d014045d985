"""Request-sharded multi-rank path on CPU (gloo, world_size 2).

Each rank runs the engine contract (virtual-clock backend here; the GPU
executor on the box) on its round-robin shard of one trace (`shard=r/N`, the
reference's multi_instance_split rule, schedulers.hpp:86-92) and the ranks
gather (makespan, wall, tokens) with one all_gather -- bench.py's
gather_run_stats, the same function the NCCL path uses."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist
import torch.multiprocessing as mp

SPEC = "n=24;input=32..96;output=2..9;seed=11;arrival=poisson:400;policy=mixed_batching;max_batch=6"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2505_03763_b200 as sw

    r = sw.sim_run(f"{SPEC};shard={rank}/{world}")
    ids = sorted(int(q_["id"]) for q_ in r.requests)
    res = {"makespan": r.report["makespan_s"], "wall": 0.0, "tokens": r.report["total_output_tokens"]}
    g = bench.gather_run_stats(dist, world, res, "cpu")
    all_ids = [None] * world
    dist.all_gather_object(all_ids, ids)
    q.put((rank, ids, res, g, all_ids))
    dist.destroy_process_group()


def test_two_rank_sharding_and_gather():
    import paper_2505_03763_b200 as sw

    full = sw.sim_run(SPEC)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    ids0, ids1 = out[0][1], out[1][1]
    assert set(ids0).isdisjoint(ids1)
    assert sorted(ids0 + ids1) == list(range(24))
    # round robin by arrival order: rank r gets arrival-order positions r, r+N, ...
    order = [int(q_["id"]) for q_ in sorted(full.requests, key=lambda x: (x["arrival_s"], x["id"]))]
    assert ids0 == sorted(order[0::2]) and ids1 == sorted(order[1::2])
    g = out[0][3]
    assert g["tokens"] == full.report["total_output_tokens"]
    assert g["makespan"] == max(out[0][2]["makespan"], out[1][2]["makespan"])
    assert out[0][3] == out[1][3]  # every rank sees the same gathered result
