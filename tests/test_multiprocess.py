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


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2505_03763_b200 as sw
    from paper_2505_03763_b200 import sharded

    r = sw.sim_run(f"{SPEC};shard={rank}/{world}")
    rows = sharded.request_rows(r)
    # fake token ids so the id payload is exercised (GPU runs carry the real greedy tokens)
    for row in rows:
        row["tokens"] = [row["id"] * 1000 + j for j in range(row["n_tokens"])]
        row["n_ids"] = row["n_tokens"]
    got, mk, wall = sharded.gather_requests(dist, world, rows, r.report["makespan_s"], 0.5 + rank, "cpu",
                                            max_requests=16, max_tokens=12)
    local = [None] * world
    dist.all_gather_object(local, rows)
    q.put((rank, got, mk, wall, local, r.report["makespan_s"]))
    dist.destroy_process_group()


def test_two_rank_request_gather_folds_like_one_process():
    """sharded.gather_requests (the product's one collective):
    every rank ends with every request's row and token ids, and the fold of
    the gathered rows equals the single-process fold of the union; the fold
    itself reproduces a run's own report percentiles (metrics.hpp:79-85)."""
    import paper_2505_03763_b200 as sw
    from paper_2505_03763_b200 import sharded

    full = sw.sim_run(SPEC)
    own = sharded.fold(sharded.request_rows(full), full.report["makespan_s"])
    for k in ("p50_ttft_s", "p99_ttft_s", "p50_tbt_s", "p99_tbt_s", "total_output_tokens"):
        assert own[k] == full.report[k], k
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    union = sorted(out[0][4][0] + out[0][4][1], key=lambda r: r["id"])
    for rank, got, mk, wall, _, _ in out:
        assert [r["id"] for r in got] == list(range(24))
        assert mk == max(o[5] for o in out) and wall == 1.5
        for g, u in zip(got, union):
            assert g["tokens"] == u["tokens"] and g["n_tokens"] == u["n_tokens"]
            assert g["ttft_s"] == u["ttft_s"] and g["tbt_mean_s"] == u["tbt_mean_s"] or (
                g["tbt_mean_s"] != g["tbt_mean_s"] and u["tbt_mean_s"] != u["tbt_mean_s"])
        assert sharded.fold(got, mk) == sharded.fold(union, mk)
    assert sharded.fold(out[0][1], 1.0)["total_output_tokens"] == full.report["total_output_tokens"]
