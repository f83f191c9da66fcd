"""The N > 1 path on CPU: world-size-2 gloo process group, one search shard
per rank (device=-1: rollouts, emission and NVRTC run, no device). Shards own
disjoint subtrees of the same deterministic frontier, and the incumbent cell
in POSIX shared memory is seen by every rank (no collective on the data
path; gloo only carries the test's own checks)."""
import os
import uuid

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.conftest import ROOT


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, shm, kind, kw, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1904_03383_b200 import Search, Space
        space = Space(kind, **kw)
        s = Search(space, device=-1, seed=7, shard_index=rank, shard_count=world, incumbent_shm=shm,
                   rollout_threads=1, compile_threads=1)
        mine = s.frontier()
        every = [None] * world
        dist.all_gather_object(every, mine)
        dist.barrier()
        if rank == 0:
            s.offer(12345.0)
        dist.barrier()
        seen = s.stats()["incumbent_ns"]
        dist.barrier()
        if rank == 1:
            s.offer(99999.0)  # worse: must not replace
            s.offer(777.0)    # better: must replace for everyone
        dist.barrier()
        after = s.stats()["incumbent_ns"]
        s.close()
        q.put((rank, every, seen, after))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,kw", [
    ("axpy", dict(n=1 << 20, factors=[[2, 4], [32, 64, 128, 256]])),
    ("sgemm", dict(m=256, n=256, k=64)),
])
def test_two_rank_shards_and_shared_incumbent(kind, kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    shm = f"/ispc_test_{uuid.uuid4().hex[:12]}"
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shm, kind, kw, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    every = res[0][1]
    a, b = set(every[0]), set(every[1])
    assert a and b and not (a & b), "shards must own disjoint subtrees"
    assert every == res[1][1]
    for _, _, seen, after in res:
        assert seen == pytest.approx(12345.0)
        assert after == pytest.approx(777.0)
    try:
        os.unlink("/dev/shm" + shm)
    except OSError:
        pass


def _best_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        mine = [(500.0, "slow", 88.0, 3.0), (117.0, "fast", 88.0, 4.5)][rank]
        q.put((rank, bench.best_over_ranks(world, *mine)))
    finally:
        dist.destroy_process_group()


def test_bench_reports_the_best_kernel_over_ranks():
    """bench.py's JSON line describes the fastest kernel any shard measured,
    whichever rank holds its candidate."""
    port = 29000 + (uuid.uuid4().int % 2000)
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_best_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    got = dict(q.get() for _ in range(2))
    assert got[0] == got[1] == (117.0, "fast", 88.0, 4.5)



def _steal_worker(rank, world, port, q, logdir):
    import json
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1904_03383_b200 import Search, Space
        space = Space("outer_product", m=4096, n=4096)
        log = os.path.join(logdir, f"r{rank}.jsonl")
        # device -2: the host pipeline alone (rollouts, emission; no NVRTC, no device)
        s = Search(space, device=-2, seed=7 + rank, shard_index=rank, shard_count=world, rollout_threads=1,
                   compile_threads=1, log_path=log)
        mine = s.frontier()
        s.step(100000, max_seconds=60)  # runs until every shard is spent (own subtrees, then stolen ones)
        st = s.stats()
        s.close()
        rows = [json.loads(x) for x in open(log)]
        q.put((rank, mine, st["frontier"], st["frontier_total"], st["stealing_since"], st["exhausted"],
               sorted({r["subtree"] for r in rows}), sorted({r["digest"] for r in rows})))
    finally:
        dist.destroy_process_group()


def test_four_rank_frontier_partition_and_stealing(tmp_path):
    """World 4 (gloo): the four shards partition one frontier (disjoint,
    union = the whole frontier); once a shard's own subtrees are spent it
    steals, producing leaves from other shards' subtrees; and the leaves the
    ranks produce together include every leaf any single rank found."""
    world = 4
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_steal_worker, args=(r, world, port, q, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = res[0][3]
    sets = [set(r[1]) for r in res]
    assert all(r[3] == total for r in res)
    assert sum(r[2] for r in res) == total == len(set().union(*sets))
    for i in range(world):
        for j in range(i + 1, world):
            assert not (sets[i] & sets[j]), "shards own disjoint subtrees"
    for rank, _, _, _, stealing_since, exhausted, subtrees, _ in res:
        assert exhausted == 1 and stealing_since >= 0, rank  # every spent shard turned to stealing
    # a steal can come up empty when the other shards drain their last
    # subtrees first (timing), but some shard produced leaves from another's
    assert any(any(t % world != rank for t in subtrees) for rank, *_, subtrees, _ in res), "nobody stole"
    union = set().union(*(set(r[7]) for r in res))
    assert all(set(r[7]) <= union for r in res) and len(union) >= max(len(r[7]) for r in res)
