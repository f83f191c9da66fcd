"""Deterministic TAG-MCTS and the seeded uniform walk of the
reference's CPU baseline. CPU only."""
import json
import os
import random
import subprocess

import pytest

from paper_1904_03383_b200.api import Space, explore_spec, tag_select

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_CPU_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_cpu_bench")
PAPER = "size,dim_kind,thread_level,mem_space,order,cache"


def test_tag_rule_examples():
    """SPEC: two children s=(5,0), t=(10,10) -> child 0; an excluded (pruned)
    child is never selected; unvisited children first; all excluded -> -1."""
    assert tag_select([5, 0], [10, 10], 20) == 0
    assert tag_select([5, 0], [10, 10], 20, excluded=[True, False]) == 1
    assert tag_select([9, 9, 0], [10, 10, 0], 20) == 2
    assert tag_select([1, 1], [1, 1], 2, excluded=[True, True]) == -1
    assert tag_select([3, 3], [5, 5], 10) == 0  # ties: lowest index


def test_tag_concentrates_on_the_better_arm():
    """SPEC: on a 2-armed synthetic bandit (10^4 rollouts) the selection
    frequencies concentrate on the better arm. Arm 0 draws costs from
    U[1, 2), arm 1 from U[1.5, 2.5); s_i counts an arm's costs in the global
    best-20 set."""
    rng = random.Random(5)
    costs = [[], []]
    pulls = [0, 0]
    best = []
    for n in range(10000):
        thr = best[-1] if len(best) >= 20 else float("inf")
        s = [sum(1 for c in costs[i] if c <= thr) for i in range(2)]
        i = tag_select(s, [float(p) for p in pulls], n)
        c = rng.uniform(1.0, 2.0) if i == 0 else rng.uniform(1.5, 2.5)
        costs[i].append(c)
        pulls[i] += 1
        best = sorted(best + [c])[:20]
    # once the top-20 set holds only arm-0 costs, s = (20, 0) and the rule's
    # steady state gives t0 / t1 = (20 + a + sqrt(40 a + a^2)) / (2 a) ~ 2.2
    # at a = ln(2 N k / delta) ~ 13.6: about 69% of the pulls
    assert pulls[0] > 0.65 * sum(pulls), pulls


def test_same_seed_gives_a_byte_identical_log(tmp_path):
    space = Space("outer_product", m=4096, n=4096)
    a, b = tmp_path / "a.jsonl", tmp_path / "b.jsonl"
    ra = explore_spec(space, 200, seed=11, log_path=str(a))
    rb = explore_spec(space, 200, seed=11, log_path=str(b))
    assert a.read_bytes() == b.read_bytes()
    assert ra["best_digest"] == rb["best_digest"] and ra["evaluations"] == rb["evaluations"]
    rows = [json.loads(x) for x in a.read_text().splitlines()]
    assert len(rows) == ra["rollouts"]
    # every record: seed, path, cost or DEADEND, the bounds of every node on the path
    for r in rows:
        assert r["seed"] == 11 and len(r["ancestor_bounds"]) == len(r["path"]) + 1
        assert r["cost"] in ("DEADEND", "PRUNED") or r["cost"] >= max(r["ancestor_bounds"]) * (1 - 1e-9)
    # best cost non-increasing over the log
    bests = [r["best"] for r in rows]
    assert all(x >= y for x, y in zip(bests, bests[1:]))


@pytest.mark.parametrize("kw", [dict(m=4096, n=4096), dict(m=1024, n=64)])
def test_pruning_safety(kw):
    """SPEC: with an exhaustive budget the best cost with bound pruning equals
    the best cost without it (admissibility: no optimum pruned)."""
    space = Space("outer_product", **kw)
    on = explore_spec(space, 10 ** 6, seed=1, pruning=True)
    off = explore_spec(space, 10 ** 6, seed=1, pruning=False)
    assert on["exhausted"] and off["exhausted"]
    assert off["evaluations"] == space.root().count_leaves() == 768
    assert on["best_cost"] == off["best_cost"] and on["best_digest"] == off["best_digest"]
    assert on["evaluations"] < off["evaluations"]  # pruning removed part of the space


def test_zero_budget_finds_no_implementation():
    r = explore_spec(Space("outer_product", m=2, n=2), 0, seed=1)
    assert r["best"] is None and r["evaluations"] == 0


def test_simulate_evaluator_returns_the_reference_cost():
    space = Space("outer_product", m=2, n=2)
    r = explore_spec(space, 40, seed=3, evaluator="simulate")
    assert r["evaluations"] == 40
    assert r["best"] is not None and r["best"].simulate()["total"] == r["best_cost"]


def test_ordered_search_on_axpy_reaches_a_finite_leaf():
    space = Space("axpy", n=1 << 16, factors=[[2, 4], [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]])
    r = explore_spec(space, 20, seed=2, order=PAPER, max_rollouts=400)
    assert r["best"] is not None and r["best_cost"] < float("inf")
    assert r["best"].bound()["total"] <= r["best_cost"]


@pytest.mark.skipif(not os.path.exists(REF_CPU_BENCH), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("kind,args,factors", [
    ("axpy", ["0", str(1 << 20), "0"], ["2,4", "2,4,8,16,32,64,128,256,512,1024"]),
    ("matmul", ["256", "256", "32"], ["2,4,8,16,32", "2,4"]),
])
def test_uniform_walk_equals_the_reference_cpu_bench(kind, args, factors):
    """The seeded uniform first-open descents our evaluator runs in the bench's
    uniform-walk mode are the reference baseline's (oracle/ref_cpu_bench.cpp
    thread 0): same leaves, same dead ends, same order."""
    env = dict(os.environ, REF_DUMP_WALKS="24")
    p = subprocess.run([REF_CPU_BENCH, kind, *args, "1", "1", *factors], capture_output=True, text=True, env=env,
                       timeout=300)
    assert p.returncode == 0, p.stderr
    ref = [int(x) for x in json.loads(p.stdout)["digests"]]
    kw = dict(n=int(args[1])) if kind == "axpy" else dict(m=int(args[0]), n=int(args[1]), k=int(args[2]))
    space = Space(kind, factors=[[int(v) for v in f.split(",")] for f in factors], **kw)
    ours = space.root().walk_digests(0x190403383, 24)
    assert ours == ref
    assert any(d == 0 for d in ref) and any(d != 0 for d in ref)  # both leaves and dead ends compared


def test_checkpoint_resume_by_replay(tmp_path):
    """SPEC.md:509 checkpoint/resume: the log of a run is its checkpoint. A run
    resumed from it re-derives every logged record (refusing a log that does
    not replay) and continues; the result equals one uninterrupted run."""
    space = Space("outer_product", m=4096, n=4096)
    a, b, c = (tmp_path / f"{x}.jsonl" for x in "abc")
    first = explore_spec(space, 60, seed=3, log_path=str(a))
    resumed = explore_spec(space, 150, seed=3, log_path=str(b), resume_log=str(a))
    fresh = explore_spec(space, 150, seed=3, log_path=str(c))
    assert resumed["replayed"] == first["rollouts"] > 0
    assert b.read_bytes() == c.read_bytes()
    assert resumed["best_digest"] == fresh["best_digest"] and resumed["evaluations"] == fresh["evaluations"]
    lines = a.read_text().splitlines()
    lines[5] = lines[5].replace('"seed": 3', '"seed": 4')
    bad = tmp_path / "bad.jsonl"
    bad.write_text("\n".join(lines) + "\n")
    with pytest.raises(ValueError, match="record 6"):
        explore_spec(space, 150, seed=3, resume_log=str(bad))
