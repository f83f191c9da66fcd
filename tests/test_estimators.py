"""Tree-size estimators, exact enumeration, dead-end rate and the decision-
order prune profile (the reference's tree_size.cpp is a
stub). CPU only: the reference space and closed-form trees."""
import json
import subprocess
import sys

import pytest

from paper_1904_03383_b200.api import DeadEnd, Space, enumerate_synthetic, estimate_synthetic

PAPER = "size,dim_kind,thread_level,mem_space,order,cache"
AXPY_1M = dict(kind="axpy", n=1 << 20, factors=[[2, 4], [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]])


def test_uniform_binary_tree_is_exact_for_both_estimators():
    """SPEC: binary depth 10 -> 1024 leaves, 2047 nodes; both estimators exact, CI width 0."""
    ex = enumerate_synthetic("uniform:2,10")
    assert (ex["leaves"], ex["nodes"]) == (1024, 2047)
    assert ex["nodes_per_depth"] == [2 ** d for d in range(11)]
    for method, it in (("knuth", 200), ("chen", 5)):
        e = estimate_synthetic("uniform:2,10", method, it, seed=7)
        assert e["leaves"] == 1024 and e["nodes"] == 2047 and e["leaves_stderr"] == 0


def test_single_node_tree():
    assert enumerate_synthetic("uniform:3,0")["leaves"] == 1
    for method in ("knuth", "chen"):
        assert estimate_synthetic("uniform:3,0", method, 10)["leaves"] == 1


def test_knuth_is_unbiased_on_random_trees():
    """SPEC: mean of 1e5-sample Knuth estimates within 2% of the exact count."""
    checked = 0
    for seed in range(1, 40):
        tree = f"random:{seed},4,8"
        exact = enumerate_synthetic(tree)["leaves"]
        if exact < 50:
            continue
        e = estimate_synthetic(tree, "knuth", 100000, seed=seed)
        assert abs(e["leaves"] - exact) <= 0.02 * exact + 4 * e["leaves_stderr"], (tree, exact, e)
        checked += 1
        if checked == 12:
            break
    assert checked >= 8


def test_chen_ci_covers_exact_count_on_random_trees():
    cover = total = 0
    for seed in range(1, 30):
        tree = f"random:{seed},4,8"
        exact = enumerate_synthetic(tree)["leaves"]
        if exact < 50:
            continue
        e = estimate_synthetic(tree, "chen", 2000, seed=seed)
        lo, hi = e["leaves_ci95"]
        cover += lo <= exact <= hi
        total += 1
    assert total >= 10 and cover >= 0.8 * total, (cover, total)


def test_chen_beats_knuth_on_the_caterpillar():
    """SPEC: a caterpillar-with-bushes tree where Knuth's CI after 1e5 descents
    is wider than Chen's after 1e3 runs (both against the exact count)."""
    tree = "caterpillar:24,10"
    exact = enumerate_synthetic(tree)["leaves"]
    assert exact == 24 + 2 ** 10
    k = estimate_synthetic(tree, "knuth", 100000, seed=3)
    c = estimate_synthetic(tree, "chen", 1000, seed=3)
    assert c["leaves"] == exact  # the (depth, remaining) strata separate spine, leaves and bush
    assert (k["leaves_ci95"][1] - k["leaves_ci95"][0]) > (c["leaves_ci95"][1] - c["leaves_ci95"][0])
    assert abs(k["leaves"] - exact) > 0.1 * exact  # Knuth almost never reaches the bush


def test_chen_rejects_a_stratifier_that_does_not_decrease():
    with pytest.raises(ValueError, match="strictly decreasing"):
        estimate_synthetic("uniform:2,5", "chen", 3, stratifier="constant")
    with pytest.raises(ValueError, match="strictly decreasing"):
        Space("outer_product", m=2, n=2).root().estimate("chen", 3, stratifier="constant")
    # the other stratifiers decrease along every edge of the reference tree
    for st in ("depth", "remaining", "depth_remaining"):
        assert Space("outer_product", m=2, n=2).root().estimate("chen", 3, stratifier=st)["leaves"] > 0


def test_estimators_on_the_reference_space():
    """outer_product(2,2) has 768 leaves (nest_test.cpp:318): Chen's strata make
    it exact, Knuth's CI covers it."""
    root = Space("outer_product", m=2, n=2).root()
    ex = root.enumerate()
    assert ex["leaves"] == 768 and ex["dead_ends"] == 0
    assert sum(ex["nodes_per_depth"]) == ex["nodes"]
    c = root.estimate("chen", 50, seed=1)
    assert c["leaves"] == 768 and c["nodes"] == ex["nodes"]
    k = root.estimate("knuth", 20000, seed=3)
    assert abs(k["leaves"] - 768) <= 4 * k["leaves_stderr"]
    # the older entry point is the same estimator
    old = root.estimate_tree(20000, seed=3)
    assert old["leaves"] == k["leaves"]


def test_chen_coverage_on_reference_subtrees():
    """SPEC: Chen's CI covers the exact count in >= 90% of repetitions, on
    enumerable subtrees of the matmul space."""
    root = Space("matmul", m=2, n=2, k=2).root()
    subtrees = []
    for seed in range(1, 8):
        try:
            c = root.descend(30, seed=seed)
            ex = c.enumerate(node_budget=20000)
        except (DeadEnd, ValueError):
            continue
        if ex["leaves"] > 100:
            subtrees.append((c, ex["leaves"]))
    assert subtrees
    cover = total = 0
    for c, exact in subtrees[:2]:
        for rep in range(50):
            e = c.estimate("chen", 10, seed=1000 + rep)
            lo, hi = e["leaves_ci95"]
            cover += lo - 1e-6 <= exact <= hi + 1e-6
            total += 1
    assert cover >= 0.9 * total, (cover, total)


def test_enumerate_refuses_oversized_spaces():
    with pytest.raises(ValueError, match="refused"):
        Space("matmul", m=2, n=2, k=2).root().enumerate(node_budget=1000)


def test_deadend_rate_and_wilson_interval():
    root = Space("outer_product", m=2, n=2).root()
    r = root.deadend_rate(1000, seed=1)
    assert r["dead_ends"] == 0 and r["ci95"][0] <= 1e-12 and r["ci95"][1] < 0.005
    assert root.deadend_exact() == 0.0
    m = Space("matmul", m=16, n=16, k=16, factors=[[2, 4], [2]]).root().deadend_rate(300, seed=1)
    lo, hi = m["ci95"]
    assert lo < m["ratio"] < hi and 0 < m["ratio"] < 0.5  # paper section 5.2: "inferior to a third" (directional)
    # the same seed walks the same descents
    assert Space("matmul", m=16, n=16, k=16, factors=[[2, 4], [2]]).root().deadend_rate(300, seed=1) == m


def test_order_compare_default_prunes_at_least_as_much_as_reversed():
    """SPEC: at the depths where both orders have >= 1e3 nodes, the paper's
    order prunes a fraction >= the reversed order's (paper section 5.4)."""
    space = Space(**AXPY_1M)
    root = space.root()
    leaf, b = root.greedy_leaf(PAPER)
    assert leaf.fully_specified and b > 0
    rev = ",".join(reversed(PAPER.split(",")))
    d = root.prune_profile(b * 1.25, 8, order=PAPER)
    r = root.prune_profile(b * 1.25, 8, order=rev)
    both = [i for i in range(8) if d["nodes"][i] >= 1000 and r["nodes"][i] >= 1000]
    assert both
    for i in both:
        assert d["fraction"][i] >= r["fraction"][i]
    assert d["fraction"][7] > 0.5  # most of depth 7 is prunable in the paper's order
    assert d["pruned"][0] == 0  # T is above the root's bound


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1904_03383_b200.cli", *args], capture_output=True, text=True,
                          timeout=300)


def test_cli_estimate_deadend_enumerate_order_compare():
    p = _cli("estimate", "outer_product", "--m", "2", "--n", "2", "--method", "both", "--probes", "2000",
             "--runs", "20")
    assert p.returncode == 0, p.stderr
    out = json.loads(p.stdout)
    assert out["chen"]["leaves"] == 768 and out["tighter"] == "chen"
    p = _cli("deadend", "outer_product", "--m", "2", "--n", "2", "--trials", "200")
    assert p.returncode == 0 and json.loads(p.stdout)["dead_ends"] == 0
    p = _cli("enumerate", "outer_product", "--m", "2", "--n", "2")
    assert p.returncode == 0 and json.loads(p.stdout)["leaves"] == 768
    p = _cli("enumerate", "matmul", "--m", "2", "--n", "2", "--k", "2", "--node-budget", "500")
    assert p.returncode == 2 and "refused" in p.stderr
    p = _cli("order-compare", "axpy", "--n", "1048576", "--factors", "2,4", "2,4,8,16,32,64,128,256,512,1024",
             "--depth", "8")
    assert p.returncode == 0, p.stderr
    out = json.loads(p.stdout)
    assert out["compared_depths"] and out["default_ge_reversed"]


def test_cli_exit_codes():
    assert _cli("deadend", "no_such_kind").returncode == 2
    assert _cli("no-such-command").returncode == 2
    # a factor list that does not divide the extent: the reference builder throws
    assert _cli("enumerate", "axpy", "--n", "100", "--factors", "3").returncode == 2
