"""Command line over the evaluation path (the reference's CLI is a stub,
proj/tools/src/main.cpp:1; its commands are specified at SPEC.md:569-604).

  python -m paper_1904_03383_b200.cli explore  axpy --n 1048576 --factors 2,4 32,64,128 --evals 64 --log run.jsonl
  python -m paper_1904_03383_b200.cli explore  gemv --m 4096 --n 4096 --evals 128
  python -m paper_1904_03383_b200.cli codegen  sgemm --m 1024 --n 1024 --k 1024 [--candidate c.json] [--seed 3]
  python -m paper_1904_03383_b200.cli bound    matmul --m 64 --n 64 --k 64 --factors 2,4 [--candidate c.json]
  python -m paper_1904_03383_b200.cli replay   run.jsonl axpy --n 1048576 --factors 2,4 32,64,128
  python -m paper_1904_03383_b200.cli estimate matmul --m 256 --n 256 --k 32 --factors 2,4,8,16,32 2,4 --method both
  python -m paper_1904_03383_b200.cli deadend  matmul --m 256 --n 256 --k 32 --factors 2,4,8,16,32 2,4 --trials 2000
  python -m paper_1904_03383_b200.cli order-compare axpy --n 1048576 --factors 2,4 2,4,8,16,32,64,128,256,512,1024
  python -m paper_1904_03383_b200.cli enumerate outer_product --m 2 --n 2

`codegen`, `bound`, `estimate`, `deadend`, `order-compare` and `enumerate`
need no GPU (Table 2's dead-end column with a Wilson CI,
section 5.3's estimators with the tighter CI flagged, section 5.4's prune
fractions per depth for the default against the reversed decision order).
Exit codes: 0 success, 2 configuration error, 3 no implementation found. `explore` and `replay` run on cuda device
`--device`. A candidate file holds the reference's text serialization
(Candidate.serialize(), candidate.cpp:445-634); `explore --log` writes the
JSONL evaluation log whose improving lines carry that serialization, and
`replay` re-measures them.
"""
from __future__ import annotations

import argparse
import json
import time
import sys

from .api import DeadEnd, EmitError, Search, Space, tile_cuda


def _space(a) -> Space:
    factors = [[int(v) for v in f.split(",")] for f in (a.factors or [])]
    return Space(a.kind, m=a.m, n=a.n, k=a.k, batch=a.batch, a_stride=a.a_stride, factors=factors)


def _candidate(space: Space, a):
    if a.candidate:
        return space.deserialize(open(a.candidate).read())
    leaf, _, _ = space.root().random_leaf(a.seed)
    return leaf


def cmd_explore(a) -> int:
    space = _space(a)
    s = Search(space, device=a.device, seed=a.seed, log_path=a.log, flush_l2=a.kind in ("gemv", "batched"),
               decision_order=a.decision_order, tree_depth=a.tree_depth)
    t0 = time.perf_counter()
    s.step(a.evals)
    wall = time.perf_counter() - t0
    st = s.stats()
    best = s.best()
    if best is None:
        print(json.dumps({"evaluations": st["evaluations"], "status": "no implementation found"}))
        s.close()
        return 3
    out = {"evaluations": st["evaluations"], "ok": st["ok"], "best_us": st["best_ns"] / 1e3,
           "bound_us": st["best_bound_ns"] / 1e3, "time_to_best_s": st["time_to_best_s"],
           "bound_violations": st["bound_violations"], "exhausted": bool(st["exhausted"]),
           "evals_per_s": round(st["evaluations"] / max(wall, 1e-9), 1), "dead_rollouts": st["dead_rollouts"],
           "rollouts": st["rollouts"]}
    if best is not None and space.tiles:
        out["config"] = best.tiles().as_dict()
    print(json.dumps(out))
    if a.out and best is not None:
        open(a.out, "w").write(best.serialize())
    s.close()
    return 0


def cmd_codegen(a) -> int:
    """Source of the given candidate, or of the first runnable random leaf
    from --seed on (the space admits leaves a B200 cannot run)."""
    space = _space(a)
    last = None
    for attempt in range(1 if a.candidate else 100):
        a2 = argparse.Namespace(**{**vars(a), "seed": a.seed + attempt})
        try:
            c = _candidate(space, a2)
            src, _ = tile_cuda(c.tiles()) if space.tiles else c.nest().cuda()
        except (EmitError, DeadEnd) as e:
            last = e
            continue
        sys.stdout.write(src)
        return 0
    print(f"no runnable leaf: {last}", file=sys.stderr)
    return 3


def cmd_bound(a) -> int:
    space = _space(a)
    c = space.root() if a.root else _candidate(space, a)
    print(json.dumps(c.bound(l2_flushed=a.l2_flushed)))
    return 0


def cmd_estimate(a) -> int:
    """Knuth's and/or Chen's estimate of the space size (the reference's
    tree_size is a stub); with --method both the tighter CI is flagged (the
    paper kept "whichever gave a better confidence interval", section 5.3)."""
    space = _space(a)
    root = space.root()
    methods = ["knuth", "chen"] if a.method == "both" else [a.method]
    out = {}
    for m in methods:
        it = a.probes if m == "knuth" else a.runs
        out[m] = root.estimate(m, it, seed=a.seed, order=a.order, stratifier=a.stratifier)
    if len(out) > 1:
        rel = {m: e["leaves_stderr"] / e["leaves"] if e["leaves"] else float("inf") for m, e in out.items()}
        out["tighter"] = min(rel, key=rel.get)
    print(json.dumps(out if len(out) > 1 else out[methods[0]]))
    return 0


PAPER_ORDER = "size,dim_kind,thread_level,mem_space,order,cache"


def cmd_deadend(a) -> int:
    """Probability that a uniform random descent ends at a dead end (paper
    section 5.2, Table 2), with its 95% Wilson interval."""
    space = _space(a)
    r = space.root().deadend_rate(a.trials, seed=a.seed, order=a.order)
    print(json.dumps(r))
    return 0


def cmd_order_compare(a) -> int:
    """Share of the nodes of each of the first levels whose B200 bound is >=
    the incumbent T, for the paper's decision order and its reverse (paper
    section 5.4). T: --T-us, else the lowest-bound leaf's bound x --slack."""
    space = _space(a)
    root = space.root()
    orders = {"default": a.order or PAPER_ORDER}
    orders["reversed"] = ",".join(reversed(orders["default"].split(",")))
    if a.T_us:
        T = a.T_us * 1e-6
    else:
        try:
            _, b = root.greedy_leaf(orders["default"])
        except DeadEnd:
            print("no implementation found (no leaf with a finite bound)", file=sys.stderr)
            return 3
        T = b * a.slack
    out = {"T_us": T * 1e6, "depth_cap": a.depth, "min_nodes": a.min_nodes}
    for name, o in orders.items():
        out[name] = dict(order=o, **root.prune_profile(T, a.depth, order=o, node_budget=a.node_budget))
    both = [d for d in range(a.depth) if out["default"]["nodes"][d] >= a.min_nodes
            and out["reversed"]["nodes"][d] >= a.min_nodes]
    out["compared_depths"] = both
    out["default_ge_reversed"] = all(out["default"]["fraction"][d] >= out["reversed"]["fraction"][d] for d in both)
    print(json.dumps(out))
    return 0


def cmd_enumerate(a) -> int:
    """Exact node / leaf / dead-end counts (refuses past --node-budget nodes)."""
    space = _space(a)
    print(json.dumps(space.root().enumerate(node_budget=a.node_budget, order=a.order)))
    return 0


def cmd_replay(a) -> int:
    from .api import Device
    space = _space(a)
    dev = Device(a.device)
    dev.bind(space.problem())
    n = 0
    for line in open(a.log_file):
        row = json.loads(line)
        if "candidate" not in row:
            continue
        c = space.deserialize(json.dumps(row["candidate"]))
        m = dev.evaluate_tiles(c.tiles(), reps=5) if space.tiles else dev.evaluate(c.nest(), watchdog=0, reps=5)
        print(json.dumps({"i": row["i"], "logged_us": row["median_ns"] / 1e3, "replayed_us": m.median_ns / 1e3,
                          "status": m.status}))
        n += 1
    dev.close()
    return 0 if n else 1


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1904_03383_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("kind")
        for d in ("m", "n", "k"):
            p.add_argument(f"--{d}", type=int, default=0)
        p.add_argument("--batch", type=int, default=1)
        p.add_argument("--a-stride", type=int, default=1)
        p.add_argument("--factors", nargs="*", help="one comma list per strip-mining universe")
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--candidate")

    p = sub.add_parser("explore")
    common(p)
    p.add_argument("--evals", type=int, default=64)
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--log")
    p.add_argument("--out", help="write the best candidate's serialization here")
    p.add_argument("--decision-order", default=None, help="comma separated choice names (default: paper order)")
    p.add_argument("--tree-depth", type=int, default=0, help="decisions kept in the Monte-Carlo tree (0: 12)")
    p.set_defaults(fn=cmd_explore)
    p = sub.add_parser("codegen")
    common(p)
    p.set_defaults(fn=cmd_codegen)
    p = sub.add_parser("bound")
    common(p)
    p.add_argument("--root", action="store_true")
    p.add_argument("--l2-flushed", action="store_true")
    p.set_defaults(fn=cmd_bound)
    p = sub.add_parser("estimate")
    common(p)
    p.add_argument("--method", default="knuth", choices=["knuth", "chen", "both"])
    p.add_argument("--probes", type=int, default=100000, help="Knuth descents (the paper's 100,000)")
    p.add_argument("--runs", type=int, default=1000, help="Chen runs (the paper's 1000)")
    p.add_argument("--stratifier", default="depth_remaining")
    p.add_argument("--order", default=None)
    p.set_defaults(fn=cmd_estimate)
    p = sub.add_parser("deadend")
    common(p)
    p.add_argument("--trials", type=int, default=1000)
    p.add_argument("--order", default=None)
    p.set_defaults(fn=cmd_deadend)
    p = sub.add_parser("order-compare")
    common(p)
    p.add_argument("--order", default=None, help="the default order (its reverse is compared)")
    p.add_argument("--depth", type=int, default=9, help="levels profiled")
    p.add_argument("--T-us", dest="T_us", type=float, default=0.0, help="incumbent (us); default: greedy leaf")
    p.add_argument("--slack", type=float, default=1.25, help="T = greedy leaf bound x slack")
    p.add_argument("--min-nodes", type=int, default=1000, help="compare depths where both orders have this many")
    p.add_argument("--node-budget", type=int, default=10 ** 6)
    p.set_defaults(fn=cmd_order_compare)
    p = sub.add_parser("enumerate")
    common(p)
    p.add_argument("--order", default=None)
    p.add_argument("--node-budget", type=int, default=10 ** 6)
    p.set_defaults(fn=cmd_enumerate)
    p = sub.add_parser("replay")
    p.add_argument("log_file")
    common(p)
    p.add_argument("--device", type=int, default=0)
    p.set_defaults(fn=cmd_replay)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # argparse: malformed command line
        return 2 if e.code else 0
    try:
        return a.fn(a)
    except DeadEnd as e:
        print(f"no implementation found: {e}", file=sys.stderr)
        return 3
    except (ValueError, OSError) as e:  # bad space / factors / candidate file, refused enumeration
        print(f"configuration error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
