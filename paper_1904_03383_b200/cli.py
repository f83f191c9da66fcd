"""Command line over the evaluation path (the reference's CLI is a stub,
proj/tools/src/main.cpp:1; its commands are specified at SPEC.md:569-604).

  python -m paper_1904_03383_b200.cli explore  axpy --n 1048576 --factors 2,4 32,64,128 --evals 64 --log run.jsonl
  python -m paper_1904_03383_b200.cli explore  gemv --m 4096 --n 4096 --evals 128
  python -m paper_1904_03383_b200.cli codegen  sgemm --m 1024 --n 1024 --k 1024 [--candidate c.json] [--seed 3]
  python -m paper_1904_03383_b200.cli bound    matmul --m 64 --n 64 --k 64 --factors 2,4 [--candidate c.json]
  python -m paper_1904_03383_b200.cli replay   run.jsonl axpy --n 1048576 --factors 2,4 32,64,128
  python -m paper_1904_03383_b200.cli estimate matmul --m 256 --n 256 --k 32 --factors 2,4,8,16,32 2,4 --probes 500

`codegen` and `bound` need no GPU. `explore` and `replay` run on cuda device
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
    """Knuth's estimate of the space size (the reference's tree_size is a stub)."""
    space = _space(a)
    print(json.dumps(space.root().estimate_tree(a.probes, seed=a.seed, order=a.order)))
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
    p.add_argument("--probes", type=int, default=1000)
    p.add_argument("--order", default=None)
    p.set_defaults(fn=cmd_estimate)
    p = sub.add_parser("replay")
    p.add_argument("log_file")
    common(p)
    p.add_argument("--device", type=int, default=0)
    p.set_defaults(fn=cmd_replay)
    a = ap.parse_args(argv)
    try:
        return a.fn(a)
    except DeadEnd as e:
        print(f"dead end: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
