"""Hill-climbing polish of a building-block search's incumbent.

The tile spaces' leaves mostly share one lower bound, so the tree search
(host/search.cpp) samples them by measured statistics and elite-guided
rollouts; the configurations it returns are often one or two decisions away
from a faster one (profiles/r2m_sweep: 47.9-50.3 us against 46.97 us for the
best sgemm configuration of the space). This pass measures the incumbent's
single-decision neighbours - each tile parameter doubled, halved, quartered or
toggled, each enum decision changed; when none improves, the pairs that double
one parameter and halve another - through the same C-ABI evaluation (NVRTC
compile, rotation timing, on-device check), moves to the fastest one that is
faster by more than the noise margin, and repeats until no neighbour improves
or the evaluation budget is spent. Every neighbour is a leaf of the same space
(decided through the reference engine), so nothing outside the space is ever
measured."""
from __future__ import annotations

from . import _native as N
from .api import Candidate, DeadEnd, Device, Space

TILE_PARAMS = ("thr_m", "thr_n", "tm", "tn", "bk", "bn", "stages", "vec", "lanes_m", "lanes_n", "warps_m",
               "warps_n", "split", "unroll", "per_cta", "threads", "grid", "lds", "pdl")
ENUMS = {"staging": N.STAGINGS, "engine": N.ENGINES, "xreduce": N.XREDUCES, "cache": N.CACHES}


def _decisions(space: Space, leaf: Candidate) -> tuple[dict, dict]:
    """The leaf's enum and tile-parameter decisions (only the parameters the
    family has: deciding an absent one raises)."""
    d = leaf.tiles().as_dict()
    enums = {k: d[k] for k in ENUMS}
    params = {}
    for p in TILE_PARAMS:
        try:
            space.root().decide("tile", [p], str(d[p]))
        except (DeadEnd, ValueError):
            continue
        params[p] = d[p]
    return enums, params


def _leaf(space: Space, enums: dict, params: dict) -> Candidate | None:
    c = space.root()
    try:
        for ch, v in enums.items():
            c.decide(ch, ["kernel"], v)
        for p, v in params.items():
            c.decide("tile", [p], str(v))
    except (DeadEnd, ValueError):
        return None
    return c if c.fully_specified else None


def neighbours(space: Space, enums: dict, params: dict, pairs: bool = False) -> list[tuple[str, dict, dict]]:
    """Single-decision neighbours (each parameter x2, /2, x4, /4, +-1 when
    small, or set to 0 / 1, a persistent grid to any SM-shaped size; each
    enum changed), or
    with `pairs` the moves that
    double one parameter and halve another (a CTA or warp reshaped at the
    same thread count, a tile traded for split-K depth)."""
    out, seen = [], set()

    def add(why, e, q):
        key = tuple(sorted(q.items())) + tuple(sorted(e.items()))
        if key not in seen:
            seen.add(key)
            out.append((why, e, q))

    if pairs:
        for p, v in params.items():
            for r, w in params.items():
                if p != r and v > 0 and w > 1:
                    add(f"{p}={v * 2},{r}={w // 2}", enums, dict(params, **{p: v * 2, r: w // 2}))
    else:
        for p, v in params.items():
            # persistent grid sizes are SM-count shaped, not powers of two
            extra = {0, 128, 144, 148, 296, 592, 1184, 2368, 4736} if p == "grid" else {0, 1}
            if 1 < v <= 16:  # ring depths and other small counts are not powers of two
                extra |= {v - 1, v + 1}
            for w in sorted(({v * 2, v // 2, v * 4, v // 4} | extra) - {v}):
                if w >= 0:
                    add(f"{p}={w}", enums, dict(params, **{p: w}))
        for ch, values in ENUMS.items():
            for w in values:
                if w != enums[ch]:
                    add(f"{ch}={w}", dict(enums, **{ch: w}), params)
    return [(why, e, q) for why, e, q in out if _leaf(space, e, q) is not None]


def polish(space: Space, leaf: Candidate, dev: Device, rotate: int, budget: int = 240, margin: float = 0.005,
           reps: int = 3) -> tuple[Candidate, dict]:
    """Returns (best leaf, report). `budget` caps the neighbour evaluations;
    a neighbour replaces the incumbent when it is faster by more than
    `margin` (relative) and passes the on-device check."""
    dev.bind(space.problem())
    enums, params = _decisions(space, leaf)
    # a screening time is one group of back-to-back launches; a candidate that
    # screens faster is confirmed on 4 groups beside a re-time of the incumbent
    # (the fastest of many one-group screens is biased low)
    confirm = 4 * max(rotate, 1)
    m = dev.evaluate_tiles(leaf.tiles(), reps=confirm, warmup=2, rotate=rotate)
    if m.status != "ok":
        return leaf, {"evaluated": 1, "status": m.status}
    best_ns, start_ns, evaluated, moves = m.median_ns, m.median_ns, 1, []
    tried = set()
    pairs = False
    while evaluated < budget:
        step_best = None
        for why, e, q in neighbours(space, enums, params, pairs):
            key = (tuple(sorted(e.items())), tuple(sorted(q.items())))
            if key in tried:
                continue
            tried.add(key)
            if evaluated >= budget:
                break
            cand = _leaf(space, e, q)
            r = dev.evaluate_tiles(cand.tiles(), reps=reps, warmup=1, rotate=rotate)
            evaluated += 1
            if r.status == "ok" and r.median_ns < best_ns * (1 - margin):
                c = dev.evaluate_tiles(cand.tiles(), reps=confirm, warmup=2, rotate=rotate)
                inc = dev.evaluate_tiles(_leaf(space, enums, params).tiles(), reps=confirm, warmup=2, rotate=rotate)
                evaluated += 2
                if inc.status == "ok":
                    best_ns = min(best_ns, inc.median_ns) if step_best is None else best_ns
                if c.status == "ok" and c.median_ns < inc.median_ns * (1 - margin):
                    if step_best is None or c.median_ns < step_best[0]:
                        step_best = (c.median_ns, why, e, q)
        if step_best is None:
            if pairs:
                break
            pairs = True  # no single move improves: try the reshaping pairs
            continue
        pairs = False
        best_ns, why, enums, params = step_best
        moves.append({"move": why, "us": round(best_ns / 1e3, 3)})
    best = _leaf(space, enums, params)
    return best, {"evaluated": evaluated, "start_us": round(start_ns / 1e3, 3), "end_us": round(best_ns / 1e3, 3),
                  "moves": moves}


def polish_many(space: Space, starts: list[Candidate], dev: Device, rotate: int, budget: int = 400,
                max_starts: int = 4) -> tuple[Candidate, dict]:
    """Hill-climbs from up to `max_starts` distinct starting leaves (the
    search's best measured ones, fastest first), splitting the budget, and
    returns the fastest end point by a final paired re-time."""
    seen, runs = set(), []
    for leaf in starts:
        key = tuple(sorted(leaf.tiles().as_dict().items()))
        if key in seen:
            continue
        seen.add(key)
        runs.append(leaf)
        if len(runs) == max_starts:
            break
    if not runs:
        return None, {"evaluated": 0}
    reports, ends = [], []
    for leaf in runs:
        end, rep = polish(space, leaf, dev, rotate, budget=budget // len(runs))
        reports.append(rep)
        ends.append(end)
    confirm = 4 * max(rotate, 1)
    best, best_ns = None, float("inf")
    for end in ends:  # final paired re-time of the end points
        m = dev.evaluate_tiles(end.tiles(), reps=confirm, warmup=2, rotate=rotate)
        if m.status == "ok" and m.median_ns < best_ns:
            best, best_ns = end, m.median_ns
    return best or runs[0], {"evaluated": sum(r.get("evaluated", 0) for r in reports) + len(ends),
                             "starts": reports, "end_us": round(best_ns / 1e3, 3)}
