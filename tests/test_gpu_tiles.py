"""GPU parity of the building-block kernels (tiles.space candidates emitted by
ispc_emit_tiles, compiled by NVRTC for sm_100a, launched through the C-ABI).

  sgemm / batched (FFMA, k ascending per output)  bit-exact vs the oracle
  gemv (shuffle / shared / DSMEM-cluster sums)     |y - y64| <= 1e-5 * sum|a||x|
  sgemm_tc TF32 / 3xTF32                           4e-3 / 1e-5 of sum|a||b|

Small shapes are read back and compared with the CPU oracle; BASELINE shapes
are checked on the device against the golden sequential kernels (themselves
pinned to the oracle by test_golden_kernels_match_oracle)."""
import numpy as np
import pytest

from paper_1904_03383_b200 import DeadEnd, Device, Space
from paper_1904_03383_b200 import _native as N
from tests.oracle_lib import Oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    d = Device(0)
    yield d
    d.close()


def _leaves(space, n):
    root = space.root()
    for seed in range(n):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        yield leaf


def _run_many(dev, space, n, min_ok):
    dev.bind(space.problem())
    counts = {"ok": 0, "illegal": 0}
    for leaf in _leaves(space, n):
        t = leaf.tiles()
        m = dev.evaluate_tiles(t, reps=1, warmup=0)
        if m.status == "illegal":
            counts["illegal"] += 1
            continue
        assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())
        counts["ok"] += 1
    assert counts["ok"] >= min_ok, counts
    return counts


def test_golden_gemv_and_batched_match_oracle(dev):
    orc = Oracle()
    for space in (Space("gemv", m=256, n=128), Space("batched", m=8, n=16, k=32, batch=6)):
        p = space.problem()
        dev.bind(p)
        for name, ref in orc.expected(p).items():
            got = dev.read(name, ref.size, expected=True)
            assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), name


def test_gemv_small_readback(dev):
    orc = Oracle()
    space = Space("gemv", m=512, n=256)
    p = space.problem()
    dev.bind(p)
    a, x = orc.fill(512 * 256, p.seed, "a"), orc.fill(256, p.seed, "x")
    y64, scale = orc.gemv_f64(a, x, 512, 256)
    ok = 0
    for leaf in _leaves(space, 80):
        m = dev.evaluate_tiles(leaf.tiles(), reps=1, warmup=0)
        if m.status == "illegal":
            continue
        assert m.status == "ok", (leaf.tiles().as_dict(), m, dev.error())
        y = dev.read("y", 512).astype(np.float64)
        assert np.max(np.abs(y - y64) / np.maximum(scale, 1e-30)) <= 1e-5
        ok += 1
    assert ok >= 10


def test_gemv_baseline_shape(dev):
    _run_many(dev, Space("gemv", m=4096, n=4096), 40, 15)


@pytest.mark.parametrize("staging", ["CP_ASYNC", "TMA"])
def test_gemv_staged_rings(dev, staging):
    """cp.async and TMA (mbarrier expect-tx) column rings, norm-wise 1e-5."""
    space = Space("gemv", m=4096, n=4096)
    dev.bind(space.problem())
    root = space.root().decide("staging", ["kernel"], staging)
    ok = 0
    for seed in range(30):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        t = leaf.tiles()
        m = dev.evaluate_tiles(t, reps=1, warmup=0)
        if m.status == "illegal":
            continue
        assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())
        ok += 1
    assert ok >= 5


def test_gemv_cluster_split_is_exercised(dev):
    space = Space("gemv", m=4096, n=4096)
    dev.bind(space.problem())
    c = space.root()
    c.decide("tile", ["split"], "8")
    c.decide("tile", ["warps_n"], "2")
    leaf = c.first_leaf()
    t = leaf.tiles()
    m = dev.evaluate_tiles(t, reps=3)
    assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())
    assert m.launch.cluster[0] == 8


def test_sgemm_small_readback_bit_exact(dev):
    orc = Oracle()
    space = Space("sgemm", m=128, n=64, k=32)
    p = space.problem()
    dev.bind(p)
    ref = orc.expected(p)["c"]
    a = orc.fill(128 * 32, p.seed, "a").reshape(32, 128).T.astype(np.float64)
    b = orc.fill(32 * 64, p.seed, "b").reshape(64, 32).T.astype(np.float64)
    c64 = (a @ b).T.ravel()
    scale = (np.abs(a) @ np.abs(b)).T.ravel()
    ok = 0
    for leaf in _leaves(space, 120):
        t = leaf.tiles()
        m = dev.evaluate_tiles(t, reps=1, warmup=0)
        if m.status == "illegal":
            continue
        assert m.status == "ok", (t.as_dict(), m, dev.error())
        got = dev.read("c", ref.size)
        if t.split > 1:  # split-K sums cluster partials: norm-wise
            assert np.max(np.abs(got - c64) / scale) <= 1e-5, t.as_dict()
        else:
            assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), t.as_dict()
        ok += 1
    assert ok >= 10


def test_sgemm_baseline_shape(dev):
    _run_many(dev, Space("sgemm", m=1024, n=1024, k=1024), 30, 10)


def test_batched_baseline_shape(dev):
    _run_many(dev, Space("batched", m=32, n=32, k=64, batch=512), 40, 10)


def test_batched_small_readback_bit_exact(dev):
    orc = Oracle()
    space = Space("batched", m=32, n=32, k=64, batch=16)
    p = space.problem()
    dev.bind(p)
    ref = orc.expected(p)["c"]
    ok = 0
    for leaf in _leaves(space, 30):
        m = dev.evaluate_tiles(leaf.tiles(), reps=1, warmup=0)
        if m.status == "illegal":
            continue
        assert m.status == "ok", (leaf.tiles().as_dict(), m, dev.error())
        got = dev.read("c", ref.size)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
        ok += 1
    assert ok >= 5


@pytest.mark.parametrize("engine", ["TF32", "TF32X3"])
def test_tcgen05_sgemm(dev, engine):
    """Random leaves of one engine: every leaf the emitter accepts runs and
    checks on the device (the device never reports illegal what the host
    emitted), and at least 8 of 40 descents reach such a leaf."""
    from paper_1904_03383_b200 import EmitError, tile_cuda
    space = Space("sgemm_tc", m=512, n=512, k=256)
    dev.bind(space.problem())
    root = space.root().decide("engine", ["kernel"], engine)
    ok = 0
    for seed in range(40):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        t = leaf.tiles()
        try:
            tile_cuda(t, "probe")
        except EmitError:
            continue  # statically illegal (e.g. a ring deeper than 227 KiB)
        m = dev.evaluate_tiles(t, reps=1, warmup=0)
        assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())
        ok += 1
    assert ok >= 8, ok


def tc_ring_fits(engine, pair, bn, stages):
    """The emitter's shared-memory rule (emit_tcgen05.cpp tc_stage): a stage
    holds A (16 KiB, 128 rows x 32 k) and this CTA's B rows (BN / pair x 128 B),
    3xTF32 adds the small halves of both; the ring plus its barriers must fit
    in 227 KiB."""
    bnl = int(bn) // (2 if int(pair) >= 2 else 1)
    stage = 16384 + bnl * 128
    if engine == "TF32X3":
        stage *= 2
    return int(stages) * stage + 1024 + 8 * (3 * int(stages) + 6) <= 232448


# static legality of the variants below (emitter rules, checked on the host):
# at 3 stages, 3xTF32 on one CTA cannot hold a BN 256 ring (96 KiB stages)
TC_ILLEGAL = {(e, s, p, b) for e in ("TF32", "TF32X3") for s in ("TMA", "SHARED") for p in ("1", "2")
              for b in ("64", "128", "256") if not tc_ring_fits(e, p, b, 3)}


@pytest.mark.parametrize("bn", ["64", "128", "256"])
@pytest.mark.parametrize("engine", ["TF32", "TF32X3"])
@pytest.mark.parametrize("staging", ["TMA", "SHARED"])
@pytest.mark.parametrize("pair", ["1", "2"])
def test_tcgen05_staging_and_pairs(dev, engine, staging, pair, bn):
    """A staged by TMA or through registers; one CTA per UMMA or a
    cta_group::2 pair (M = 256 over two SMs, B split between them). Every
    variant outside TC_ILLEGAL must run and check."""
    from paper_1904_03383_b200 import EmitError, tile_cuda
    space = Space("sgemm_tc", m=512, n=768, k=192)
    dev.bind(space.problem())
    c = space.root()
    c.decide("engine", ["kernel"], engine).decide("staging", ["kernel"], staging)
    c.decide("tile", ["split"], pair).decide("tile", ["bn"], bn).decide("tile", ["stages"], "3")
    t = c.first_leaf().tiles()
    if (engine, staging, pair, bn) in TC_ILLEGAL:
        with pytest.raises(EmitError):
            tile_cuda(t, "probe")
        return
    m = dev.evaluate_tiles(t, reps=1, warmup=0)
    assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())
    assert m.launch.cluster[0] == (2 if pair == "2" else 0)


@pytest.mark.parametrize("engine", ["TF32", "TF32X3"])
@pytest.mark.parametrize("pair", ["1", "2", "4"])
@pytest.mark.parametrize("staging,bn", [("TMA", "64"), ("SHARED", "128")])
def test_tcgen05_persistent(dev, engine, pair, staging, bn):
    """Persistent grid (148 CTAs): several tiles per CTA through one running
    ring and a double-buffered TMEM accumulator; split 4 = two pairs sharing
    the A boxes by TMA multicast (so it needs TMA-staged A)."""
    from paper_1904_03383_b200 import EmitError, tile_cuda
    space = Space("sgemm_tc", m=2048, n=2048, k=96)
    dev.bind(space.problem())
    c = space.root()
    c.decide("engine", ["kernel"], engine).decide("staging", ["kernel"], staging)
    c.decide("tile", ["split"], pair).decide("tile", ["bn"], bn).decide("tile", ["stages"], "4")
    c.decide("tile", ["grid"], "148")
    t = c.first_leaf().tiles()
    if pair == "4" and staging == "SHARED":
        with pytest.raises(EmitError, match="multicast"):
            tile_cuda(t, "probe")
        return
    if not tc_ring_fits(engine, pair, bn, 4):
        with pytest.raises(EmitError, match="227 KiB"):
            tile_cuda(t, "probe")
        return
    m = dev.evaluate_tiles(t, reps=2, warmup=1)
    assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())
    assert m.launch.grid_x == 148


@pytest.mark.parametrize("split", ["2", "4", "8"])
def test_sgemm_split_k_cluster(dev, split):
    """Split-K over a cluster, partials summed through DSMEM (norm-wise 1e-5)."""
    space = Space("sgemm", m=1024, n=1024, k=1024)
    dev.bind(space.problem())
    root = space.root().decide("tile", ["split"], split)
    ok = 0
    for seed in range(20):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        t = leaf.tiles()
        m = dev.evaluate_tiles(t, reps=1, warmup=0)
        if m.status == "illegal":
            continue
        assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())
        assert m.launch.cluster[0] == int(split)
        ok += 1
    assert ok >= 3


def test_cli_explore_then_replay(tmp_path, capsys):
    """explore writes the JSONL log (improving lines carry the candidate);
    replay re-measures every logged improvement through the C-ABI."""
    import json

    from paper_1904_03383_b200 import cli
    log = tmp_path / "gemv.jsonl"
    args = ["gemv", "--m", "1024", "--n", "1024"]
    assert cli.main(["explore", *args, "--evals", "16", "--log", str(log)]) == 0
    out = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert out["evaluations"] >= 1 and out["ok"] >= 1
    assert cli.main(["replay", str(log), *args]) == 0
    rows = [json.loads(l) for l in capsys.readouterr().out.strip().splitlines()]
    assert rows and all(r["status"] == "ok" for r in rows)


def test_axpy_stream_full_size_bit_exact(dev):
    _run_many(dev, Space("axpy_stream", n=1 << 26), 30, 10)


@pytest.mark.parametrize("knobs", [{"ISPC_ROLLOUT": "deep"}, {"ISPC_ROLLOUT": "ancestor"},
                                   {"ISPC_ELITE_Q": "0.5"}, {"ISPC_GREEDY_P": "0.5", "ISPC_SHARP": "0"},
                                   {"ISPC_LAZY": "0"}, {"ISPC_ASPIRE": "0"}])
def test_search_policy_knobs(monkeypatch, capsys, knobs):
    """Every rollout policy the experiments in DESIGN.md section 5 compare
    runs a search to measured, correct kernels with an admissible bound."""
    import json

    from paper_1904_03383_b200 import cli
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    assert cli.main(["explore", "axpy", "--n", str(1 << 20), "--factors", "2,4", "2,4,8,16,32,64,128,256",
                     "--evals", "48", "--seed", "5"]) == 0
    out = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert out["evaluations"] >= 1 and out["ok"] >= 1
    assert out["bound_violations"] == 0


@pytest.mark.parametrize("engine", ["TF32", "TF32X3"])
@pytest.mark.parametrize("pair", ["1", "2"])
def test_tcgen05_persistent_tail_split(dev, engine, pair):
    """BN 256 persistent grid: the last, partial round of
    tiles is cut into half-width tiles (UMMA N = 128) spread over twice as many
    clusters (160 / 320 tiles over 74 / 148 clusters)."""
    space = Space("sgemm_tc", m=4096, n=2560, k=64)
    dev.bind(space.problem())
    c = space.root()
    c.decide("engine", ["kernel"], engine).decide("staging", ["kernel"], "TMA")
    stages = "2" if engine == "TF32X3" else "3"  # 3xTF32 stages carry B big + small
    c.decide("tile", ["split"], pair).decide("tile", ["bn"], "256").decide("tile", ["stages"], stages)
    c.decide("tile", ["grid"], "148")
    t = c.first_leaf().tiles()
    from paper_1904_03383_b200 import tile_cuda
    src, _ = tile_cuda(t, "k_ts")
    assert "width = 128" in src  # the tail split is emitted
    m = dev.evaluate_tiles(t, reps=2, warmup=1)
    assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())


@pytest.mark.parametrize("cfg", [
    # balanced row blocks: 37 clusters of 8 CTAs, 112 rows each
    dict(staging="DIRECT", vec=4, lanes_m=32, lanes_n=1, warps_m=1, warps_n=16, split=8, unroll=8, grid=296),
    # persistent TMA ring: 37 clusters of 4 CTAs walking 16-row blocks
    dict(staging="TMA", vec=4, lanes_m=4, lanes_n=8, warps_m=1, warps_n=8, split=4, bk=128, stages=8, grid=148),
])
def test_gemv_grid_variants_through_the_abi(dev, cfg):
    """The gemv variants kept out of the search space (measured slower) stay
    correct through ispc_evaluate_tiles (norm-wise 1e-5 of sum |a||x|)."""
    orc = Oracle()
    space = Space("gemv", m=4096, n=4096)
    p = space.problem()
    dev.bind(p)
    t = space.root().first_leaf().tiles()
    t.staging = N.STAGINGS.index(cfg.pop("staging"))
    for k, v in cfg.items():
        setattr(t, k, v)
    m = dev.evaluate_tiles(t, reps=2, warmup=1)
    assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())
    a, x = orc.fill(4096 * 4096, p.seed, "a"), orc.fill(4096, p.seed, "x")
    y64, scale = orc.gemv_f64(a, x, 4096, 4096)
    y = dev.read("y", 4096).astype(np.float64)
    assert np.max(np.abs(y - y64) / np.maximum(scale, 1e-30)) <= 1e-5


@pytest.mark.parametrize("kind,kw", [
    ("gemv", dict(m=512, n=256)),
    ("sgemm", dict(m=256, n=256, k=128)),
    ("batched", dict(m=32, n=32, k=64, batch=64)),
    ("sgemm_tc", dict(m=256, n=256, k=256)),
    ("axpy_stream", dict(n=1 << 20)),
])
def test_pdl_kernels_match_their_plain_twins(dev, kind, kw):
    """Programmatic dependent launch (tile decision `pdl`): the same
    configuration with pdl = 1, launched back to back with the PDL attribute
    over rotating input copies, passes the on-device check and leaves exactly
    the output its pdl = 0 twin leaves (griddepcontrol.wait orders every
    memory access after the previous grid)."""
    space = Space(kind, **kw)
    dev.bind(space.problem())
    out_name, out_n = {"gemv": ("y", kw.get("m", 0)), "axpy_stream": ("z", kw.get("n", 0))}.get(
        kind, ("c", kw.get("m", 0) * kw.get("n", 0) * kw.get("batch", 1)))
    checked = 0
    root = space.root().decide("tile", ["pdl"], "1")
    for seed in range(40):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        t1 = leaf.tiles()
        m1 = dev.evaluate_tiles(t1, reps=4, warmup=1, rotate=3)
        if m1.status == "illegal":
            continue
        assert m1.status == "ok" and m1.mismatches == 0, (t1.as_dict(), m1, dev.error())
        got1 = dev.read(out_name, out_n)
        t0 = leaf.tiles()
        t0.pdl = 0
        m0 = dev.evaluate_tiles(t0, reps=1, warmup=0)
        assert m0.status == "ok", (t0.as_dict(), m0, dev.error())
        got0 = dev.read(out_name, out_n)
        assert np.array_equal(got1.view(np.uint32), got0.view(np.uint32)), t1.as_dict()
        checked += 1
        if checked >= 3:
            break
    assert checked >= 1, kind


def test_polish_keeps_the_search_in_its_space_and_checked(dev):
    """The config searches' polish (hill climbing from the search's best
    measured leaves): every kernel it ends on is a leaf of the space that passes
    the on-device check, and it never returns something slower than where it
    started by more than the timing noise."""
    from paper_1904_03383_b200 import Search
    from paper_1904_03383_b200.measure import rotation
    from paper_1904_03383_b200.polish import polish_many
    space = Space("batched", m=32, n=32, k=64, batch=128)
    s = Search(space, device=0, seed=11, reps=3, warmup=1)
    s.step(48, max_seconds=120)
    best, elites = s.best(), s.elites()
    s.close()
    assert best is not None and elites, "the search measured nothing"
    rot = rotation(space, dev.info()["l2_bytes"])
    end, rep = polish_many(space, [best] + elites, dev, rot, budget=60)
    assert end.fully_specified and rep["evaluated"] <= 60 + 4 * 3 + 4  # each start may overshoot by a confirm pair
    dev.bind(space.problem())
    m = dev.evaluate_tiles(end.tiles(), reps=8, warmup=2, rotate=rot)
    assert m.status == "ok" and m.mismatches == 0, (end.tiles().as_dict(), m)
    for run in rep["starts"]:
        assert run["end_us"] <= run["start_us"] * 1.001, run
