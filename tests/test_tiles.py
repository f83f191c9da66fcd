"""Building-block spaces (host/tiles.space through the reference's
build_space): space construction, propagation facts, the B200 lower bound,
and the emitted kernels executed by the CPU emulator against the oracle
(bit-exact for the FFMA sgemm / batched kernels, norm-wise 1e-5 against the
fp64 oracle for the reordered gemv)."""
import numpy as np
import pytest

from paper_1904_03383_b200 import DeadEnd, EmitError, Space, tile_cuda
from paper_1904_03383_b200 import _native as N
from tests import emu
from tests.oracle_lib import Oracle

SEED = 0x190403383


def _leaves(space, n, order=None, root=None):
    root = root or space.root()
    out = []
    for seed in range(n):
        try:
            leaf, _, _ = root.random_leaf(seed, order=order)
        except DeadEnd:
            continue
        out.append(leaf)
    return out


@pytest.mark.parametrize("kind,kw", [
    ("gemv", dict(m=4096, n=4096)),
    ("sgemm", dict(m=1024, n=1024, k=1024)),
    ("batched", dict(m=32, n=32, k=64, batch=512)),
    ("sgemm_tc", dict(m=4096, n=4096, k=4096)),
    ("sgemm_tc_x3", dict(m=4096, n=4096, k=4096)),
])
def test_space_builds_and_is_deterministic(kind, kw):
    a, b = Space(kind, **kw), Space(kind, **kw)
    sa, sb = a.stats(), b.stats()
    assert sa["root_digest"] == sb["root_digest"]
    assert sa["instances"] > 0 and sa["root_open"] > 0
    leaf = a.root().first_leaf()
    assert leaf.fully_specified
    assert leaf.digest == b.deserialize(leaf.serialize()).digest


def test_gemv_lane_split_propagates():
    """warp_lanes() == 32: deciding lanes_m fixes lanes_n through the counter."""
    s = Space("gemv", m=256, n=256)
    c = s.root()
    c.decide("tile", ["lanes_m"], "8")
    with pytest.raises(DeadEnd):
        c.clone().decide("tile", ["lanes_n"], "8")
    c.clone().decide("tile", ["lanes_n"], "4")
    leaf = c.first_leaf()
    t = leaf.tiles()
    assert t.lanes_m * t.lanes_n == 32


def test_sgemm_thread_and_register_counters():
    s = Space("sgemm", m=256, n=256, k=64)
    for leaf in _leaves(s, 40):
        t = leaf.tiles()
        assert 32 <= t.thr_m * t.thr_n <= 1024
        assert t.tm * t.tn <= 128
        assert N.STAGINGS[t.staging] in ("SHARED", "CP_ASYNC") and N.ENGINES[t.engine] == "FFMA"
    c = s.root()
    c.decide("tile", ["thr_m"], "256")
    with pytest.raises(DeadEnd):
        c.clone().decide("tile", ["thr_n"], "8")  # 2048 threads


def test_tcgen05_space_stages_in_shared_memory():
    s = Space("sgemm_tc", m=512, n=512, k=512)
    for leaf in _leaves(s, 10):
        t = leaf.tiles()
        assert N.STAGINGS[t.staging] in ("TMA", "SHARED") and N.ENGINES[t.engine] in ("TF32", "TF32X3")
        assert t.split in (1, 2, 4)
    # cta_group::2 pairs need M divisible by 256
    s2 = Space("sgemm_tc", m=384, n=512, k=512)
    assert all(leaf.tiles().split == 1 for leaf in _leaves(s2, 6))
    c = s.root().decide("tile", ["split"], "2").first_leaf()
    src, L = tile_cuda(c.tiles(), "k_pair")
    assert "cta_group::2" in src and L.cluster[0] == 2 and L.grid_x == (512 // 256) * (512 // c.tiles().bn) * 2


@pytest.mark.parametrize("kind,kw", [
    ("gemv", dict(m=4096, n=4096)),
    ("sgemm", dict(m=1024, n=1024, k=1024)),
    ("batched", dict(m=32, n=32, k=64, batch=512)),
])
def test_bound_is_monotone_along_descents(kind, kw):
    s = Space(kind, **kw)
    root = s.root()
    b0 = root.bound()["total"]
    assert b0 > 0
    for leaf in _leaves(s, 8):
        bl = leaf.bound()["total"]
        assert bl >= b0 * (1 - 1e-12)


def _regions(orc, p):
    nan = lambda n: np.full(n, np.nan, dtype=np.float32)  # noqa: E731
    if p.kind == 3:
        return {"a": orc.fill(p.m * p.n, p.seed, "a"), "x": orc.fill(p.n, p.seed, "x"), "y": nan(p.m)}
    bt = max(int(p.batch), 1)
    return {"a": orc.fill(bt * p.m * p.k, p.seed, "a"), "b": orc.fill(bt * p.k * p.n, p.seed, "b"),
            "c": nan(bt * p.m * p.n)}


def _emulate_all(space, want, max_threads=256, n=30, root=None):
    orc = Oracle()
    p = space.problem()
    checked = 0
    for leaf in _leaves(space, n, root=root):
        t = leaf.tiles()
        try:
            src, L = tile_cuda(t, "k_emu")
        except EmitError:
            continue
        if L.block[0] > max_threads or L.cluster[0] > 1 or L.num_tmaps:
            continue  # clusters and TMA need the device (tests/test_gpu_tiles.py)
        regs = _regions(orc, p)
        emu.run(src, L, regs)
        want(regs, t)
        checked += 1
    return checked


def test_sgemm_kernels_bit_exact_on_emulator():
    s = Space("sgemm", m=32, n=32, k=32)
    orc = Oracle()
    p = s.problem()
    r = _regions(orc, p)
    ref = orc.matmul(r["a"], r["b"], 32, 32, 32)

    def want(regs, t):
        assert np.array_equal(regs["c"].view(np.uint32), ref.view(np.uint32)), t.as_dict()

    # clusters (split-K) need concurrent CTAs: checked on the GPU
    assert _emulate_all(s, want, n=80, root=s.root().decide("tile", ["split"], "1")) >= 5


@pytest.mark.parametrize("cfg", [
    dict(thr_m=8, thr_n=4, tm=4, tn=4, bk=8, stages=2),
    dict(thr_m=4, thr_n=8, tm=8, tn=4, bk=4, stages=3),
    dict(thr_m=16, thr_n=4, tm=4, tn=8, bk=16, stages=2),
])
def test_warp_tiled_ffma2_sgemm_bit_exact_on_emulator(cfg):
    """The warp-tiled FFMA2 building block (CP_ASYNC, vec 4, tm/tn multiples of
    4, whole warps): B transposed by 4-byte cp.async, fragments double
    buffered, two fmas per FFMA2 in ascending k: bit-identical to the oracle."""
    s = Space("sgemm", m=64, n=32, k=32)
    c = s.root().decide("staging", ["kernel"], "CP_ASYNC")
    for k, v in dict(cfg, vec=4, split=1).items():
        c = c.decide("tile", [k], str(v))
    t = c.first_leaf().tiles()
    src, L = tile_cuda(t, "k_emu")
    assert "__ffma2_rn" in src and "ispc_cp_async_ca4" in src
    orc = Oracle()
    r = _regions(orc, s.problem())
    ref = orc.matmul(r["a"], r["b"], 64, 32, 32)
    emu.run(src, L, r)
    assert np.array_equal(r["c"].view(np.uint32), ref.view(np.uint32)), t.as_dict()


def test_batched_kernels_bit_exact_on_emulator():
    s = Space("batched", m=8, n=8, k=16, batch=8)
    orc = Oracle()
    p = s.problem()
    r = _regions(orc, p)
    ref = orc.batched(r["a"], r["b"], 8, 8, 8, 16)

    def want(regs, t):
        assert np.array_equal(regs["c"].view(np.uint32), ref.view(np.uint32)), t.as_dict()

    assert _emulate_all(s, want) >= 5


def test_gemv_kernels_normwise_on_emulator():
    s = Space("gemv", m=128, n=128)
    orc = Oracle()
    p = s.problem()
    r = _regions(orc, p)
    y64, scale = orc.gemv_f64(r["a"], r["x"], 128, 128)

    def want(regs, t):
        err = np.abs(regs["y"].astype(np.float64) - y64) / np.maximum(scale, 1e-30)
        assert np.all(np.isfinite(regs["y"])) and err.max() <= 1e-5, (t.as_dict(), err.max())

    assert _emulate_all(s, want, max_threads=1024, n=200) >= 5


def test_illegal_configurations_are_rejected():
    s = Space("gemv", m=64, n=64)
    t = s.root().first_leaf().tiles()
    t.split = 16
    with pytest.raises(EmitError):
        tile_cuda(t)
    t = Space("sgemm", m=64, n=64, k=64).root().first_leaf().tiles()
    t.bk = 3
    with pytest.raises(EmitError):
        tile_cuda(t)


def test_cli_codegen_and_bound(capsys):
    from paper_1904_03383_b200 import cli
    assert cli.main(["codegen", "sgemm", "--m", "64", "--n", "64", "--k", "64", "--seed", "2"]) == 0
    src = capsys.readouterr().out
    assert "__global__" in src and "__fmaf_rn" in src
    assert cli.main(["bound", "gemv", "--m", "4096", "--n", "4096", "--root"]) == 0
    b = __import__("json").loads(capsys.readouterr().out)
    assert b["dram"] > 8e-6 and b["total"] >= b["dram"]
    assert cli.main(["codegen", "axpy", "--n", "1024", "--factors", "4", "2,8,32", "--seed", "1"]) == 0
    assert "__global__" in capsys.readouterr().out


def test_axpy_stream_bit_exact_on_emulator():
    s = Space("axpy_stream", n=4096)
    orc = Oracle()
    p = s.problem()
    x, y = orc.fill(4096, p.seed, "x"), orc.fill(4096, p.seed, "y")
    ref = orc.axpy(x, y, p.alpha)
    checked = 0
    for leaf in _leaves(s, 40):
        t = leaf.tiles()
        if t.grid == 0 or t.threads > 256:
            continue  # keep the fiber emulation small
        src, L = tile_cuda(t, "k_emu")
        regs = {"x": x.copy(), "y": y.copy(), "z": np.full(4096, np.nan, dtype=np.float32)}
        emu.run(src, L, regs, p.alpha)
        assert np.array_equal(regs["z"].view(np.uint32), ref.view(np.uint32)), t.as_dict()
        checked += 1
    assert checked >= 3


def test_tcgen05_cluster_and_grid_rules():
    """Emitter rules of the tensor-core tile: A multicast needs TMA-staged A,
    a persistent grid must hold whole clusters, and the BN 256 persistent
    grid splits its partial last round into half-width tiles."""
    s = Space("sgemm_tc", m=4096, n=4096, k=4096)

    def leaf(**kv):
        c = s.root().decide("engine", ["kernel"], "TF32")
        c.decide("staging", ["kernel"], kv.pop("staging", "TMA"))
        for k, v in kv.items():
            c.decide("tile", [k], str(v))
        return c.first_leaf().tiles()

    with pytest.raises(EmitError):
        tile_cuda(leaf(staging="SHARED", split=4, grid=148, bn=128, stages=2))
    src, L = tile_cuda(leaf(split=2, bn=256, stages=4, grid=148))
    assert "width = 128" in src and L.grid_x == 148 and L.cluster[0] == 2  # 256 tiles = 3 x 74 + 34 halves
    src, L = tile_cuda(leaf(split=2, bn=256, stages=4, grid=128))
    assert "width = 128" not in src  # 256 tiles = 4 x 64 exactly: no tail
    t = leaf(split=2, bn=256, stages=4, grid=128)
    t.grid = 127  # not a whole number of pairs
    with pytest.raises(EmitError):
        tile_cuda(t)


def test_gemv_grid_requires_a_streaming_staging():
    t = Space("gemv", m=4096, n=4096).root().first_leaf().tiles()
    t.staging = N.STAGINGS.index("CP_ASYNC")
    t.bk, t.stages, t.grid = 64, 2, 296
    with pytest.raises(EmitError):
        tile_cuda(t)


def test_pdl_is_a_decision_of_every_family_and_shapes_the_kernel():
    """`pdl` (programmatic dependent launch) is a tile decision of every
    building-block family; pdl = 1 makes griddepcontrol.wait the kernel's first
    statement and sets ispc_launch.pdl, pdl = 0 emits neither, and the two are
    different kernels to time (different source hashes). The emulator runs a
    pdl = 1 sgemm bit-exactly (the wait and trigger are no-ops there)."""
    for kind, kw in [("gemv", dict(m=256, n=128)), ("sgemm", dict(m=64, n=64, k=32)),
                     ("batched", dict(m=8, n=16, k=32, batch=6)), ("sgemm_tc", dict(m=256, n=256, k=128)),
                     ("axpy_stream", dict(n=1 << 12))]:
        s = Space(kind, **kw)
        leaves = {}
        for v in ("0", "1"):
            for leaf in _leaves(s, 40, root=s.root().decide("tile", ["pdl"], v)):
                try:
                    src, L = tile_cuda(leaf.tiles(), "k_pdl")
                except EmitError:
                    continue
                leaves[v] = (leaf.tiles(), src, L)
                break
        assert set(leaves) == {"0", "1"}, kind
        t1, src1, L1 = leaves["1"]
        t0, src0, L0 = leaves["0"]
        assert t1.pdl == 1 and L1.pdl == 1 and t0.pdl == 0 and L0.pdl == 0
        sig = src1.index(" k_pdl(")
        body = src1[src1.index(") {\n", sig) + 4:]
        assert body.startswith("  ispc_grid_dep_wait();\n  ispc_grid_dep_trigger();\n"), kind
        assert "ispc_grid_dep" not in src0
        t0.pdl = 1
        src01, L01 = tile_cuda(t0, "k_pdl")
        assert L01.source_hash != L0.source_hash and src01.replace("  ispc_grid_dep_wait();\n  ispc_grid_dep_trigger();\n", "") == src0
    # bit-exact on the emulator with pdl
    s = Space("sgemm", m=32, n=32, k=32)
    orc = Oracle()
    p = s.problem()
    r = _regions(orc, p)
    ref = orc.matmul(r["a"], r["b"], 32, 32, 32)

    def want(regs, t):
        assert t.pdl == 1
        assert np.array_equal(regs["c"].view(np.uint32), ref.view(np.uint32)), t.as_dict()

    root = s.root().decide("tile", ["split"], "1").decide("tile", ["pdl"], "1")
    assert _emulate_all(s, want, n=80, root=root) >= 3


def test_polish_neighbours_are_leaves_of_the_space():
    """The config searches' hill-climbing polish (paper_1904_03383_b200/polish.py)
    only ever measures leaves of the same space: every single-decision and
    reshaping-pair neighbour is a fully specified candidate decided through the
    reference engine, differs from the incumbent, and round-trips its
    decisions."""
    from paper_1904_03383_b200 import polish as P
    for kind, kw in [("sgemm", dict(m=1024, n=1024, k=1024)), ("gemv", dict(m=4096, n=4096)),
                     ("batched", dict(m=32, n=32, k=64, batch=512)), ("sgemm_tc", dict(m=4096, n=4096, k=4096))]:
        s = Space(kind, **kw)
        leaf = _leaves(s, 10)[0]
        enums, params = P._decisions(s, leaf)
        assert "pdl" in params
        singles, pairs = P.neighbours(s, enums, params), P.neighbours(s, enums, params, pairs=True)
        assert singles, kind
        for why, e, q in singles + pairs:
            assert (e, q) != (enums, params), why
            c = P._leaf(s, e, q)
            assert c is not None and c.fully_specified
            e2, q2 = P._decisions(s, c)
            assert (e2, q2) == (e, q), why
