"""GPU parity at every BASELINE.json shape, read back and compared on the host
with the CPU oracle (oracle/numeric.c through tests/oracle_lib.py):

  axpy 2^26, FFMA sgemm 1024^3 (split 1), batched 512 x 32x32x64   bit-exact
  gemv 4096^2 (the searched best)           |y - y64| <= 1e-5 * sum|a||x|
  tcgen05 sgemm 4096^3  TF32 / 3xTF32       |c - c64| <= 4e-3 / 1e-5 * sum|a||b|

c64 / y64 are float64 products of the oracle's inputs (numpy, OpenBLAS). The
device golden kernels (the on-device checker of the search) are pinned to the
oracle bit for bit at the same shapes. Every listed configuration must run:
none may come back illegal."""
import numpy as np
import pytest

from paper_1904_03383_b200 import DeadEnd, Device, Search, Space
from tests.oracle_lib import Oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    d = Device(0)
    yield d
    d.close()


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def _colmajor(v, rows, cols):
    """A column-major rows x cols operand (the builders' layout) as an array."""
    return v.reshape(cols, rows).T


def _configured(space, **d):
    c = space.root()
    for k in ("engine", "staging"):
        if k in d:
            c.decide(k, ["kernel"], d.pop(k))
    for k, v in d.items():
        c.decide("tile", [k], str(v))
    return c.first_leaf().tiles()


# ---------------------------------------------------------------- golden kernels

@pytest.mark.parametrize("spec", [
    dict(kind="axpy_stream", n=1 << 26),
    dict(kind="gemv", m=4096, n=4096),
    dict(kind="sgemm", m=1024, n=1024, k=1024),
    dict(kind="batched", m=32, n=32, k=64, batch=512),
], ids=lambda s: s["kind"])
def test_golden_kernels_match_oracle_at_baseline_shapes(dev, orc, spec):
    space = Space(**spec)
    p = space.problem()
    dev.bind(p)
    for name, ref in orc.expected(p).items():
        got = dev.read(name, ref.size, expected=True)
        assert np.array_equal(_bits(got), _bits(ref)), name


def test_golden_sgemm_4096_matches_oracle_on_sampled_columns(dev, orc):
    """The sequential golden kernel at 4096^3: 8 columns of C recomputed by the
    oracle (k ascending fmaf) from the same seeded inputs, bit for bit."""
    m = n = k = 4096
    space = Space("sgemm_tc", m=m, n=n, k=k)
    p = space.problem()
    dev.bind(p)
    a = orc.fill(m * k, p.seed, "a")
    b = _colmajor(orc.fill(k * n, p.seed, "b"), k, n)
    cols = [0, 1, 127, 128, 2047, 3000, 4094, 4095]
    bsub = np.ascontiguousarray(b[:, cols].T).ravel()
    ref = orc.matmul(a, bsub, m, len(cols), k)
    got = _colmajor(dev.read("c", m * n, expected=True), m, n)[:, cols]
    assert np.array_equal(_bits(np.ascontiguousarray(got.T).ravel()), _bits(ref))


# ---------------------------------------------------------------- FFMA sgemm 1024^3

SGEMM_1024 = [
    dict(staging="CP_ASYNC", thr_m=16, thr_n=16, tm=8, tn=8, bk=16, stages=3, vec=4, split=1),
    dict(staging="SHARED", thr_m=16, thr_n=16, tm=4, tn=8, bk=8, stages=2, vec=4, split=1),
    dict(staging="CP_ASYNC", thr_m=16, thr_n=8, tm=4, tn=8, bk=16, stages=2, vec=4, split=1),
]


@pytest.fixture(scope="module")
def sgemm_1024_ref(orc):
    space = Space("sgemm", m=1024, n=1024, k=1024)
    p = space.problem()
    return space, p, orc.expected(p)["c"]


@pytest.mark.parametrize("cfg", SGEMM_1024, ids=lambda c: f"{c['staging']}-{c['thr_m']}x{c['thr_n']}-{c['tm']}x{c['tn']}")
def test_sgemm_1024_split1_bit_exact_readback(dev, sgemm_1024_ref, cfg):
    space, p, ref = sgemm_1024_ref
    dev.bind(p)
    t = _configured(space, **dict(cfg))
    m = dev.evaluate_tiles(t, reps=1, warmup=0)
    assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())
    got = dev.read("c", ref.size)
    assert np.array_equal(_bits(got), _bits(ref)), t.as_dict()


def test_sgemm_1024_random_split1_leaves_bit_exact(dev, sgemm_1024_ref):
    """Random split-1 leaves of the FFMA space at 1024^3: every runnable one
    is read back and equals the oracle bit for bit."""
    space, p, ref = sgemm_1024_ref
    dev.bind(p)
    root = space.root().decide("tile", ["split"], "1")
    counts = {"ok": 0, "illegal": 0}
    for seed in range(24):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        t = leaf.tiles()
        m = dev.evaluate_tiles(t, reps=1, warmup=0)
        if m.status == "illegal":
            counts["illegal"] += 1
            continue
        assert m.status == "ok", (t.as_dict(), m, dev.error())
        assert np.array_equal(_bits(dev.read("c", ref.size)), _bits(ref)), t.as_dict()
        counts["ok"] += 1
    assert counts["ok"] >= 6, counts


# ---------------------------------------------------------------- batched 512

def test_batched_512_bit_exact_readback(dev, orc):
    space = Space("batched", m=32, n=32, k=64, batch=512)
    p = space.problem()
    dev.bind(p)
    ref = orc.expected(p)["c"]
    root = space.root()
    counts = {"ok": 0, "illegal": 0}
    for seed in range(30):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        t = leaf.tiles()
        m = dev.evaluate_tiles(t, reps=1, warmup=0)
        if m.status == "illegal":
            counts["illegal"] += 1
            continue
        assert m.status == "ok", (t.as_dict(), m, dev.error())
        assert np.array_equal(_bits(dev.read("c", ref.size)), _bits(ref)), t.as_dict()
        counts["ok"] += 1
    assert counts["ok"] >= 8, counts
    # the hand-picked best of round 1 (4x4 outputs per thread, 16-byte
    # cp.async, one problem per CTA) must be in the space and exact
    t = _configured(Space("batched", m=32, n=32, k=64, batch=512), staging="CP_ASYNC", tm=4, tn=4, vec=4, per_cta=1)
    m = dev.evaluate_tiles(t, reps=1, warmup=0)
    assert m.status == "ok", (t.as_dict(), m, dev.error())
    assert np.array_equal(_bits(dev.read("c", ref.size)), _bits(ref))


# ---------------------------------------------------------------- gemv 4096^2

def test_gemv_4096_searched_best_readback(dev, orc):
    """A short search of the gemv space; its best kernel read back against the
    float64 oracle (norm-wise 1e-5 of sum |a||x|)."""
    space = Space("gemv", m=4096, n=4096)
    p = space.problem()
    s = Search(space, device=0, seed=7, reps=3, warmup=1, rotate=4)
    s.step(48, max_seconds=240)
    best = s.best()
    s.close()
    assert best is not None
    dev.bind(p)
    t = best.tiles()
    m = dev.evaluate_tiles(t, reps=1, warmup=0)
    assert m.status == "ok", (t.as_dict(), m, dev.error())
    a, x = orc.fill(4096 * 4096, p.seed, "a"), orc.fill(4096, p.seed, "x")
    y64, scale = orc.gemv_f64(a, x, 4096, 4096)
    y = dev.read("y", 4096).astype(np.float64)
    assert np.max(np.abs(y - y64) / np.maximum(scale, 1e-30)) <= 1e-5, t.as_dict()


# ---------------------------------------------------------------- tcgen05 4096^3

TC_4096 = [
    dict(engine="TF32", staging="TMA", split=1, bn=128, stages=4),
    dict(engine="TF32", staging="TMA", split=2, bn=256, stages=4),
    dict(engine="TF32", staging="SHARED", split=2, bn=256, stages=4),
    dict(engine="TF32", staging="TMA", split=2, bn=256, stages=6, grid=128),
    dict(engine="TF32", staging="TMA", split=4, bn=256, stages=4, grid=128),
    dict(engine="TF32X3", staging="TMA", split=2, bn=128, stages=3),
    dict(engine="TF32X3", staging="SHARED", split=1, bn=128, stages=3),
    dict(engine="TF32X3", staging="TMA", split=2, bn=256, stages=2, grid=148),
]


@pytest.fixture(scope="module")
def tc_4096_ref(orc):
    m = n = k = 4096
    space = Space("sgemm_tc", m=m, n=n, k=k)
    p = space.problem()
    a = _colmajor(orc.fill(m * k, p.seed, "a"), m, k).astype(np.float64)
    b = _colmajor(orc.fill(k * n, p.seed, "b"), k, n).astype(np.float64)
    c64 = a @ b
    scale = np.abs(a) @ np.abs(b)
    return space, p, c64, scale


@pytest.mark.parametrize("cfg", TC_4096,
                         ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items() if k not in ("staging",))
                         + "-" + c["staging"])
def test_tcgen05_4096_readback(dev, tc_4096_ref, cfg):
    space, p, c64, scale = tc_4096_ref
    dev.bind(p)
    tol = 4e-3 if cfg["engine"] == "TF32" else 1e-5
    t = _configured(space, **dict(cfg))
    m = dev.evaluate_tiles(t, reps=1, warmup=0)
    assert m.status == "ok" and m.mismatches == 0, (t.as_dict(), m, dev.error())
    got = _colmajor(dev.read("c", 4096 * 4096), 4096, 4096).astype(np.float64)
    err = np.abs(got - c64) / np.maximum(scale, 1e-30)
    assert np.isfinite(got).all()
    assert err.max() <= tol, (t.as_dict(), float(err.max()))
