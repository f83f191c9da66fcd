"""GPU parity: emitted sm_100a kernels against the CPU oracle (bit-exact for
the parity-mode FFMA/FMUL/FADD paths), through the C-ABI (libispc)."""
import numpy as np
import pytest

from paper_1904_03383_b200 import DeadEnd, Device, EmitError, Space
from tests import emu
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


SMALL_SPACES = [
    dict(kind="axpy", n=64, factors=[[2, 4], [2, 4, 8]]),
    dict(kind="axpy", n=1024, factors=[[4], [2, 8, 32]]),
    dict(kind="outer_product", m=4, n=3),
    dict(kind="outer_product", m=16, n=8),
    dict(kind="matmul", m=8, n=8, k=8, factors=[[2, 4]]),
    dict(kind="matmul", m=16, n=8, k=4, factors=[[2], [2, 4]]),
    dict(kind="matmul", m=8, n=4, k=4, factors=[[2]], a_stride=3),
]


@pytest.mark.parametrize("spec", SMALL_SPACES, ids=lambda s: "-".join(str(v) for v in s.values()))
def test_golden_kernels_match_oracle(dev, orc, spec):
    space = Space(**spec)
    p = space.problem()
    dev.bind(p)
    for name, ref in orc.expected(p).items():
        got = dev.read(name, ref.size, expected=True)
        assert np.array_equal(_bits(got), _bits(ref)), name


@pytest.mark.parametrize("spec", SMALL_SPACES, ids=lambda s: "-".join(str(v) for v in s.values()))
def test_random_leaves_bit_exact(dev, orc, spec):
    space = Space(**spec)
    p = space.problem()
    dev.bind(p)
    expected = orc.expected(p)
    root = space.root()
    counts = {"ok": 0, "illegal": 0}
    for seed in range(40):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        nest = leaf.nest()
        m = dev.evaluate(nest, reps=1, warmup=0, budget_ns=5e8)
        if m.status == "illegal":
            counts["illegal"] += 1
            continue
        if m.status == "timeout":
            # legal but hopelessly slow schedules (e.g. one thread walking
            # every loop sequentially): the device watchdog stopped them
            counts["timeout"] = counts.get("timeout", 0) + 1
            continue
        if m.status == "mismatch":
            # The reference space admits schedules whose value flow through a
            # temporary runs against a shared sequential loop (DESIGN.md
            # "invalid schedules"). Such a kernel must be wrong on the CPU
            # emulation too; a GPU-only mismatch would be an emitter bug.
            src, L = nest.cuda("k_emu")
            regs = _inputs(orc, p)
            try:
                emu.run(src, L, regs, p.alpha)
            except emu.TooLong:
                counts["unconfirmed"] = counts.get("unconfirmed", 0) + 1
                continue
            same = all(np.array_equal(_bits(regs[k]), _bits(v)) for k, v in expected.items())
            assert not same, (seed, "GPU-only mismatch", leaf.reference_source())
            counts["invalid"] = counts.get("invalid", 0) + 1
            continue
        assert m.status == "ok", (seed, m, dev.error(), leaf.reference_source())
        assert m.mismatches == 0
        for name, ref in expected.items():
            got = dev.read(name, ref.size)
            assert np.array_equal(_bits(got), _bits(ref)), (seed, name, leaf.reference_source())
        counts["ok"] += 1
    assert counts["ok"] >= 5, counts


def _inputs(orc, p):
    """Problem regions for the CPU emulation, outputs NaN-filled."""
    s = max(int(p.a_stride), 1)
    nan = lambda n: np.full(n, np.nan, dtype=np.float32)  # noqa: E731
    if p.kind == 0:
        return {"x": orc.fill(p.n, p.seed, "x"), "y": orc.fill(p.n, p.seed, "y"), "z": nan(p.n)}
    if p.kind == 1:
        return {"a": orc.fill(p.m, p.seed, "a"), "b": orc.fill(p.n, p.seed, "b"), "c": nan(p.m * p.n)}
    if p.kind == 2:
        return {"a": orc.fill(p.m * p.k * s, p.seed, "a"), "b": orc.fill(p.k * p.n, p.seed, "b"),
                "c": nan(p.m * p.n)}
    raise ValueError(p.kind)


def _fused_axpy(n, vec, threads):
    space = Space("axpy", n=n, factors=[[vec], [threads]])
    c = space.root()
    for a, b in [("load_x", "mul"), ("mul", "add"), ("load_y", "add"), ("add", "store_z")]:
        for lvl in ("_n_r", "_n0", "_n1"):
            c.decide("order", [a + lvl, b + lvl], "MERGED")
    c.decide("dim_kind", ["load_x_n_r"], "BLOCK")
    c.decide("dim_kind", ["load_x_n0"], "VECTOR")
    c.decide("dim_kind", ["load_x_n1"], "THREAD")
    for i in ("load_x", "load_y", "store_z"):
        c.decide("cache", [i], "NONE")
    return space, c.first_leaf()


def test_axpy_full_size_bit_exact(dev, orc):
    """BASELINE config 1 at full size (n = 2^26): a coalesced float4 schedule."""
    n = 1 << 26
    space, leaf = _fused_axpy(n, 4, 256)
    p = space.problem()
    dev.bind(p)
    m = dev.evaluate(leaf.nest(), reps=5)
    assert m.status == "ok" and m.mismatches == 0, (m, dev.error())
    z = dev.read("z", n)
    ref = orc.expected(p)["z"]
    assert np.array_equal(_bits(z), _bits(ref))
    gbs = 12.0 * n / m.median_ns
    assert gbs > 1000, gbs  # sanity: a coalesced stream on HBM3e


def test_matmul_scaled_fused_bit_exact(dev, orc):
    """The golden fused matmul schedule (nest_test.cpp:386) at 64^3."""
    space = Space("matmul", m=64, n=64, k=64, factors=[[4]])
    c = space.root()
    merges = [("load_a_m0", "mad_m0"), ("load_a_m_r", "mad_m_r"), ("load_a_k_r", "mad_k_r"),
              ("load_b_k_r", "mad_k_r"), ("load_b_n0", "mad_n0"), ("load_b_n_r", "mad_n_r"),
              ("init_c_m0", "mad_m0"), ("init_c_m_r", "mad_m_r"), ("init_c_n0", "mad_n0"),
              ("init_c_n_r", "mad_n_r"), ("mad_m0", "store_c_m0"), ("mad_m_r", "store_c_m_r"),
              ("mad_n0", "store_c_n0"), ("mad_n_r", "store_c_n_r")]
    for a, b in merges:
        c.decide("order", [a, b], "MERGED")
    c.decide("dim_kind", ["mad_m_r"], "BLOCK")
    c.decide("dim_kind", ["mad_n_r"], "BLOCK")
    c.decide("dim_kind", ["mad_n0"], "THREAD")
    c.decide("dim_kind", ["mad_m0"], "UNROLL")
    c.decide("order", ["mad_m_r", "mad_n_r"], "OUTER")
    c.decide("order", ["mad_n0", "mad_m0"], "OUTER")
    c.decide("order", ["mad_m0", "mad_k_r"], "OUTER")
    c.decide("order", ["init_c", "mad_k_r"], "BEFORE")
    c.decide("order", ["store_c", "mad_k_r"], "AFTER")
    leaf = c.first_leaf()
    p = space.problem()
    dev.bind(p)
    m = dev.evaluate(leaf.nest(), reps=3)
    assert m.status == "ok" and m.mismatches == 0, (m, dev.error())
    got = dev.read("c", 64 * 64)
    assert np.array_equal(_bits(got), _bits(orc.expected(p)["c"]))


def test_b200_mode_shared_staging_bit_exact(dev, orc):
    """B200 MachineParams mode (227 KiB of shared memory per block instead of
    the reference's 48 KiB, host_api.cpp machine_for): single-block axpy
    schedules whose 64 KiB temporaries live in shared memory run bit-exact."""
    from paper_1904_03383_b200 import _native as N
    space = Space("axpy", n=16384, factors=[[4], [64]], mode=N.SPACE_B200)
    dev.bind(space.problem())
    p = space.problem()
    ref = orc.axpy(orc.fill(p.n, p.seed, "x"), orc.fill(p.n, p.seed, "y"), p.alpha)
    ok = 0
    for seed in range(1, 300):
        try:
            leaf, _, _ = space.root().random_leaf(seed)
            nest = leaf.nest()
            src, _ = nest.cuda()
        except (DeadEnd, EmitError, ValueError):
            continue
        if "__shared__" not in src:
            continue
        m = dev.evaluate(nest, reps=1, warmup=0)
        if m.status == "timeout":
            continue
        assert m.status == "ok", (seed, m, dev.error())
        assert np.array_equal(_bits(dev.read("z", p.n)), _bits(ref)), seed
        ok += 1
        if ok == 4:
            break
    assert ok >= 2
