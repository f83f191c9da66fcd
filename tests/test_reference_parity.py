"""Search-side parity with the reference (bit-exact counts): the host library
links the reference's search-space engine unchanged, so instance counts, root
facts, leaf counts, simulated costs and pseudo-sources must be the reference's
own known answers (nest_test.cpp, gpu_space_test.cpp, and the
survey's probes of the BASELINE spaces). Also proves the flat C-ABI nest
(ispc_nest) carries the whole schedule: the backend's pseudo-source rendering
of the flat nest equals the reference's emit_source() byte for byte."""
import pytest

from paper_1904_03383_b200 import DeadEnd, Space

AXPY_FACTORS = [[2, 4], [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]]
MM_FACTORS = [[2, 4, 8, 16, 32], [2, 4]]


def test_axpy_baseline_space_counts():
    """SURVEY.md 6 [probe]: axpy 2^26 with the paper factors."""
    s = Space("axpy", n=1 << 26, factors=AXPY_FACTORS).stats()
    assert (s["instances"], s["enum_instances"], s["int_instances"], s["counter_instances"]) == (690, 676, 10, 4)
    assert s["root_open"] == 337
    assert s["objects"] == 52 and s["lowerings"] == 4


def test_matmul_baseline_space_counts():
    """SURVEY.md 6 [probe]: matmul 1024^3 with {2..32} x {2,4}."""
    s = Space("matmul", m=1024, n=1024, k=1024, factors=MM_FACTORS).stats()
    assert (s["instances"], s["enum_instances"], s["int_instances"], s["counter_instances"]) == (1359, 1339, 16, 4)
    assert s["root_open"] == 795


def test_outer_product_leaf_count():
    """nest_test.cpp:318: 768 leaves of outer_product(2, 2)."""
    s = Space("outer_product", m=2, n=2)
    assert s.root().count_leaves() == 768


def _vector_axpy():
    s = Space("axpy", n=8, factors=[[4]])
    c = s.root()
    for a, b in [("load_x_n0", "mul_n0"), ("load_x_n_r", "mul_n_r"), ("mul_n0", "add_n0"), ("mul_n_r", "add_n_r"),
                 ("load_y_n0", "add_n0"), ("load_y_n_r", "add_n_r"), ("add_n0", "store_z_n0"),
                 ("add_n_r", "store_z_n_r")]:
        c.decide("order", [a, b], "MERGED")
    c.decide("dim_kind", ["load_x_n0"], "VECTOR")
    c.decide("dim_kind", ["load_x_n_r"], "LOOP")
    c.decide("order", ["load_x_n_r", "load_x_n0"], "OUTER")
    return s, c.first_leaf()


def test_vector_axpy_known_answer():
    """nest_test.cpp:447-482: compute 8, memory 24, total 24, nothing fired."""
    _, leaf = _vector_axpy()
    assert leaf.fired == 0
    r = leaf.simulate()
    assert (r["compute"], r["memory"], r["total"]) == (8, 24, 24)
    src = leaf.reference_source()
    assert "vec" in src and ".v4" in src


@pytest.mark.parametrize("spec", [
    dict(kind="axpy", n=64, factors=[[2, 4], [2, 4, 8]]),
    dict(kind="outer_product", m=4, n=4),
    dict(kind="matmul", m=8, n=8, k=8, factors=[[2, 4]]),
    dict(kind="matmul", m=8, n=4, k=4, factors=[[2]], a_stride=3),
], ids=lambda s: s["kind"])
def test_flat_nest_renders_reference_source(spec):
    space = Space(**spec)
    root = space.root()
    seen = 0
    for seed in range(25):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        assert leaf.nest().pseudo() == leaf.reference_source()
        seen += 1
    assert seen >= 10


def test_bound_is_admissible_on_leaves_and_monotone():
    """B200 bound (seconds): a child's bound never drops below its parent's."""
    space = Space("axpy", n=1 << 20, factors=[[2, 4], [32, 64, 128, 256]])
    root = space.root()
    b_root = root.bound()["total"]
    for seed in range(10):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        assert leaf.bound()["total"] >= b_root * (1 - 1e-12)


def test_serialization_round_trip_keeps_digest():
    space = Space("matmul", m=8, n=8, k=8, factors=[[2, 4]])
    leaf, _, _ = space.root().random_leaf(3)
    again = space.deserialize(leaf.serialize())
    assert again.digest == leaf.digest and again.fully_specified


def test_knuth_estimate_matches_exact_count():
    """Knuth's estimator over the same first-open tree count_leaves walks."""
    s = Space("outer_product", m=2, n=2)
    est = s.root().estimate_tree(20000, seed=3)
    assert abs(est["leaves"] - 768) <= 4 * est["leaves_stderr"] + 1e-9
    assert est["dead_probe_ratio"] == 0.0


def test_b200_mode_admits_shared_staging_the_parity_machine_cannot():
    """machine_for(ISPC_SPACE_B200) raises shared_capacity to 227 KiB: at
    axpy n = 16384 (64 KiB temporaries) no parity-mode leaf stages in shared
    memory, most B200-mode leaves do; both spaces keep the reference's
    instance table (same choices, same counts)."""
    from paper_1904_03383_b200 import DeadEnd, EmitError
    from paper_1904_03383_b200 import _native as N
    counts = {}
    for mode in (N.SPACE_PARITY, N.SPACE_B200):
        s = Space("axpy", n=16384, factors=[[4], [64]], mode=mode)
        assert s.stats()["instances"] == Space("axpy", n=16384, factors=[[4], [64]]).stats()["instances"]
        shared = total = 0
        for seed in range(1, 300):
            try:
                leaf, _, _ = s.root().random_leaf(seed)
                src, _ = leaf.nest().cuda()
            except (DeadEnd, EmitError, ValueError):
                continue
            total += 1
            shared += "__shared__" in src
        counts[mode] = (shared, total)
    assert counts[N.SPACE_PARITY][0] == 0 and counts[N.SPACE_PARITY][1] > 20
    assert counts[N.SPACE_B200][0] > counts[N.SPACE_B200][1] // 2


def test_order_decisions_round_trip_through_the_schedule_tree():
    """nest_test.cpp:309-334: for all 768 leaves of outer_product(2, 2),
    derive_orders(reconstruct(leaf)) yields 15 pairs, each the value of the
    leaf's order decision."""
    r = Space("outer_product", m=2, n=2).root().order_round_trip()
    assert r == {"leaves": 768, "pairs": 768 * 15, "mismatches": 0}


def test_threadidx_z_above_64_is_illegal():
    """The reference space holds schedules whose outermost of three thread
    levels has 128 or 256 threads; threadIdx.z is capped at 64, so the
    emitter rejects them (ISPC_E_ILLEGAL) instead of the launch failing with
    CUDA_ERROR_INVALID_VALUE (one such launch error in the r2u headline)."""
    import pytest

    from paper_1904_03383_b200 import EmitError
    sp = Space("axpy", n=1 << 26, factors=[[2, 4], [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]])
    leaf = sp.root().random_leaf(117)[0]
    with pytest.raises(EmitError, match="threadIdx.z"):
        leaf.nest().cuda("k")
