"""The CPU oracle (oracle/numeric.c) against golden vectors produced by
interpreting the reference's own Kernel backbones (oracle/ref_golden.cpp,
regenerate with `oracle/_ref/ref_golden tests/golden/backbone_outputs.json`)."""
import json
import os

import numpy as np
import pytest

from tests.oracle_lib import Oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "backbone_outputs.json")
DATA = json.load(open(GOLDEN))


class P:  # duck-typed ispc_problem
    def __init__(self, c):
        self.kind = {"axpy": 0, "outer_product": 1, "matmul": 2}[c["kind"]]
        self.m, self.n, self.k = c["m"], c["n"], c["k"]
        self.a_stride = c["a_stride"]
        self.batch = 1
        self.seed = DATA["seed"]
        self.alpha = DATA["alpha"]


@pytest.mark.parametrize("case", DATA["cases"], ids=lambda c: c["label"])
def test_oracle_matches_reference_backbone(case):
    got = Oracle().expected(P(case))[case["output"]]
    want = np.array(case["bits"], dtype=np.uint32)
    assert got.size == want.size
    assert np.array_equal(got.view(np.uint32), want)


def test_generator_is_exact_grid():
    v = Oracle().fill(1 << 16, 7, "x")
    assert v.min() >= -1.0 and v.max() < 1.0
    assert np.all(v * np.float32(2 ** 23) == np.round(v * np.float32(2 ** 23)))


@pytest.mark.parametrize("case", [c for c in DATA["cases"] if c["kind"] == "matmul" and c["n"] == 1],
                         ids=lambda c: c["label"])
def test_gemv_and_batched_oracles_match_reference_matmul(case):
    """gemv (no reference builder) is the reference matmul with n = 1, batched
    is independent matmuls: both oracle entry points reproduce its bits."""
    o = Oracle()
    p = P(case)
    m, k = case["m"], case["k"]
    a, x = o.fill(m * k, p.seed, "a"), o.fill(k, p.seed, "b")
    want = np.array(case["bits"], dtype=np.uint32)
    assert np.array_equal(o.gemv(a, x, m, k).view(np.uint32), want)
    two = o.batched(np.concatenate([a, a]), np.concatenate([x, x]), 2, m, 1, k)
    assert np.array_equal(two.view(np.uint32), np.concatenate([want, want]))
