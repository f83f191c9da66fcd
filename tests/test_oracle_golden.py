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
