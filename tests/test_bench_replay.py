"""bench.py replays every logged mismatch / launch error on the CPU emulator
against the golden outputs (a device stub here: CPU only)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1904_03383_b200 as P  # noqa: E402
from paper_1904_03383_b200 import Space  # noqa: E402
from tests.oracle_lib import Oracle  # noqa: E402


def _leaf(space):
    c = space.root()
    for a, b in [("load_x", "mul"), ("mul", "add"), ("load_y", "add"), ("add", "store_z")]:
        for lvl in ("_n_r", "_n0", "_n1"):
            c.decide("order", [a + lvl, b + lvl], "MERGED")
    c.decide("dim_kind", ["load_x_n_r"], "BLOCK")
    c.decide("dim_kind", ["load_x_n0"], "VECTOR")
    c.decide("dim_kind", ["load_x_n1"], "THREAD")
    return c.first_leaf()


def test_replay_verdicts(tmp_path, monkeypatch):
    space = Space("axpy", n=1 << 12, factors=[[4], [64]])
    leaf = _leaf(space)
    orc = Oracle()
    p = space.problem()
    x, y = orc.fill(p.n, p.seed, "x"), orc.fill(p.n, p.seed, "y")
    z = orc.axpy(x, y, p.alpha)
    log = tmp_path / "search.jsonl"
    log.write_text(json.dumps({"i": 7, "status": "mismatch", "hash": "h", "candidate": json.loads(leaf.serialize())})
                   + "\n" + json.dumps({"i": 8, "status": "ok"}) + "\n")
    for golden, verdict in ((z, "emulator agrees"), (np.zeros_like(z), "emulator differs")):
        class StubDevice:
            def __init__(self, ordinal):
                pass

            def bind(self, problem):
                pass

            def read(self, name, n, expected=False, golden=golden):
                if expected and name != "z":
                    raise RuntimeError("not an output")
                return {"x": x, "y": y, "z": golden}[name][:n].copy()

            def close(self):
                pass

        monkeypatch.setattr(P, "Device", StubDevice)
        out = bench.replay_failures(str(log), space, 0)
        assert len(out) == 1 and out[0]["i"] == 7 and out[0]["verdict"].startswith(verdict), out


def test_config_mismatch_replayed_at_a_small_shape(tmp_path):
    """A mismatch the reference's matmul 1024^3 space produced on the B200
    (tests/golden/matmul_invalid_schedule.json: the accumulator initialised
    inside the k loop, the staged temporary read before it is written) is
    re-decided at 128^3 and run on the emulator against the CPU oracle: the
    schedule itself computes other values ("emulator differs")."""
    rec = json.load(open(os.path.join(ROOT, "tests", "golden", "matmul_invalid_schedule.json")))["record"]
    kw = dict(m=1024, n=1024, k=1024, factors=[[2, 4, 8, 16, 32], [2, 4]])
    log = tmp_path / "config_matmul.jsonl"
    log.write_text(json.dumps(rec) + "\n" + json.dumps({"i": 9, "status": "ok"}) + "\n")
    out = bench.replay_scaled(str(log), "matmul", kw)
    assert len(out) == 1 and out[0]["i"] == rec["i"] and out[0]["replayed_at"] == 128
    assert out[0]["verdict"].startswith("emulator differs"), out
    assert out[0]["emulator_mismatches"] > 0
