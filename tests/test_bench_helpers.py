"""bench.py's host-side helpers on CPU: the per-stage algorithmic work
(SURVEY.md §8(d)), the roofline / floor table, and the batch sharding of the
strong-scaling mode."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_stage_work_c2(bench):
    w = bench.stage_work(64, 512, 768, 12, 2, True, 23_959_230)
    assert w["score"] == ("tensor", pytest.approx(25.77e9, rel=1e-3))          # 2 B H n^2 64
    assert w["apply"][1] == w["score"][1]
    assert w["projection"] == ("tensor", pytest.approx(77.3e9, rel=1e-3))      # 2 * 2 B n d H 64
    assert w["encode"] == ("hbm", pytest.approx(103.5e6, rel=2e-3))            # 103.5 MB at C2
    assert bench.stage_work(64, 512, 768, 12, 2, False, 0)["projection"][1] == 0.0


def test_kernel_table(bench):
    w = bench.stage_work(64, 512, 768, 12, 2, True, 23_959_230)
    ms = {"projection": 0.06, "score": 0.11, "budgets": 0.015, "encode": 0.2, "apply": 0.09}
    peaks = {"hbm_gbs": 6560.6, "bf16_tflops": 1622.3}
    t = bench.kernel_table(w, ms, peaks, 1965.0)
    assert set(t) == set(ms)
    assert t["encode"]["bound"] == "hbm" and t["encode"]["frac"] == pytest.approx(103.5e6 / 0.2e-3 / 1e9 / 6560.6,
                                                                                 rel=2e-3)
    assert 0 < t["encode"]["frac_of_smem_floor"] < 1 and 0 < t["encode"]["frac_of_fma_floor"] < 1
    assert t["score"]["mufu_floor_ms"] == pytest.approx(64 * 12 * 512 * 512 / (148 * 16 * 1.965e9) * 1e3)
    assert t["apply"]["mufu_floor_ms"] == pytest.approx(t["score"]["mufu_floor_ms"] / 2)
    assert t["projection"]["unit"] == "TFLOP/s"


def test_shard_modes(bench):
    class A:
        config = "c3"
        global_batch = 128
    for world in (1, 2, 4, 8):
        parts = [bench._shard(A, r, world) for r in range(world)]
        assert sum(p[0] for p in parts) == 128 and all(p[3] == "strong" for p in parts)
        assert [p[1] for p in parts] == [sum(q[0] for q in parts[:r]) for r in range(world)]
    A.config, A.global_batch = "c2", 0
    assert bench._shard(A, 3, 8) == (64, 192, 512, "weak")
