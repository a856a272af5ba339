"""amm, attention and metrics modules of the fp64 oracle against the SPEC's
examples, its invariants and the ten acceptance criteria
(SPEC.md:499-508), at desk scale. This is what makes the oracle trustworthy as
the GPU path's checker (the reference ships no tests or fixtures)."""
import json
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------- amm
def test_optimal_probs_examples(orc):
    np.testing.assert_array_equal(orc.optimal_probs(np.eye(2), np.eye(2)).probs, [0.5, 0.5])
    a = np.array([[1.0, 0.0], [0.0, 1.0]])                                       # col norms [1, 1]
    b = np.array([[3.0, 0.0], [0.0, 1.0]])                                       # row norms [3, 1]
    np.testing.assert_allclose(orc.optimal_probs(a, b).probs, [0.75, 0.25], atol=1e-16)  # :198
    b0 = np.array([[1.0, 2.0], [0.0, 0.0]])
    assert orc.optimal_probs(np.eye(2), b0).probs[1] == 0.0                      # :199
    with pytest.raises(orc.OracleDegenerateError):
        orc.optimal_probs(np.zeros((2, 2)), np.eye(2))                            # :195


def test_weight_probs_examples(orc):
    d = 6
    np.testing.assert_allclose(orc.weight_probs(np.eye(d)).probs, [1 / d] * d, atol=1e-16)
    np.testing.assert_allclose(orc.weight_probs([[3, 0], [0, 4]]).probs, [9 / 25, 16 / 25], atol=1e-16)  # :208
    p = orc.weight_probs([[1, 1], [0, 0], [2, 0]]).probs                          # :209
    np.testing.assert_allclose(p, [2 / 6, 0, 4 / 6], atol=1e-16)
    with pytest.raises(orc.OracleDegenerateError):
        orc.weight_probs(np.zeros((3, 3)))                                        # :205


def test_approx_matmul_point_mass(orc):
    a = np.arange(6.0).reshape(2, 3)
    b = np.zeros((3, 2))
    b[1] = [2.0, -3.0]
    dist = orc.make_distribution([0, 1, 0])
    assert np.array_equal(orc.approx_matmul(a, b, dist, 1, seed=1), a @ b)
    # r > 1: exact "up to scaling arithmetic" (r terms of 1/(r p) each)
    np.testing.assert_allclose(orc.approx_matmul(a, b, dist, 5, seed=5), a @ b, rtol=1e-15, atol=0)


def test_approx_matmul_enumeration(orc):
    # 1x2 a, 2x1 b, probs [0.5, 0.5], r=1: the two outcomes average to the exact product
    a, b = np.array([[1.5, -2.0]]), np.array([[4.0], [0.5]])
    dist = orc.make_distribution([1, 1])
    outcomes = set()
    for s in range(64):
        outcomes.add(float(orc.approx_matmul(a, b, dist, 1, seed=s)[0, 0]))
    assert outcomes == {2 * 1.5 * 4.0, 2 * -2.0 * 0.5}
    assert np.mean(list(outcomes)) == (a @ b)[0, 0]


def test_approx_matmul_rejects_zero_prob_contributor(orc):
    with pytest.raises(orc.OracleDegenerateError):
        orc.approx_matmul(np.eye(2), np.eye(2), orc.make_distribution([1, 0]), 3, seed=1)


def test_approx_encode_row_examples(orc):
    rng = np.random.default_rng(4)
    w = rng.standard_normal((5, 3))
    e = np.zeros(5)
    e[2] = 1.0
    dist = orc.make_distribution([0, 0, 1, 0, 0])
    assert np.array_equal(orc.approx_encode_row(e, w, dist, 1, 1, 0), w[2])
    np.testing.assert_allclose(orc.approx_encode_row(e, w, dist, 9, 1, 0), w[2], rtol=1e-15, atol=0)
    dist = orc.weight_probs(w)
    assert np.array_equal(orc.approx_encode_row(np.zeros(5), w, dist, 7, 1, 0), np.zeros(3))  # :228


def test_criterion2_unbiasedness(orc):
    assert orc.verify_unbiased(100_000) >= 0.95


def test_criterion3_lemma1(orc):
    assert orc.verify_lemma1(fixtures=10, trials=10_000) <= 1.0


def test_criterion4_error_scaling_slope(orc):
    assert -0.6 <= orc.verify_scaling(trials=4_000) <= -0.4


# --------------------------------------------------------------- attention
def test_attention_matrix_examples(orc):
    rng = np.random.default_rng(5)
    wq, wk = rng.standard_normal((4, 4)), rng.standard_normal((4, 4))
    a = orc.attention_matrix(np.zeros((5, 4)), wq, wk)
    assert np.array_equal(a, np.full((5, 5), 0.2))
    assert orc.attention_matrix(rng.standard_normal((1, 4)), wq, wk)[0, 0] == 1.0  # :293
    x = rng.standard_normal((3, 4))                                                # :294
    s = (x @ wq) @ (x @ wk).T / 2.0
    ref = np.exp(s - s.max(axis=1, keepdims=True))
    ref /= ref.sum(axis=1, keepdims=True)
    np.testing.assert_allclose(orc.attention_matrix(x, wq, wk), ref, rtol=0, atol=1e-12)


def test_sample_budgets_examples(orc):
    n = 16
    b, e = orc.sample_budgets(np.full((n, n), 1.0 / n), alpha=1.0, d=64)          # SPEC.md:302 (n power of 2)
    assert np.all(b == 1) and not e.any()
    attn = np.full((4, 4), 0.5 / 3)
    np.fill_diagonal(attn, 0.5)                                                   # column max 0.5
    b, e = orc.sample_budgets(attn, alpha=0.2, d=64)                              # :303 raw = 100 >= 64
    assert np.all(b == 64) and e.all()
    b, e = orc.sample_budgets(attn, alpha=0.2, d=1024)
    assert np.all(b == 100) and not e.any()


def test_criterion7_budget_formula(orc):
    """Eq. 9 on crafted attention matrices: uniform, one-hot,
    clamped; α-halving quadruples the unclamped raw budgets exactly."""
    with open(os.path.join(GOLDEN, "budgets.json")) as f:
        for c in json.load(f)["cases"]:
            assert orc.budget_for(c["cmax"], c["n"], c["alpha"], c["min_samples"], c["d"]) == (c["r"], c["exact"])
    one_hot = np.zeros((8, 8))
    one_hot[:, 3] = 1.0
    b, e = orc.sample_budgets(one_hot, alpha=0.5, d=128)
    assert e[3] and b[3] == 128 and np.all(b[np.arange(8) != 3] == 1)
    # α halving quadruples raw exactly; with integer raw the budgets quadruple too
    cm = np.array([1 / 64, 3 / 128, 1 / 32, 5 / 128])  # integer raw at both alphas
    b1, _ = orc.sample_budgets_from_cmax(cm, 64, 0.5, 1, 10_000)
    b2, _ = orc.sample_budgets_from_cmax(cm, 64, 0.25, 1, 10_000)
    assert np.array_equal(b2, 4 * b1)


def test_budget_monotonicity(orc):
    rng = np.random.default_rng(9)
    cm = np.sort(rng.uniform(0, 0.3, 200))
    prev = None
    for alpha in (0.1, 0.2, 0.4, 0.8, 1.0):
        b, _ = orc.sample_budgets_from_cmax(cm, 128, alpha, 1, 768)
        assert np.all(np.diff(b) >= 0)                                            # non-decreasing in col_max
        if prev is not None:
            assert np.all(b <= prev)                                              # non-increasing in alpha
        prev = b


def _weights(rng, d, dq=None, dout=None):
    dq = dq or d
    dout = dout or d
    return rng.standard_normal((d, dq)), rng.standard_normal((d, dq)), rng.standard_normal((d, dout)) * 0.1


def test_mca_forward_exact_clamp_equals_regular(orc):
    rng = np.random.default_rng(10)
    x = rng.standard_normal((6, 8))
    wq, wk, w = _weights(rng, 8)
    approx = orc.forward(x, wq, wk, w, alpha=1e-6, seed=3)
    exact = orc.forward(x, wq, wk, w, mode="regular")
    assert approx.exact.all()
    np.testing.assert_allclose(approx.y, exact.y, rtol=0, atol=1e-10)


def test_mca_forward_n1_unbiased(orc):
    rng = np.random.default_rng(11)
    x = rng.standard_normal((1, 5))
    wq, wk, w = _weights(rng, 5)
    exact = x @ w
    ys = np.array([orc.forward(x, wq, wk, w, alpha=1.0, seed=s).y[0] for s in range(20_000)])
    se = ys.std(axis=0) / math.sqrt(len(ys))
    assert np.all(np.abs(ys.mean(axis=0) - exact[0]) <= 3.5 * se)


def test_mca_forward_theorem1_small_fixture(orc):
    rng = np.random.default_rng(12)
    x = rng.standard_normal((6, 8))
    wq, wk, w = _weights(rng, 8)
    y = orc.forward(x, wq, wk, w, mode="regular").y
    beta = np.mean(np.linalg.norm(x, axis=1))
    bound = 0.5 * beta * np.linalg.norm(w)
    errs = np.array([np.linalg.norm(orc.forward(x, wq, wk, w, alpha=0.5, seed=s).y - y, axis=1)
                     for s in range(2_000)])
    assert np.all(errs.mean(axis=0) <= bound)


def test_mca_forward_determinism_and_draws(orc):
    rng = np.random.default_rng(13)
    x = rng.standard_normal((10, 12))
    wq, wk, w = _weights(rng, 12)
    a = orc.forward(x, wq, wk, w, alpha=0.6, seed=99)
    b = orc.forward(x, wq, wk, w, alpha=0.6, seed=99)
    assert np.array_equal(a.y, b.y) and np.array_equal(a.draws, b.draws)
    dist = orc.weight_probs(w)
    for j in range(10):                                                           # SamplePlan.draws == the drawn indices
        if not a.exact[j]:
            assert np.array_equal(a.draws[j, : a.budgets[j]], orc.draw_indices(dist, int(a.budgets[j]), 99, j))


def test_mca_forward_requires_approx_mode_and_valid_alpha(orc):
    rng = np.random.default_rng(14)
    x = rng.standard_normal((4, 4))
    wq, wk, w = _weights(rng, 4)
    with pytest.raises(orc.OracleDomainError):
        orc.forward(x, wq, wk, w, alpha=0.0)
    with pytest.raises(orc.OracleDegenerateError):
        orc.forward(x, wq, wk, np.zeros((4, 4)), alpha=0.5)


def test_regular_forward_examples(orc):
    rng = np.random.default_rng(15)
    wq, wk, w = _weights(rng, 4)
    assert np.array_equal(orc.forward(np.zeros((3, 4)), wq, wk, w, mode="regular").y, np.zeros((3, 4)))  # :322
    y = orc.forward([[2.0]], [[1.0]], [[1.0]], [[3.0]], mode="regular").y        # :323 d=1, n=1 -> A=1, y=x w
    assert y[0, 0] == 6.0


def test_criterion1_exactness(orc):
    assert orc.verify_exactness(20) <= 1e-12


def test_multihead_examples(orc):
    rng = np.random.default_rng(16)
    n, d = 5, 8
    x = rng.standard_normal((n, d))
    wq, wk, w = _weights(rng, d)
    one = orc.multihead_forward(x, wq[None], wk[None], w[None], heads=1, alpha=0.5, seed=4)
    ref = orc.forward(x, wq, wk, w, alpha=0.5, seed=4)
    assert np.array_equal(one.y, ref.y)
    # heads = 2, regular mode == blockwise concatenation
    dh = d // 2
    WQ, WK = rng.standard_normal((2, d, dh)), rng.standard_normal((2, d, dh))
    W = rng.standard_normal((2, d, dh))
    two = orc.multihead_forward(x, WQ, WK, W, heads=2, mode="regular")
    for h in range(2):
        blk = orc.forward(x, WQ[h], WK[h], W[h], mode="regular").y
        np.testing.assert_allclose(two.y[:, h * dh:(h + 1) * dh], blk, rtol=0, atol=1e-12)
    # identical heads draw from independent streams
    same = orc.multihead_forward(x, np.stack([WQ[0]] * 2), np.stack([WK[0]] * 2), np.stack([W[0]] * 2),
                                 heads=2, alpha=1.0, seed=8)
    assert not np.array_equal(same.y[:, :dh], same.y[:, dh:])
    with pytest.raises(orc.OracleConfigError):
        orc.multihead_forward(rng.standard_normal((n, 7)), WQ, WK, W, heads=2)


def test_criteria5_6_theorem1_bounds(orc):
    """Theorem 1 mean bound (every row) and Markov tail at δ = 0.1, n=16, d=128,
    10^4 trials, α ∈ {0.2, 0.4, 0.6, 1.0}."""
    errs = []
    for alpha in (0.2, 0.4, 0.6, 1.0):
        worst_mean, worst_tail, mean_err = orc.verify_theorem1(alpha, n=16, d=128, trials=10_000)
        assert worst_mean <= 1.0
        assert worst_tail <= 0.12
        errs.append(mean_err)
    assert errs[0] < errs[2] < errs[3]                                            # criterion 10


def test_cancellation_identity(orc):
    rng = np.random.default_rng(17)
    x = rng.standard_normal((20, 16))
    wq, wk, _ = _weights(rng, 16)
    a = orc.attention_matrix(x, wq, wk)
    assert np.all(a / a.max(axis=0, keepdims=True) <= 1.0)


# ----------------------------------------------------------------- metrics
def test_flops_examples(orc):
    n, d = 10, 768
    f = orc.flops_for_plan([d] * n, [1] * n, d)
    assert f.reduction_factor == 1.0
    f = orc.flops_for_plan([96] * n, [0] * n, d)                                  # :391
    assert f.reduction_factor == pytest.approx(2 * 768**2 / (96 * (2 * 768 + 3)))
    assert round(f.reduction_factor, 2) == 7.98
    f = orc.flops_for_plan([1] * n, [0] * n, 4096)                                # :392
    assert f.reduction_factor == pytest.approx(2 * 4096**2 / (2 * 4096 + 3))


def test_criterion8_flops_mechanics(orc):
    d = 128
    n = 16
    uni = np.full((n, n), 1.0 / n)
    assert orc.predicted_reduction(uni, 1.0, d) == pytest.approx(2 * d * d / (2 * d + 3), abs=1e-9)
    peaked = np.full((n, n), 0.02 / (n - 1))
    peaked[:, 0] = 0.98
    peaked_n = peaked / peaked.sum(axis=1, keepdims=True)
    moderate = np.full((n, n), 1.0 / n) + np.random.default_rng(0).uniform(0, 0.05, (n, n))
    moderate /= moderate.sum(axis=1, keepdims=True)
    assert orc.predicted_reduction(peaked_n, 0.4, d) > orc.predicted_reduction(moderate, 0.4, d)  # :402
    # the instrumented plan counter equals the model on random plans
    rng = np.random.default_rng(1)
    for _ in range(20):
        b = rng.integers(1, d + 1, 33)
        e = b == d
        f = orc.flops_for_plan(b, e, d)
        assert f.approx_encoding == sum(2 * d * d if ee else int(bb) * (2 * d + 3) for bb, ee in zip(b, e))


def test_predicted_matches_forward(orc):
    rng = np.random.default_rng(18)
    x = rng.standard_normal((12, 16))
    wq, wk, w = _weights(rng, 16)
    out = orc.forward(x, wq, wk, w, alpha=0.4, seed=1)
    a = orc.attention_matrix(x, wq, wk)
    assert orc.predicted_reduction(a, 0.4, 16) == out.flops.reduction_factor


# ------------------------------------------------------ batched / criterion 9
def test_batched_forward_matches_multihead(orc):
    """The device-layout forward (b=0, Q/K given) equals SPEC multihead_forward
    with per-head slices W_h = W_V[:, h-slice]."""
    rng = np.random.default_rng(19)
    n, d, H = 9, 12, 3
    dh = d // H
    x = rng.standard_normal((n, d))
    WQ, WK, W = (rng.standard_normal((H, d, dh)) for _ in range(3))
    ref = orc.multihead_forward(x, WQ, WK, W, heads=H, alpha=0.3, seed=5)
    q = np.concatenate([x @ WQ[h] for h in range(H)], axis=1)[None]
    k = np.concatenate([x @ WK[h] for h in range(H)], axis=1)[None]
    wv = np.concatenate([W[h] for h in range(H)], axis=1)
    got = orc.batched_forward(q, k, x[None], wv, heads=H, alpha=0.3, seed=5)
    assert np.array_equal(got.budgets[0], ref.budgets)
    np.testing.assert_allclose(got.y[0], ref.y, rtol=0, atol=1e-12)


def test_criterion9_thread_count_invariance(orc):
    rng = np.random.default_rng(20)
    B, n, H, dh, d_in = 3, 24, 4, 8, 32
    q, k = rng.standard_normal((B, n, H * dh)), rng.standard_normal((B, n, H * dh))
    x, w = rng.standard_normal((B, n, d_in)), rng.standard_normal((d_in, H * dh))
    a = orc.batched_forward(q, k, x, w, heads=H, alpha=0.4, seed=3, threads=1)
    b = orc.batched_forward(q, k, x, w, heads=H, alpha=0.4, seed=3, threads=8)
    assert np.array_equal(a.y, b.y) and np.array_equal(a.budgets, b.budgets)
    orc.set_threads(os.cpu_count() or 1)


def test_batched_shard_invariance(orc):
    """Sharding the batch (b_offset) gives bitwise the same result as one call:
    the multi-GPU contract of DESIGN.md §6 restated on the oracle."""
    rng = np.random.default_rng(21)
    B, n, H, dh, d_in = 4, 16, 2, 8, 16
    q, k = rng.standard_normal((B, n, H * dh)), rng.standard_normal((B, n, H * dh))
    x, w = rng.standard_normal((B, n, d_in)), rng.standard_normal((d_in, H * dh))
    full = orc.batched_forward(q, k, x, w, heads=H, alpha=0.4, seed=3)
    for s in range(0, B, 2):
        part = orc.batched_forward(q[s:s + 2], k[s:s + 2], x[s:s + 2], w, heads=H, alpha=0.4, seed=3, b_offset=s)
        assert np.array_equal(part.y, full.y[s:s + 2])


def test_golden_forward(orc):
    with open(os.path.join(GOLDEN, "forward_small.json")) as f:
        g = json.load(f)
    res = orc.batched_forward(np.array(g["q"]), np.array(g["k"]), np.array(g["x"]), np.array(g["w"]),
                              heads=g["H"], alpha=g["alpha"], seed=g["seed"])
    assert res.budgets.tolist() == g["budgets"]
    assert res.exact.astype(int).tolist() == g["exact"]
    np.testing.assert_allclose(res.y, np.array(g["y"]), rtol=1e-12, atol=1e-12)
    assert [res.flops.exact_encoding, res.flops.approx_encoding, res.flops.aggregation] == g["flops"]
