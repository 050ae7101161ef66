"""Pins of the float64 oracle against things other than itself (-m "not gpu").

Each pin is chosen so that a plausible mistake (dropped term, wrong sign, wrong
exponent row, transposed operand, wrong swap slot, mask leak) fails at least one:
  * paper-printed values (tests/golden/paper_values.json) and SPEC worked values
  * textbook closed forms of the named divergences
  * brute-force nested loops of eq:contraction_structure / eq:num
  * the hand-derived Lee-Seung NMF updates (P:235 cites lee2000algorithms)
  * calculus: dL/dy = (b - a)/alpha (from eq:prop at lambda = 1), checked by finite differences
  * Theorem 1 / Theorem 2 monotonicity after every factor update
  * fixed point of an exact factorization, mask invariance
"""
import itertools
import math

import numpy as np
import pytest

from oracle import nef_oracle as O

RNG = np.random.default_rng(12345)


# ------------------------------------------------------------------ parse / swap / count
def test_swap_examples(golden):
    for ex in golden["swap_examples"]:
        assert O.swap(ex["model"], ex["ell"]) == ex["value"], ex["cite"]


def test_swap_involution():
    for ms in ["ir,jr,kr->ijk", "ia,jb,kc,abc->ijk", "ik,jk,tl,dl,kl->ijtd", "wr,dr,hr,irk,jrk->wdhij"]:
        ops, _ = O.parse(ms)
        for ell in range(len(ops)):
            assert O.swap(O.swap(ms, ell), ell) == ms


@pytest.mark.parametrize("bad", ["ir,jr", "ir,,jr->ij", "ii,jr->ij", "ir,jr->ijz", "i1,jr->ij", "ir,jr->iij"])
def test_parse_errors(bad):
    with pytest.raises(ValueError):
        O.parse(bad)


def test_parse_classification():
    ops, out = O.parse("ij,jk,ik->ijk")
    assert ops == ["ij", "jk", "ik"] and out == "ijk"
    assert O.parse(" ir , jr -> ij ") == (["ir", "jr"], "ij")


def test_param_count_paper(golden):
    g = golden["uber_param_count"]
    assert O.param_count(g["model"], g["shape"], g["ranks"]) == g["value"], g["cite"]
    e = golden["uber_entries"]
    assert math.prod(e["shape"]) == e["value"]
    assert O.param_count("ir,jr->ij", (3, 4), (2,)) == 14
    assert O.param_count("ia,jb,kc,abc->ijk", (3, 4, 5), (2, 2, 2)) == 32


# ------------------------------------------------------------------ contraction
def test_contract_examples(golden):
    for ex in golden["contract_examples"]:
        got = O.contract(ex["model"], [np.array(o, dtype=float) for o in ex["ops"]])
        np.testing.assert_array_equal(got, np.array(ex["value"], dtype=float), err_msg=ex["cite"])


TINY_MODELS = [
    ("ir,jr,kr->ijk", (3, 4, 5), (2,)),
    ("ia,jb,kc,abc->ijk", (3, 2, 4), (2, 3, 2)),
    ("ik,jk,tl,dl,kl->ijtd", (2, 3, 2, 3), (2, 3)),
    ("iab,jbc,kca->ijk", (2, 3, 2), (2, 2, 3)),       # tensor-train ring-like
    ("ij,jk,ik->ijk", (2, 3, 4), ()),                   # many-body
    ("ir,jkr->ijk", (3, 2, 3), (2,)),                   # custom P:94
    ("i,jr,kr->ijk", (2, 3, 2), (3,)),                  # custom P:95
    ("ia,jb,kb,ab->ijk", (2, 3, 2), (2, 3)),            # custom P:96
    ("ir,jr,ak,kr,tr->ijat", (2, 2, 3, 2), (2, 2)),     # ICEWS custom P:296-300
]


def _rand_factors(ms, shape, ranks, lo=0.1, hi=1.0, rng=RNG):
    return [rng.uniform(lo, hi, size=s) for s in O.factor_shapes(ms, shape, ranks)]


@pytest.mark.parametrize("ms,shape,ranks", TINY_MODELS)
def test_contract_vs_bruteforce(ms, shape, ranks):
    f = _rand_factors(ms, shape, ranks)
    np.testing.assert_allclose(O.contract(ms, f), O.contract_bruteforce(ms, f), rtol=1e-12)


def test_cp_is_tucker_with_diagonal_core():
    A, B, C = (RNG.uniform(size=(n, 3)) for n in (4, 5, 6))
    core = np.zeros((3, 3, 3))
    for r in range(3):
        core[r, r, r] = 1.0
    np.testing.assert_allclose(O.contract("ir,jr,kr->ijk", [A, B, C]),
                               O.contract("ia,jb,kc,abc->ijk", [A, B, C, core]), rtol=1e-13)


def test_all_ones_factors():
    ms, shape, ranks = "ik,jk,tl,dl,kl->ijtd", (3, 2, 2, 4), (5, 7)
    f = [np.ones(s) for s in O.factor_shapes(ms, shape, ranks)]
    np.testing.assert_array_equal(O.contract(ms, f), np.full(shape, 35.0))


# ------------------------------------------------------------------ divergence closed forms
def _textbook(name, x, y):
    return {
        "KL": x * np.log(x / y) - x + y,
        "reverse_KL": y * np.log(y / x) - y + x,
        "squared_Euclidean": 0.5 * (x - y) ** 2,
        "Itakura_Saito": x / y - np.log(x / y) - 1.0,
        "squared_Hellinger": 2.0 * (np.sqrt(x) - np.sqrt(y)) ** 2,
        "Neyman_chi2": (x - y) ** 2 / (2.0 * x),
        "Pearson_chi2": (x - y) ** 2 / (2.0 * y),
    }[name]


def test_named_divergences(golden):
    # own generator: the draws must not depend on which tests ran before (xdist order).
    # atol: near x == y both sides are differences of O(1) terms that cancel to ~1e-3, so
    # fp64 rounding of the general (alpha, beta) form leaves ~1e-15 absolute there.
    rng = np.random.default_rng(123)
    x = rng.uniform(0.1, 10, 200)
    y = rng.uniform(0.1, 10, 200)
    for name, ab in golden["named_divergences"].items():
        if name.startswith("_"):
            continue
        a, b = ab
        np.testing.assert_allclose(O.divergence(x, y, a, b), _textbook(name, x, y), rtol=1e-11,
                                   atol=1e-13, err_msg=name)


def test_worked_values(golden):
    for ex in golden["worked_losses"]:
        assert O.divergence(ex["x"], ex["y"], ex["alpha"], ex["beta"]) == pytest.approx(ex["value"], rel=1e-14)
    for ex in golden["worked_ab"]:
        assert O.a_fn(ex["x"], ex["y"], ex["alpha"], ex["beta"]) == pytest.approx(ex["a"])
        assert O.b_fn(ex["x"], ex["y"], ex["alpha"], ex["beta"]) == pytest.approx(ex["b"])


AB_GRID = [(1, 0), (1, 1), (1, -1), (0.5, 0.5), (2, -1), (-1, 2), (0.5, 0), (1, -0.5), (1, 0.5), (1, 2),
           (0.5, 1), (0.7, 0), (1.3, 1), (1.2, 0.3), (0, 1), (0.8, -0.8), (1.3, 0)]


@pytest.mark.parametrize("ab", AB_GRID + [(0, 0)])
def test_divergence_zero_at_equal(ab):
    x = RNG.uniform(0.1, 10, 50)
    np.testing.assert_allclose(O.divergence(x, x, *ab), 0.0, atol=1e-12)
    y = x * RNG.uniform(1.1, 2.0, 50)
    assert np.all(O.divergence(x, y, *ab) > 0)


def test_divergence_continuity():
    x = RNG.uniform(0.1, 10, 50)
    y = RNG.uniform(0.1, 10, 50)
    # generic case near a special case: truncation O(delta), cancellation O(1e-16/delta)
    d, kw = 1e-6, dict(rtol=1e-4, atol=1e-5)
    for a in (0.5, 1.0, 1.7):
        np.testing.assert_allclose(O.divergence(x, y, a, d), O.divergence(x, y, a, 0.0), **kw)
        np.testing.assert_allclose(O.divergence(x, y, a, -a + d), O.divergence(x, y, a, -a), **kw)
    for b in (0.5, 1.0):
        np.testing.assert_allclose(O.divergence(x, y, d, b), O.divergence(x, y, 0.0, b), **kw)
    np.testing.assert_allclose(O.divergence(x, y, 1e-4, -1e-4 + 1e-6), O.divergence(x, y, 0.0, 0.0),
                               rtol=2e-2, atol=1e-3)


@pytest.mark.parametrize("ab", AB_GRID)
def test_dldy_equals_b_minus_a(ab):
    """eq:prop at lambda = 1: dL/dy = c(1)[g(1) b - a]; with the P:531-539 table this is
    (b - a)/alpha for alpha != 0 and -a for (0, 1).  Central finite differences."""
    alpha, beta = ab
    x = RNG.uniform(0.2, 5, 40)
    y = RNG.uniform(0.2, 5, 40)
    h = 1e-6 * y
    fd = (O.divergence(x, y + h, alpha, beta) - O.divergence(x, y - h, alpha, beta)) / (2 * h)
    a = O.a_fn(x, y, alpha, beta)
    b = O.b_fn(x, y, alpha, beta)
    want = -a if alpha == 0 else (b - a) / alpha
    np.testing.assert_allclose(fd, want, rtol=2e-6, atol=1e-9)


def test_a_b_zero_data():
    # x = 0 with alpha > 0: a = 0, b = y^(alpha+beta-1)
    assert O.a_fn(0.0, 2.0, 0.5, 0.0) == 0.0
    assert O.b_fn(0.0, 4.0, 0.5, 0.0) == pytest.approx(0.5)
    # 0 log 0 = 0 in the beta = 0 case: L(0, y) = y^alpha / alpha^2
    assert O.divergence(0.0, 3.0, 1.0, 0.0) == pytest.approx(3.0)
    assert O.divergence(0.0, 4.0, 0.5, 0.0) == pytest.approx(8.0)


def test_alpha_zero_rejected():
    with pytest.raises(ValueError):
        O.a_fn(1.0, 1.0, 0.0, 0.5)
    with pytest.raises(ValueError):
        O.g_case(0.0, 2.0)


@pytest.mark.parametrize("ab,case,expo", [((1, 0), "alpha", 1.0), ((2, -1), "alpha", 0.5), ((1, 1), "alpha", 1.0),
                                          ((1, -0.5), "1-beta", 2 / 3), ((0.5, 0), "1-beta", 1.0),
                                          ((1, 2), "alpha+beta-1", 0.5), ((0.5, 1), "alpha", 2.0),
                                          ((1, 0.5), "alpha", 1.0), ((1, -1), "1-beta", 0.5)])
def test_g_table(ab, case, expo):
    """P:531-539 row selection and the inverse exponent (SPEC S:220-221 examples)."""
    assert O.g_case(*ab) == case
    t = RNG.uniform(0.1, 4, 20)
    np.testing.assert_allclose(O.g_inv(t, *ab), t ** expo, rtol=1e-14)
    np.testing.assert_allclose(O.g_fn(O.g_inv(t, *ab), *ab), t, rtol=1e-12)


def test_g_log_case():
    t = RNG.uniform(-2, 2, 20)
    np.testing.assert_allclose(O.g_inv(t, 0, 1), np.exp(t))
    assert O.g_inv(0.0, 0, 1) == 1.0


# ------------------------------------------------------------------ one update step
def _bruteforce_num_den(ms, Y, M, factors, ell, alpha, beta):
    """Literal eq:num: for every element of Theta^(ell), sum over observed i
    and contracted r of a(y_i, yhat_i) * 1(i_l in i, r_l in r) * prod_{l' != l} theta."""
    ops, out = O.parse(ms)
    dims = {}
    for op, t in zip(ops, factors):
        dims.update(zip(op, np.shape(t)))
    con = [c for c in dict.fromkeys("".join(ops)) if c not in out]
    yhat = np.maximum(O.contract_bruteforce(ms, factors), O.EPS_Y)
    A = np.zeros(np.shape(factors[ell]))
    B = np.zeros(np.shape(factors[ell]))
    for obs in itertools.product(*[range(dims[c]) for c in out]):
        if M is not None and M[obs] == 0:
            continue
        a = float(O.a_fn(Y[obs], yhat[obs], alpha, beta))
        b = float(O.b_fn(Y[obs], yhat[obs], alpha, beta))
        env = dict(zip(out, obs))
        for rr in itertools.product(*[range(dims[c]) for c in con]):
            env.update(zip(con, rr))
            g = 1.0
            for l2, (op, t) in enumerate(zip(ops, factors)):
                if l2 != ell:
                    g *= float(t[tuple(env[c] for c in op)])
            idx = tuple(env[c] for c in ops[ell])
            A[idx] += a * g
            B[idx] += b * g
    return A, B


@pytest.mark.parametrize("ms,shape,ranks", TINY_MODELS[:4] + TINY_MODELS[5:])
def test_num_den_vs_bruteforce(ms, shape, ranks):
    f = _rand_factors(ms, shape, ranks)
    Y = RNG.poisson(3.0, size=shape).astype(float)
    M = (RNG.random(shape) > 0.2).astype(np.uint8)
    for ell in range(len(f)):
        A, B = O.numerator_denominator(ms, Y, M, f, ell, 1.0, -0.5)
        A2, B2 = _bruteforce_num_den(ms, Y, M, f, ell, 1.0, -0.5)
        np.testing.assert_allclose(A, A2, rtol=1e-11)
        np.testing.assert_allclose(B, B2, rtol=1e-11)


def test_lee_seung_euclidean_and_kl():
    """Hand-derived Lee-Seung NMF updates (W <- W (Y H)/(Yhat H); KL: W <- W ((Y/Yhat) H)/(1 H))
    written with matrix products, independently of einsum/swap; masked variants use M*Y, M."""
    I, J, R = 7, 6, 3
    W = RNG.uniform(0.1, 1, (I, R))
    H = RNG.uniform(0.1, 1, (J, R))
    Y = RNG.uniform(0.1, 3, (I, J))
    M = (RNG.random((I, J)) > 0.3).astype(np.uint8)
    Yh = W @ H.T
    for mask in (None, M):
        Mf = np.ones((I, J)) if mask is None else mask.astype(float)
        want = W * ((Mf * Y) @ H) / ((Mf * Yh) @ H)
        np.testing.assert_allclose(O.update_factor("ir,jr->ij", Y, mask, [W, H], 0, 1, 1), want, rtol=1e-13)
        want = W * ((Mf * Y / Yh) @ H) / (Mf @ H)
        np.testing.assert_allclose(O.update_factor("ir,jr->ij", Y, mask, [W, H], 0, 1, 0), want, rtol=1e-13)
        # second factor: H <- H (Y^T W)/(Yhat^T W)
        want = H * ((Mf * Y).T @ W) / ((Mf * Yh).T @ W)
        np.testing.assert_allclose(O.update_factor("ir,jr->ij", Y, mask, [W, H], 1, 1, 1), want, rtol=1e-13)


def test_rank1_euclidean_exact():
    """Y = u v^T, Theta1 = u  =>  one Euclidean update of Theta2 gives v."""
    u = RNG.uniform(0.5, 2, (6, 1))
    v = RNG.uniform(0.5, 2, (5, 1))
    Y = u @ v.T
    new = O.update_factor("ir,jr->ij", Y, None, [u, RNG.uniform(0.1, 1, (5, 1))], 1, 1, 1)
    np.testing.assert_allclose(new, v, rtol=1e-13)


@pytest.mark.parametrize("ab", [(1, 0), (0.5, 1), (2, -1), (1, 1), (1.3, -0.3)])
def test_single_factor_one_step(ab):
    """'i->i' with g(lambda)=lambda^alpha (row 4 of P:531-539): A/B = (y/theta)^alpha,
    so one update lands exactly on y (S:292 for KL)."""
    y = RNG.uniform(0.5, 4, 9)
    assert O.g_case(*ab) == "alpha"
    new = O.update_factor("i->i", y, None, [RNG.uniform(0.1, 1, 9)], 0, *ab)
    np.testing.assert_allclose(new, y, rtol=1e-12)


@pytest.mark.parametrize("ab", AB_GRID)
def test_exact_factorization_is_fixed_point(ab):
    ms, shape, ranks = "ik,jk,tl,dl,kl->ijtd", (3, 4, 2, 3), (2, 3)
    f = _rand_factors(ms, shape, ranks, 0.5, 1.5)
    Y = O.contract(ms, f)
    for ell in range(len(f)):
        np.testing.assert_allclose(O.update_factor(ms, Y, None, f, ell, *ab), f[ell], rtol=1e-12)


@pytest.mark.parametrize("ab", [(1, 0), (1, 1), (0.5, 0), (1, -0.5), (1, 2), (0, 1)])
def test_gradient_identity(ab):
    """B - A = alpha * dLoss/dTheta (from dL/dy = (b-a)/alpha); (0,1): B*g(1) - A = -A = dLoss."""
    ms, shape, ranks = "ia,jb,kc,abc->ijk", (3, 4, 3), (2, 2, 2)
    f = _rand_factors(ms, shape, ranks)
    Y = RNG.uniform(0.2, 3, shape)
    M = (RNG.random(shape) > 0.25).astype(np.uint8)
    alpha, beta = ab
    for ell in range(len(f)):
        A, B = O.numerator_denominator(ms, Y, M, f, ell, alpha, beta)
        grad = np.zeros_like(f[ell])
        for idx in itertools.product(*[range(n) for n in f[ell].shape]):
            h = 1e-6 * f[ell][idx]
            fp = [x.copy() for x in f]
            fm = [x.copy() for x in f]
            fp[ell][idx] += h
            fm[ell][idx] -= h
            grad[idx] = (O.loss(ms, Y, M, fp, alpha, beta)[0] - O.loss(ms, Y, M, fm, alpha, beta)[0]) / (2 * h)
        want = -A if alpha == 0 else (B - A)
        scale = grad if alpha == 0 else alpha * grad
        np.testing.assert_allclose(scale, want, rtol=1e-5, atol=1e-7 * np.abs(want).max())


def test_mask_invariance_bit_exact():
    ms, shape, ranks = "ir,jr,kr->ijk", (5, 6, 4), (3,)
    f = _rand_factors(ms, shape, ranks)
    Y = RNG.poisson(2.0, size=shape).astype(float)
    M = (RNG.random(shape) > 0.3).astype(np.uint8)
    ref, tr = O.fit(ms, Y, M, f, 1, -0.5, 3)
    for fill in (np.nan, np.inf, 1e30, -5.0):
        Y2 = np.where(M != 0, Y, fill)
        got, tr2 = O.fit(ms, Y2, M, f, 1, -0.5, 3)
        for a, b in zip(ref, got):
            assert np.array_equal(a, b)
        assert tr == tr2


# ------------------------------------------------------------------ sweeps (Theorem 2)
@pytest.mark.parametrize("ab", AB_GRID)
@pytest.mark.parametrize("ms,shape,ranks", [("ir,jr,kr->ijk", (6, 5, 4), (3,)),
                                            ("ia,jb,kc,abc->ijk", (5, 4, 6), (2, 3, 2)),
                                            ("ik,jk,tl,dl,kl->ijtd", (4, 3, 3, 5), (3, 2))])
def test_monotone_every_update(ab, ms, shape, ranks):
    f = _rand_factors(ms, shape, ranks)
    truth = _rand_factors(ms, shape, ranks, 0.2, 1.5)
    Y = RNG.poisson(O.contract(ms, truth)).astype(float) + (0.5 if ab[0] <= 0 or sum(ab) <= 0 else 0.0)
    M = (RNG.random(shape) > 0.15).astype(np.uint8)
    _, tr = O.fit(ms, Y, M, f, *ab, 15, check_monotone=True)
    assert all(t1 <= t0 * (1 + 1e-12) for t0, t1 in zip(tr, tr[1:]))
    assert tr[-1] < tr[0]


def test_planted_recovery():
    """noiseless rank-2 CP 5x6x7, fit rank 4 under KL -> mean loss <= 1e-6 in >= 1 of 5 seeds."""
    ms = "ir,jr,kr->ijk"
    best = np.inf
    for seed in range(5):
        rng = np.random.default_rng(seed)
        truth = [rng.uniform(0.1, 1, (n, 2)) for n in (5, 6, 7)]
        Y = O.contract(ms, truth)
        init = [rng.uniform(0.1, 1, (n, 4)) for n in (5, 6, 7)]
        _, tr = O.fit(ms, Y, None, init, 1, 0, 2000)
        best = min(best, tr[-1] / Y.size)
        if best <= 1e-6:
            break
    assert best <= 1e-6


def test_loss_masked_sum_and_count():
    Y = np.array([[3.0, 5.0]])
    yh = [np.array([[1.0]]), np.array([[1.0], [1.0]])]
    s, n = O.loss("ir,jr->ij", Y, np.array([[1, 0]], dtype=np.uint8), yh, 1, 1)
    assert (s, n) == (2.0, 1)
    s, n = O.loss("ir,jr->ij", Y, None, yh, 1, 1)
    assert (s, n) == (10.0, 2)
