"""Pins of the oracle's App. B losses and of the train / validation / heldout
protocol with its stopping rules, against things other than the oracle
(-m "not gpu"):

  * the likelihoods the paper derives them from, evaluated by scipy.stats (negative binomial,
    Bernoulli, binomial) and scipy.special.kl_div (Jensen-Shannon as the mean KL to the midpoint)
  * calculus: eq:prop at lambda = 1 and at lambda in {0.5, 2} with the paper's own
    convex / concave splits, by central finite differences
  * Theorem 1 / 2 monotonicity after every factor update, exact factorizations as fixed points
  * the stopping rules on hand-made traces; label-invariance of the split fit
"""
import numpy as np
import pytest
from scipy import special, stats

from nef_inputs import split_labels
from oracle import nef_oracle as O

RNG = np.random.default_rng(2602)

SPECS = [O.make_loss("negbin", phi=1.0), O.make_loss("negbin", phi=3.5), O.make_loss("bernoulli"),
         O.make_loss("binomial", n=7.0), O.make_loss("js")]


def test_spec_examples():
    # NegBinomial phi = 1, x = 0, y = 2 -> a = 0, b = 1/3
    nb = O.make_loss("negbin", phi=1.0)
    assert O.loss_a(nb, 0.0, 2.0) == 0.0
    assert O.loss_b(nb, 0.0, 2.0) == pytest.approx(1.0 / 3.0, rel=1e-15)
    # JS g^{-1}(0) = 1
    assert O.loss_ginv(O.make_loss("js"), 0.0) == 1.0
    # g(lambda) = lambda for the odds / NB losses: identity inverse
    t = RNG.uniform(0.1, 3, 10)
    for k in ("negbin", "bernoulli", "binomial"):
        np.testing.assert_array_equal(O.loss_ginv(O.make_loss(k, phi=1.0, n=2.0), t), t)
    with pytest.raises(ValueError):
        O.make_loss("poisson")


def test_negbin_is_the_nb_likelihood():
    """L(x, y) = (phi + x) log(phi + y) - x log y is the NB negative log-likelihood in
    its mean y up to terms free of y: differences in y match scipy's nbinom exactly."""
    for phi in (0.5, 1.0, 4.0):
        spec = O.make_loss("negbin", phi=phi)
        x = RNG.integers(0, 30, 50).astype(float)
        y1, y2 = RNG.uniform(0.1, 20, 50), RNG.uniform(0.1, 20, 50)
        nll = lambda y: -stats.nbinom.logpmf(x, phi, phi / (phi + y))
        np.testing.assert_allclose(O.loss_value(spec, x, y1) - O.loss_value(spec, x, y2), nll(y1) - nll(y2),
                                   rtol=1e-9, atol=1e-9)
        # per-entry phi through aux equals the scalar spec
        np.testing.assert_array_equal(O.loss_value(O.make_loss("negbin"), x, y1, np.full(50, phi)),
                                      O.loss_value(spec, x, y1))


def test_bernoulli_is_the_odds_likelihood():
    """L(x, mu) = log(1 + mu) - x log mu equals -log Bern(x | mu / (1 + mu)) exactly."""
    spec = O.make_loss("bernoulli")
    x = RNG.integers(0, 2, 60).astype(float)
    mu = RNG.uniform(0.01, 9, 60)
    np.testing.assert_allclose(O.loss_value(spec, x, mu), -stats.bernoulli.logpmf(x, mu / (1 + mu)), rtol=1e-12)


def test_binomial_is_the_odds_likelihood():
    """with n trials the odds NLL is n log(1 + mu) - x log mu up to log C(n, x)."""
    n = RNG.integers(1, 12, 60).astype(float)
    x = np.floor(RNG.uniform(0, 1, 60) * (n + 1))
    mu = RNG.uniform(0.01, 9, 60)
    spec = O.make_loss("binomial")
    want = -stats.binom.logpmf(x, n, mu / (1 + mu)) + np.log(special.comb(n, x))
    np.testing.assert_allclose(O.loss_value(spec, x, mu, n), want, rtol=1e-10, atol=1e-12)


def test_js_is_mean_kl_to_midpoint():
    """JS(x, y) = 1/2 KL(x || m) + 1/2 KL(y || m), m = (x + y)/2 (generalized KL,
    scipy.special.kl_div); zero at x = y; x = 0 gives (y / 2) log 2."""
    spec = O.make_loss("js")
    x = np.concatenate([RNG.uniform(0, 8, 40), [0.0, 0.0]])
    y = np.concatenate([RNG.uniform(0.05, 8, 40), [1.0, 3.0]])
    m = (x + y) / 2
    np.testing.assert_allclose(O.loss_value(spec, x, y), 0.5 * special.kl_div(x, m) + 0.5 * special.kl_div(y, m),
                               rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(O.loss_value(spec, y, y), 0.0, atol=1e-13)
    assert O.loss_value(spec, 0.0, 3.0) == pytest.approx(1.5 * np.log(2), rel=1e-14)


# paper's convex / concave splits and c(lambda), g(lambda)
def _split(kind, x, aux):
    if kind == "negbin":
        return (lambda y: -x * np.log(y)), (lambda y: (aux + x) * np.log(aux + y)), (lambda l: 1 / l), (lambda l: l)
    if kind == "bernoulli":
        return (lambda y: -x * np.log(y)), (lambda y: np.log1p(y)), (lambda l: 1 / l), (lambda l: l)
    if kind == "binomial":
        return (lambda y: -x * np.log(y)), (lambda y: aux * np.log1p(y)), (lambda l: 1 / l), (lambda l: l)
    return ((lambda y: 0.5 * (special.xlogy(x, x) + y * np.log(y))),
            (lambda y: -(x + y) / 2 * np.log((x + y) / 2)), (lambda l: 0.5 + 0 * l), np.log)


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: "%s-%s" % (s["kind"], s["phi"] or s["n"]))
def test_eq_prop_decomposition(spec):
    """eq:prop: d/dy L_vex(x, lambda y) + d/dy L_cave(x, y) = c(lambda) [g(lambda) b - a]
    for lambda in {0.5, 1, 2}, with the paper's splits; at lambda = 1 this is dL/dy."""
    kind = spec["kind"]
    x = RNG.uniform(0.1, 6, 30) if kind != "bernoulli" else RNG.integers(0, 2, 30).astype(float)
    y = RNG.uniform(0.2, 6, 30)
    aux = spec["phi"] if kind == "negbin" else spec["n"]
    vex, cave, c, g = _split(kind, x, aux)
    a, b = O.loss_a(spec, x, y), O.loss_b(spec, x, y)
    for lam in (0.5, 1.0, 2.0):
        h = 1e-6 * y
        hl = 1e-6 * lam * y      # the derivative of L_vex in its 2nd argument, taken at lambda y
        dvex = (vex(lam * y + hl) - vex(lam * y - hl)) / (2 * hl)
        dcave = (cave(y + h) - cave(y - h)) / (2 * h)
        np.testing.assert_allclose(dvex + dcave, c(lam) * (g(lam) * b - a), rtol=1e-6, atol=1e-8)
    h = 1e-6 * y
    fd = (O.loss_value(spec, x, y + h) - O.loss_value(spec, x, y - h)) / (2 * h)
    np.testing.assert_allclose(fd, c(1.0) * (g(1.0) * b - a), rtol=1e-6, atol=1e-8)


MODELS = [("ir,jr,kr->ijk", (6, 5, 4), (3,)), ("ia,jb,kc,abc->ijk", (5, 4, 6), (2, 3, 2)),
          ("ik,jk,tl,dl,kl->ijtd", (4, 3, 3, 5), (3, 2))]


def _data(kind, ms, shape, ranks, rng):
    fs = O.factor_shapes(ms, shape, ranks)
    truth = [rng.gamma(1.0, 1.0, s) for s in fs]
    yh = O.contract(ms, truth)
    aux = None
    if kind == "bernoulli":
        Y = (rng.random(shape) < yh / (1 + yh)).astype(float)
    elif kind == "binomial":
        aux = rng.integers(1, 9, shape).astype(float)
        Y = rng.binomial(aux.astype(int), yh / (1 + yh)).astype(float)
    elif kind == "negbin":
        aux = rng.uniform(0.5, 3.0, shape)
        Y = rng.negative_binomial(aux, aux / (aux + yh)).astype(float)
    else:
        Y = rng.poisson(yh).astype(float)
    init = [rng.uniform(0.1, 1, s) for s in fs]
    return Y, aux, init


@pytest.mark.parametrize("kind", ["negbin", "bernoulli", "binomial", "js"])
@pytest.mark.parametrize("ms,shape,ranks", MODELS)
def test_monotone_every_update(kind, ms, shape, ranks):
    """Theorem 1 / 2: the loss never increases across a factor update, for the
    App. B losses too (per-entry phi / n through aux; a 15 % mask)."""
    rng = np.random.default_rng(hash((kind, ms)) % (1 << 30))
    Y, aux, init = _data(kind, ms, shape, ranks, rng)
    M = (rng.random(shape) > 0.15).astype(np.uint8)
    spec = O.make_loss(kind)
    _, tr = O.fit(ms, Y, M, init, spec, None, 25, check_monotone=True, aux=aux)
    assert tr[-1] < tr[0]


@pytest.mark.parametrize("kind", ["negbin", "bernoulli", "binomial", "js"])
def test_exact_fit_is_fixed_point(kind):
    """a = b pointwise at the loss's minimiser makes A = B and g^{-1}(1) = 1 (JS: a = 0, exp(0) = 1):
    data equal to the model's mean (NB, JS: y = yhat; odds: x = yhat / (1 + yhat), n yhat / (1 + yhat))
    is a fixed point of every update."""
    ms, shape, ranks = "ir,jr,kr->ijk", (5, 4, 6), (2,)
    rng = np.random.default_rng(4)
    th = [rng.uniform(0.2, 1.5, s) for s in O.factor_shapes(ms, shape, ranks)]
    yh = O.contract(ms, th)
    aux = None
    if kind == "bernoulli":
        Y = yh / (1 + yh)
    elif kind == "binomial":
        aux = rng.integers(1, 6, shape).astype(float)
        Y = aux * yh / (1 + yh)
    else:
        Y = yh.copy()
        aux = rng.uniform(0.5, 2, shape) if kind == "negbin" else None
    spec = O.make_loss(kind)
    for ell in range(3):
        np.testing.assert_allclose(O.update_factor(ms, Y, None, th, ell, spec, aux=aux), th[ell], rtol=1e-12)


# ------------------------------------------------------------------ split protocol / stopping
RULE = {"max_iters": 5000, "min_rel_decrease": 1e-6, "val_patience": 5}


def test_stop_rules_on_hand_traces():
    """P:497 with the readings R29-R31: strict increases vs the previous sweep, counted
    consecutively (an equal value resets); relative training-loss decrease; max_iters; priority
    patience > plateau > max_iters."""
    tr = [100.0 - t for t in range(12)]
    val = [10, 9, 8, 8.5, 8.6, 8.7, 8.8, 8.9, 9.0, 9.1, 9.2, 9.3]
    got = [O.stop_decision(tr, val, t, RULE) for t in range(12)]
    assert got[:7] == [None] * 7 and got[7] == "patience"        # increases at t = 3..7
    val2 = [10, 9, 8, 8.5, 8.6, 8.6, 8.7, 8.8, 8.9, 9.0, 9.1, 9.2]
    got2 = [O.stop_decision(tr, val2, t, RULE) for t in range(12)]
    assert got2.index("patience") == 10                           # the tie at t = 5 resets the count
    assert O.stop_decision([10.0, 10.0 - 9e-6], [0, 0], 1, RULE) == "plateau"      # 9e-7 relative
    assert O.stop_decision([10.0, 10.0 - 2e-5], [0, 0], 1, RULE) is None
    assert O.stop_decision([10.0, 10.0 - 5e-6], [0, 0], 1, RULE) == "plateau"
    assert O.stop_decision([10.0, 10.5], [0, 0], 1, RULE) == "plateau"              # an increase is no decrease
    assert O.stop_decision([10.0, 9.0, 8.0], [0, 0, 0], 2, dict(RULE, max_iters=2)) == "max_iters"
    assert O.stop_decision([10.0], [0], 0, dict(RULE, max_iters=0)) == "max_iters"
    # priority: a patience stop on the same sweep as a plateau
    assert O.stop_decision([1, 1, 1, 1, 1, 1], [1, 2, 3, 4, 5, 6], 5, RULE) == "patience"


def test_split_labels_law():
    """train w.p. 0.9, else heldout; 5 % of train to validation: fractions within 4
    sigma of the binomial expectation; seeded."""
    shape = (200, 150, 40)
    lab = split_labels(shape, 0.1, 0.05, seed=3)
    n = lab.size
    for r, p in ((1, 0.9 * 0.95), (2, 0.9 * 0.05), (3, 0.1)):
        f = np.count_nonzero(lab == r)
        assert abs(f - n * p) < 4 * np.sqrt(n * p * (1 - p)), (r, f / n)
    assert np.array_equal(lab, split_labels(shape, 0.1, 0.05, seed=3))
    assert set(np.unique(lab)) <= {1, 2, 3}
    miss = np.zeros(shape, dtype=bool)
    miss[0] = True
    lab2 = split_labels(shape, 0.1, 0.05, seed=3, missing=miss)
    assert np.all(lab2[0] == 0) and np.array_equal(lab2[1:], lab[1:])


def test_split_fit_trains_on_train_role_only():
    """The fitted factors and the train trace depend only on the train entries (SPEC S:316 mask
    independence): arbitrary values at validation / heldout / excluded entries leave them
    bit-identical; the validation and heldout traces are the loss sums of those roles."""
    ms, shape, ranks = "ir,jr,kr->ijk", (7, 6, 5), (3,)
    rng = np.random.default_rng(8)
    fs = O.factor_shapes(ms, shape, ranks)
    Y = rng.poisson(O.contract(ms, [rng.gamma(1, 1, s) for s in fs])).astype(float)
    lab = split_labels(shape, 0.2, 0.2, seed=9)
    lab[0, 0, :2] = 0
    init = [rng.uniform(0.1, 1, s) for s in fs]
    spec = O.make_loss("ab", 1.0, 0.0)
    rule = dict(RULE, max_iters=6, min_rel_decrease=-np.inf, val_patience=0)
    th, traces, counts, t, reason = O.fit_split(ms, Y, lab, init, spec, rule)
    assert (t, reason) == (6, "max_iters") and len(traces[0]) == 7
    assert counts == [int(np.sum(lab == r)) for r in (1, 2, 3)]
    Y2 = np.where(lab == 1, Y, 1e6 * RNG.random(shape))
    th2, traces2, _, _, _ = O.fit_split(ms, Y2, lab, init, spec, rule)
    for a, b in zip(th, th2):
        assert np.array_equal(a, b)
    assert traces[0] == traces2[0]
    assert traces2[2] != traces[2]
    # the train trace is non-increasing (Theorem 2) and the heldout mean is sum / count
    assert all(b <= a * (1 + 1e-12) for a, b in zip(traces[0], traces[0][1:]))


def test_split_fit_patience_stop_on_overfit():
    """An over-parameterised fit of noisy counts eventually raises the validation loss: the run
    stops with 'patience' exactly when the last `val_patience` sweeps each raised it."""
    ms, shape, ranks = "ir,jr,kr->ijk", (8, 7, 6), (12,)
    rng = np.random.default_rng(11)
    fs = O.factor_shapes(ms, shape, ranks)
    Y = rng.poisson(3.0 * O.contract(ms, [rng.gamma(1, 1, (s[0], 1)) for s in fs])).astype(float)
    lab = split_labels(shape, 0.1, 0.3, seed=12)
    init = [rng.uniform(0.1, 1, s) for s in fs]
    rule = dict(RULE, max_iters=3000, min_rel_decrease=0.0, val_patience=3)
    _, traces, _, t, reason = O.fit_split(ms, Y, lab, init, O.make_loss("ab", 1.0, 0.0), rule)
    assert reason == "patience", (reason, t)
    v = traces[1]
    assert all(v[s] > v[s - 1] for s in range(t - 2, t + 1)) and not (v[t - 3] > v[t - 4])
