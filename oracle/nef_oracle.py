"""NNEinFact float64 CPU ORACLE — test infrastructure only.

THIS MODULE IS TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import it.  The
product path (``paper_2602_02759_b200``) never imports, links or executes it, and
it shares no code with the CUDA path (no kernels, headers, tables or helpers).

It is a plain, slow, obviously-correct transcription of arxiv 2602.02759 in
float64 numpy.  Citations ``P:N`` are lines of the paper's LaTeX:

* model family / einsum string .................. P:43-54  (eq:contraction_structure, eq:einsum, eq:einstr)
* objective, Theta >= eps ........................ P:102-106 (eq:obj)
* multiplicative update (Theorem 1) .............. P:119-125 (eq:explicit-update)
* numerator as einsum(einstr_l), swap ............ P:137-149 (eq:num, einstr_l)
* Algorithm 1 (Gauss-Seidel sweep) ............... P:152-182
* (alpha,beta)-divergence, 5 cases ............... P:500-525
* a(x,y), b(x,y) ................................. P:529
* g(lambda) 4-case table ......................... P:531-539
* masking "replace Y, Yhat by M*Y, M*Yhat" ....... P:321 (read as zeroing a and b at
  missing entries, reading R5)
* other decomposable losses (App. B) ............. P:541-610 (negative binomial, Bernoulli and
  binomial odds, Jensen-Shannon): a, b, g and the loss as the paper writes them
* train / validation / heldout protocol .......... P:318-326 (splits, masked training loss,
  average heldout loss); stopping criteria P:497

Readings where the paper is silent (all listed in DESIGN.md §Readings):
  eps = 1e-12 (R3), Yhat floor eps_y = 1e-30 (R4), mask nonzero = observed (R6),
  loss trace = SUM over observed entries (R7), B == 0 -> multiplier 1 (R10),
  0*log 0 = 0 (R8), trace[0] = loss at init, trace[t] = after sweep t (R9).

Parity pins: every function here is pinned by tests/test_oracle_pins.py against
closed forms, worked values, brute-force loops and textbook (Lee-Seung) updates.
The one exception is noted at ``fit`` (full-trajectory values have no closed
form; the trajectory is pinned only through its per-step pins + Theorem 2
monotonicity), see DESIGN.md "parity unpinned".
"""
from __future__ import annotations

import itertools
import math
import re

import numpy as np

EPS = 1e-12     # reading R3: "very small epsilon"
EPS_Y = 1e-30   # reading R4: floor on Yhat inside a, b and the loss

# --------------------------------------------------------------------------------------
# model strings and swap
# --------------------------------------------------------------------------------------
_IDX = re.compile(r"^[A-Za-z]+$")


def parse(model_str: str):
    """Parse ``'i1r1,...,iLrL->i1...iM'`` (eq:einsum).

    Returns (operands: list[str], output: str).  Spaces are ignored.  Raises
    ValueError on: missing '->', empty operand, illegal character, repeated index
    inside one operand, output index absent from every operand, repeated output index.
    """
    s = model_str.replace(" ", "")
    if s.count("->") != 1:
        raise ValueError("missing '->'")
    lhs, out = s.split("->")
    ops = lhs.split(",")
    for op in ops:
        if op == "":
            raise ValueError("empty operand")
        if not _IDX.match(op):
            raise ValueError("illegal character in operand %r" % op)
        if len(set(op)) != len(op):
            raise ValueError("repeated index in operand %r" % op)
    if out == "" or not _IDX.match(out):
        raise ValueError("empty or illegal output")
    if len(set(out)) != len(out):
        raise ValueError("repeated output index")
    for c in out:
        if not any(c in op for op in ops):
            raise ValueError("output index %r absent from operands" % c)
    return ops, out


def swap(model_str: str, ell: int) -> str:
    """einstr_ell = swap(model_str, ell): exchange the output subscript with operand
    ell's subscript.  ``ell`` is 0-based here (paper is 1-based)."""
    ops, out = parse(model_str)
    if not 0 <= ell < len(ops):
        raise ValueError("ell out of range")
    new = list(ops)
    new[ell] = out
    return ",".join(new) + "->" + ops[ell]


def index_dims(model_str: str, shape, ranks):
    """Bind index letters to sizes: observed indices from ``shape`` in output order,
    contracted indices from ``ranks`` in order of first appearance (reading R18)."""
    ops, out = parse(model_str)
    if len(shape) != len(out):
        raise ValueError("shape rank mismatch")
    dims = {c: int(n) for c, n in zip(out, shape)}
    contracted = []
    for op in ops:
        for c in op:
            if c not in dims and c not in contracted:
                contracted.append(c)
    if len(ranks) != len(contracted):
        raise ValueError("rank count mismatch")
    for c, r in zip(contracted, ranks):
        dims[c] = int(r)
    return dims


def factor_shapes(model_str, shape, ranks):
    ops, _ = parse(model_str)
    d = index_dims(model_str, shape, ranks)
    return [tuple(d[c] for c in op) for op in ops]


# --------------------------------------------------------------------------------------
# contraction: eq:einstr.  A library primitive (np.einsum) is the step.
# --------------------------------------------------------------------------------------
def contract(model_str: str, operands):
    """Yhat = einsum(model_str, Theta) (eq:einstr), float64."""
    parse(model_str)
    return np.einsum(model_str.replace(" ", ""), *[np.asarray(o, dtype=np.float64) for o in operands],
                     optimize="greedy")


def contract_bruteforce(model_str: str, operands):
    """Literal nested loops of eq:contraction_structure: for every observed
    multi-index i, sum over every contracted multi-index r of prod_l theta^(l).
    Pure Python; tiny inputs only."""
    ops, out = parse(model_str)
    dims = {}
    for op, t in zip(ops, operands):
        for c, n in zip(op, np.shape(t)):
            if dims.setdefault(c, n) != n:
                raise ValueError("inconsistent size for index %r" % c)
    contracted = [c for c in dict.fromkeys("".join(ops)) if c not in out]
    res = np.zeros([dims[c] for c in out], dtype=np.float64)
    for obs in itertools.product(*[range(dims[c]) for c in out]):
        env = dict(zip(out, obs))
        total = 0.0
        for con in itertools.product(*[range(dims[c]) for c in contracted]):
            env.update(zip(contracted, con))
            term = 1.0
            for op, t in zip(ops, operands):
                term *= float(t[tuple(env[c] for c in op)])
            total += term
        res[obs] = total
    return res


# --------------------------------------------------------------------------------------
# (alpha,beta)-divergence, a/b, g
# --------------------------------------------------------------------------------------
def check_ab(alpha: float, beta: float):
    """'when alpha = 0 and beta != 1, we could not derive a decomposition'."""
    if alpha == 0 and beta != 1:
        raise ValueError("alpha=0 requires beta=1 (P:529)")


def divergence(x, y, alpha: float, beta: float):
    """Elementwise L_{alpha,beta}(x, y), x = data, y = model, float64.

    x = 0 is handled by the limits x^p -> 0 (p > 0) and x^p log x -> 0 (reading R8).
    """
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    a, b = float(alpha), float(beta)
    with np.errstate(divide="ignore", invalid="ignore"):
        if a != 0 and b != 0 and a + b != 0:
            xab = np.where(x > 0, np.power(np.where(x > 0, x, 1.0), a + b), 0.0 if a + b > 0 else np.inf)
            xa = np.where(x > 0, np.power(np.where(x > 0, x, 1.0), a), 0.0 if a > 0 else np.inf)
            return (1.0 / (a * b)) * (a / (a + b) * xab + b / (a + b) * np.power(y, a + b) - xa * np.power(y, b))
        if b == 0 and a != 0:
            xs = np.where(x > 0, x, 1.0)
            xa = np.where(x > 0, np.power(xs, a), 0.0)
            xalog = np.where(x > 0, np.power(xs, a) * np.log(xs / y), 0.0)
            return (1.0 / a ** 2) * (np.power(y, a) - xa + a * xalog)
        if a == -b and a != 0:
            return (1.0 / a ** 2) * (np.power(x, a) / np.power(y, a) - 1.0 + a * np.log(y / x))
        if a == 0 and b != 0:
            return (1.0 / b ** 2) * (b * np.power(y, b) * np.log(y / x) - np.power(y, b) + np.power(x, b))
        return 0.5 * (np.log(x) - np.log(y)) ** 2


def a_fn(x, y, alpha: float, beta: float):
    """a(x, y): x^alpha y^(beta-1) for alpha != 0; log(x/y) for (0, 1)."""
    check_ab(alpha, beta)
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if alpha != 0:
        with np.errstate(divide="ignore"):
            xa = np.where(x > 0, np.power(np.where(x > 0, x, 1.0), alpha), 0.0 if alpha > 0 else np.inf)
        return xa * np.power(y, beta - 1.0)
    with np.errstate(divide="ignore"):
        return np.log(x / y)


def b_fn(x, y, alpha: float, beta: float):
    """b(x, y): y^(alpha+beta-1) for alpha != 0; 1 for (0, 1)."""
    check_ab(alpha, beta)
    y = np.asarray(y, dtype=np.float64)
    if alpha != 0:
        return np.power(y, alpha + beta - 1.0) * np.ones_like(np.asarray(x, dtype=np.float64))
    return np.ones(np.broadcast(np.asarray(x), y).shape)


def g_case(alpha: float, beta: float) -> str:
    """Which row of the g(lambda) table applies."""
    check_ab(alpha, beta)
    if alpha == 0 and beta == 1:
        return "log"
    q = (1.0 - beta) / alpha
    if q > 1:
        return "1-beta"
    if q < 0:
        return "alpha+beta-1"
    return "alpha"


def g_fn(lam, alpha: float, beta: float):
    """g(lambda)."""
    lam = np.asarray(lam, dtype=np.float64)
    case = g_case(alpha, beta)
    if case == "log":
        return np.log(lam)
    if case == "1-beta":
        return np.power(lam, 1.0 - beta)
    if case == "alpha+beta-1":
        return np.power(lam, alpha + beta - 1.0)
    return np.power(lam, alpha)


def g_inv(t, alpha: float, beta: float):
    """g^{-1}(t): the inverse of g_fn, row by row of P:532-538."""
    t = np.asarray(t, dtype=np.float64)
    case = g_case(alpha, beta)
    if case == "log":
        return np.exp(t)
    with np.errstate(divide="ignore"):
        if case == "1-beta":
            return np.power(t, 1.0 / (1.0 - beta))
        if case == "alpha+beta-1":
            return np.power(t, 1.0 / (alpha + beta - 1.0))
        return np.power(t, 1.0 / alpha)


# --------------------------------------------------------------------------------------
# loss specifications: the (alpha,beta) family and the other decomposable
# losses of App. B.  A spec is a plain dict; `aux` is an optional per-entry
# tensor (same shape as Y): the dispersion phi_i (negative binomial) or the number of
# trials n_i (binomial); without it the scalar in the spec is used for every entry.
# --------------------------------------------------------------------------------------
LOSS_KINDS = ("ab", "negbin", "bernoulli", "binomial", "js")


def make_loss(kind="ab", alpha=None, beta=None, phi=None, n=None):
    """Loss spec.  'ab': (alpha, beta); 'negbin': dispersion phi > 0;
    'bernoulli': odds; 'binomial': n trials; 'js'."""
    if kind not in LOSS_KINDS:
        raise ValueError("unknown loss kind %r" % kind)
    if kind == "ab":
        check_ab(alpha, beta)
    return {"kind": kind, "alpha": alpha, "beta": beta, "phi": phi, "n": n}


def _spec(alpha, beta):
    """Accept a spec dict (beta None) or a plain (alpha, beta) pair."""
    if isinstance(alpha, dict):
        return alpha
    return make_loss("ab", alpha, beta)


def _aux(loss, key, aux, shape):
    if aux is not None:
        return np.asarray(aux, dtype=np.float64)
    return np.full(shape, float(loss[key]))


def loss_a(loss, x, y, aux=None):
    """a(x, y) of the loss (NB / Bernoulli / binomial a = x / y P:558, P:582, P:589;
    JS a = log((x + y) / (2y)) P:605)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    k = loss["kind"]
    if k == "ab":
        return a_fn(x, y, loss["alpha"], loss["beta"])
    if k in ("negbin", "bernoulli", "binomial"):
        return x / y
    return np.log((x + y) / (2.0 * y))


def loss_b(loss, x, y, aux=None):
    """b(x, y): NB (phi + x) / (phi + y); Bernoulli 1 / (1 + y); binomial
    n / (1 + y) (the update's denominator); JS 1."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    k = loss["kind"]
    if k == "ab":
        return b_fn(x, y, loss["alpha"], loss["beta"])
    if k == "negbin":
        phi = _aux(loss, "phi", aux, np.broadcast(x, y).shape)
        return (phi + x) / (phi + y)
    if k == "bernoulli":
        return 1.0 / (1.0 + y) * np.ones_like(x)
    if k == "binomial":
        n = _aux(loss, "n", aux, np.broadcast(x, y).shape)
        return n / (1.0 + y)
    return np.ones(np.broadcast(x, y).shape)


def _xlogy(x, y):
    """x log y with 0 log(.) = 0 (reading R8)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(x > 0, x * np.log(np.where(x > 0, y, 1.0)), 0.0)


def loss_value(loss, x, y, aux=None):
    """Per-entry loss: the (alpha,beta)-divergence; NB (phi + x) log(phi + y) - x log y
    (P:548); Bernoulli log(1 + mu) - x log mu; binomial n log(1 + mu) - x log mu (the
    binomial NLL in the odds up to terms free of mu, P:587-591 with P:570); JS
    -(x + y)/2 log((x + y)/2) + (x log x + y log y)/2."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    k = loss["kind"]
    if k == "ab":
        return divergence(x, y, loss["alpha"], loss["beta"])
    if k == "negbin":
        phi = _aux(loss, "phi", aux, np.broadcast(x, y).shape)
        return (phi + x) * np.log(phi + y) - _xlogy(x, y)
    if k == "bernoulli":
        return np.log1p(y) - _xlogy(x, y)
    if k == "binomial":
        n = _aux(loss, "n", aux, np.broadcast(x, y).shape)
        return n * np.log1p(y) - _xlogy(x, y)
    m = (x + y) / 2.0
    return -m * np.log(m) + 0.5 * (_xlogy(x, x) + y * np.log(y))


def loss_ginv(loss, t):
    """g^{-1}: the (alpha,beta) table; g(lambda) = lambda for NB, Bernoulli and
    binomial; g = log for JS."""
    k = loss["kind"]
    if k == "ab":
        return g_inv(t, loss["alpha"], loss["beta"])
    t = np.asarray(t, dtype=np.float64)
    if k == "js":
        return np.exp(t)
    return t


# --------------------------------------------------------------------------------------
# objective (eq:obj) with mask
# --------------------------------------------------------------------------------------
def _obs(mask, shape):
    if mask is None:
        return np.ones(shape, dtype=bool)
    return np.asarray(mask) != 0          # reading R6: nonzero = observed


def _aux_at(aux, obs):
    if aux is None:
        return None
    return np.where(obs, np.asarray(aux, dtype=np.float64), 1.0)


def loss(model_str, Y, mask, factors, alpha, beta=None, eps_y=EPS_Y, aux=None):
    """Sum over observed entries of L(y_i, max(yhat_i, eps_y)) (eq:obj; reading R7: sum,
    not mean).  ``alpha`` is either the (alpha, beta) pair's alpha or a loss spec (make_loss).
    Returns (sum, n_observed)."""
    spec = _spec(alpha, beta)
    Y = np.asarray(Y, dtype=np.float64)
    obs = _obs(mask, Y.shape)
    yhat = np.maximum(contract(model_str, factors), eps_y)
    vals = loss_value(spec, np.where(obs, Y, 1.0), yhat, _aux_at(aux, obs))
    return float(np.sum(np.where(obs, vals, 0.0))), int(np.count_nonzero(obs))


# --------------------------------------------------------------------------------------
# one multiplicative update (Theorem 1; Algorithm 1 lines 6-9)
# --------------------------------------------------------------------------------------
def numerator_denominator(model_str, Y, mask, factors, ell, alpha, beta=None, eps_y=EPS_Y, aux=None):
    """(A, B) of Algorithm 1 lines 7-8 for factor ``ell`` (0-based):
    Yhat = einsum(model_str, Theta); A = einsum(einstr_ell, ..., a(Y,Yhat), ...);
    B = einsum(einstr_ell, ..., b(Y,Yhat), ...), with a, b zeroed at missing entries."""
    spec = _spec(alpha, beta)
    Y = np.asarray(Y, dtype=np.float64)
    obs = _obs(mask, Y.shape)
    yhat = np.maximum(contract(model_str, factors), eps_y)          # Alg. 1 line 6
    xs = np.where(obs, Y, 1.0)                                       # masked values never read
    ax = _aux_at(aux, obs)
    a = np.where(obs, loss_a(spec, xs, yhat, ax), 0.0)
    b = np.where(obs, loss_b(spec, xs, yhat, ax), 0.0)
    einstr = swap(model_str, ell)
    ops = [np.asarray(f, dtype=np.float64) for f in factors]
    A = contract(einstr, ops[:ell] + [a] + ops[ell + 1:])             # Alg. 1 line 7
    B = contract(einstr, ops[:ell] + [b] + ops[ell + 1:])             # Alg. 1 line 8
    return A, B


def update_factor(model_str, Y, mask, factors, ell, alpha, beta=None, eps=EPS, eps_y=EPS_Y, aux=None):
    """Theta^(ell) <- max(eps, Theta^(ell) * g^{-1}(A / B)) (eq:explicit-update P:121;
    Alg. 1 line 9).  B == 0 -> multiplier 1 (reading R10).  Returns the
    new factor (float64); does not modify ``factors``."""
    spec = _spec(alpha, beta)
    A, B = numerator_denominator(model_str, Y, mask, factors, ell, spec, eps_y=eps_y, aux=aux)
    theta = np.asarray(factors[ell], dtype=np.float64)
    pos = B > 0
    ratio = np.where(pos, A / np.where(pos, B, 1.0), 1.0)
    mult = np.where(pos, loss_ginv(spec, ratio), 1.0)
    return np.maximum(eps, theta * mult)


def fit(model_str, Y, mask, factors, alpha, beta, iters, eps=EPS, eps_y=EPS_Y, check_monotone=False, aux=None):
    """Algorithm 1: ``iters`` full sweeps over ell = 1..L in string order,
    Yhat recomputed before every factor update.  Returns (factors, trace) with
    trace[0] = loss at init and trace[t] = loss after sweep t (reading R9).  ``alpha`` may be
    a loss spec (then ``beta`` is ignored).

    check_monotone asserts Theorem 1 after EVERY factor update (relative slack 1e-12).
    Parity unpinned as a whole trajectory: no closed form exists for it; it is pinned
    through its steps (tests/test_oracle_pins.py) and Theorem 2 monotonicity.
    """
    spec = _spec(alpha, beta)
    th = [np.array(f, dtype=np.float64) for f in factors]
    trace = [loss(model_str, Y, mask, th, spec, eps_y=eps_y, aux=aux)[0]]
    for _ in range(iters):
        for ell in range(len(th)):
            before = loss(model_str, Y, mask, th, spec, eps_y=eps_y, aux=aux)[0] if check_monotone else None
            th[ell] = update_factor(model_str, Y, mask, th, ell, spec, eps=eps, eps_y=eps_y, aux=aux)
            if check_monotone:
                after = loss(model_str, Y, mask, th, spec, eps_y=eps_y, aux=aux)[0]
                assert after <= before + 1e-12 * abs(before) + 1e-300, (ell, before, after)
        trace.append(loss(model_str, Y, mask, th, spec, eps_y=eps_y, aux=aux)[0])
    return th, trace


# --------------------------------------------------------------------------------------
# train / validation / heldout protocol and stopping criteria
# labels: 0 = excluded (missing data), 1 = train, 2 = validation (V), 3 = heldout (H)
# --------------------------------------------------------------------------------------
ROLE_TRAIN, ROLE_VAL, ROLE_HELDOUT = 1, 2, 3


def role_losses(model_str, Y, labels, factors, loss_spec, eps_y=EPS_Y, aux=None):
    """Loss sums and entry counts of the three roles (train, validation, heldout) at the current
    factors; the heldout mean sum / count is the paper's evaluation metric."""
    labels = np.asarray(labels)
    sums, counts = [], []
    for r in (ROLE_TRAIN, ROLE_VAL, ROLE_HELDOUT):
        s_, n_ = loss(model_str, Y, labels == r, factors, loss_spec, eps_y=eps_y, aux=aux)
        sums.append(s_)
        counts.append(n_)
    return sums, counts


def stop_decision(train, val, t, rule):
    """Stopping criteria of P:497 after sweep t (traces hold entries 0..t): validation loss
    increasing (strictly, vs the previous sweep) for ``val_patience`` consecutive sweeps; a
    decrease of the training loss of less than ``min_rel_decrease`` relative to its previous
    value; ``max_iters`` sweeps.  Readings R29-R31.  Returns None or the reason."""
    p = int(rule["val_patience"])
    if p > 0 and t >= p and all(val[s] > val[s - 1] for s in range(t - p + 1, t + 1)):
        return "patience"
    if t >= 1 and (train[t - 1] - train[t]) < rule["min_rel_decrease"] * abs(train[t - 1]):
        return "plateau"
    if t >= rule["max_iters"]:
        return "max_iters"
    return None


def fit_split(model_str, Y, labels, factors, loss_spec, rule, eps=EPS, eps_y=EPS_Y, aux=None):
    """Algorithm 1 trained on the train role only (labels == 1), with the train,
    validation and heldout losses after every sweep and the stopping rules of P:497.  Returns
    (factors, traces[3], counts[3], sweeps_run, reason): traces[r][t] = loss sum of role r after
    sweep t, t = 0..sweeps_run; factors = the iterate after sweep ``sweeps_run``."""
    train_mask = (np.asarray(labels) == ROLE_TRAIN).astype(np.uint8)
    th = [np.array(f, dtype=np.float64) for f in factors]
    sums, counts = role_losses(model_str, Y, labels, th, loss_spec, eps_y, aux)
    traces = [[v] for v in sums]
    t = 0
    reason = stop_decision(traces[0], traces[1], 0, rule)
    while reason is None:
        for ell in range(len(th)):
            th[ell] = update_factor(model_str, Y, train_mask, th, ell, loss_spec, eps=eps, eps_y=eps_y, aux=aux)
        t += 1
        sums, _ = role_losses(model_str, Y, labels, th, loss_spec, eps_y, aux)
        for tr, v in zip(traces, sums):
            tr.append(v)
        reason = stop_decision(traces[0], traces[1], t, rule)
    return th, traces, counts, t, reason


def param_count(model_str, shape, ranks) -> int:
    """Sum over operands of the product of their bound dims."""
    return int(sum(math.prod(s) for s in factor_shapes(model_str, shape, ranks)))
