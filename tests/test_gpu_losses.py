"""GPU parity (-m gpu) of the App. B losses and of the train / validation / heldout
fit with the P:497 stopping rules, through the C ABI, against the float64 oracle.

Bars as in test_gpu_parity.py: factors after one sweep within 1e-4 relative, loss trajectories
within 1e-3; label / mask handling bit-exact (counts exact, garbage at non-train entries changes
nothing the fit computes)."""
import numpy as np
import pytest

from nef_inputs import split_labels
from oracle import nef_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FACTOR_RTOL = 1e-4
TRACE_RTOL = 1e-3


@pytest.fixture(scope="module")
def nef():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_02759_b200 import nef as n
    n.nef_set_kernel_policy(0)
    return n


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30)))


def _data(kind, ms, shape, ranks, seed, per_entry=False):
    """Planted data of each likelihood: NB counts (dispersion phi), Bernoulli / binomial outcomes
    with odds yhat, Poisson counts for JS."""
    rng = np.random.default_rng(seed)
    fs = O.factor_shapes(ms, shape, ranks)
    truth = [rng.gamma(1.0, 1.0, s) for s in fs]
    yh = O.contract(ms, truth)
    yh = yh / yh.mean() * 2.0
    aux = None
    if kind == "negbin":
        phi = rng.uniform(0.5, 4.0, shape) if per_entry else np.full(shape, 2.0)
        Y = rng.negative_binomial(phi, phi / (phi + yh))
        aux, param = (phi, 0.0) if per_entry else (None, 2.0)
    elif kind == "bernoulli":
        Y, param = (rng.random(shape) < yh / (1 + yh)), 0.0
    elif kind == "binomial":
        n = rng.integers(1, 9, shape).astype(float) if per_entry else np.full(shape, 5.0)
        Y = rng.binomial(n.astype(int), yh / (1 + yh))
        aux, param = (n, 0.0) if per_entry else (None, 5.0)
    else:
        Y, param = rng.poisson(yh), 0.0
    init = [rng.uniform(0.1, 1, s).astype(np.float32) for s in fs]
    return Y.astype(np.float32), (aux.astype(np.float32) if aux is not None else None), param, init


def _spec_pair(nef, kind, param, aux_dev, alpha=1.0, beta=0.0):
    spec = nef.loss_spec(kind, alpha, beta, param, aux_dev)
    if kind == "ab":
        return spec, O.make_loss("ab", alpha, beta)
    return spec, O.make_loss(kind, phi=param or None, n=param or None)


CASES = [("ir,jr,kr->ijk", (160, 144, 96), (32,), True),     # tcgen05 (c3-like)
         ("ia,jb,kc,abc->ijk", (96, 80, 64), (16, 16, 16), True),
         ("ir,jr,kr->ijk", (50, 40, 30), (5,), False)]        # CUDA-core (c1 shape)


@pytest.mark.parametrize("kind", ["negbin", "bernoulli", "binomial", "js"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[1])))
@pytest.mark.parametrize("pm", [0.0, 0.1])
def test_appb_loss_parity(nef, kind, case, pm):
    ms, shape, ranks, tc = case
    Y, _, param, init = _data(kind, ms, shape, ranks, seed=31)
    M = (np.random.default_rng(32).random(shape) >= pm).astype(np.uint8) if pm > 0 else None
    plan = nef.Plan(ms, shape, ranks)
    assert all(L["tc"] for L in plan.describe()["lowerings"]) == tc
    spec, ospec = _spec_pair(nef, kind, param, None)
    Yd = torch.from_numpy(Y).cuda()
    Md = torch.from_numpy(M).cuda() if M is not None else None
    F = [torch.from_numpy(f.copy()).cuda() for f in init]
    tr1 = plan.fit_ex(Yd, Md, spec, F, 1)
    ref, rtr = O.fit(ms, Y, M, init, ospec, None, 1)
    errs = [_rel(g.cpu().numpy(), r) for g, r in zip(F, ref)]
    assert max(errs) <= FACTOR_RTOL, errs
    assert _rel(tr1, rtr) <= TRACE_RTOL, (tr1, rtr)
    F = [torch.from_numpy(f.copy()).cuda() for f in init]
    tr = plan.fit_ex(Yd, Md, spec, F, 8)
    _, rtr = O.fit(ms, Y, M, init, ospec, None, 8)
    assert _rel(tr, rtr) <= TRACE_RTOL, _rel(tr, rtr)
    s, n = plan.loss_ex(Yd, Md, spec, [torch.from_numpy(f).cuda() for f in init])
    rs, rn = O.loss(ms, Y, M, init, ospec)
    assert n == rn and abs(s - rs) <= 1e-5 * abs(rs), (s, rs)


@pytest.mark.parametrize("kind", ["negbin", "binomial"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[1])))
@pytest.mark.parametrize("pm", [0.0, 0.1])
def test_per_entry_parameter_stream(nef, kind, case, pm):
    """NB with a per-entry dispersion phi_i and binomial with per-entry trials n_i:
    the parameter tensor is streamed with Y - a second TMA ring of the tcgen05 kernel next to the
    sentinel copy (masked) or the raw Y (unmasked), or the CUDA-core kernel (c1 shape)."""
    ms, shape, ranks, _ = case
    Y, aux, _, init = _data(kind, ms, shape, ranks, seed=33, per_entry=True)
    M = (np.random.default_rng(34).random(shape) >= pm).astype(np.uint8) if pm > 0 else None
    plan = nef.Plan(ms, shape, ranks)
    Ad = torch.from_numpy(aux).cuda()
    spec = nef.loss_spec(kind, aux=Ad)
    Yd, Md = torch.from_numpy(Y).cuda(), (torch.from_numpy(M).cuda() if M is not None else None)
    F = [torch.from_numpy(f.copy()).cuda() for f in init]
    tr = plan.fit_ex(Yd, Md, spec, F, 1, aux=Ad)
    ref, rtr = O.fit(ms, Y, M, init, O.make_loss(kind), None, 1, aux=aux)
    errs = [_rel(g.cpu().numpy(), r) for g, r in zip(F, ref)]
    assert max(errs) <= FACTOR_RTOL, errs
    assert _rel(tr, rtr) <= TRACE_RTOL


@pytest.mark.parametrize("pm", [0.0, 0.1])
def test_log_case_on_tcgen05(nef, pm):
    """(alpha, beta) = (0, 1): a = log(x / yhat) < 0 where x < yhat.  The sentinel path
    must keep negative numerator weights (select on x, not a clamp at zero)."""
    ms, shape, ranks = "ir,jr,kr->ijk", (160, 144, 96), (32,)
    Y, _, _, init = _data("js", ms, shape, ranks, seed=35)
    Y = Y + 0.5
    M = (np.random.default_rng(36).random(shape) >= pm).astype(np.uint8) if pm > 0 else None
    plan = nef.Plan(ms, shape, ranks)
    assert all(L["tc"] for L in plan.describe()["lowerings"])
    F = [torch.from_numpy(f.copy()).cuda() for f in init]
    tr = plan.fit(torch.from_numpy(Y).cuda(), torch.from_numpy(M).cuda() if M is not None else None, 0.0, 1.0, F, 1)
    ref, rtr = O.fit(ms, Y, M, init, 0.0, 1.0, 1)
    errs = [_rel(g.cpu().numpy(), r) for g, r in zip(F, ref)]
    assert max(errs) <= FACTOR_RTOL, errs
    assert _rel(tr, rtr) <= TRACE_RTOL


# ------------------------------------------------------------------ split protocol (N2)
SPLIT_CASES = [("ir,jr,kr->ijk", (160, 144, 96), (32,), (1.0, 0.0)),
               ("ik,jk,tl,dl,kl->ijtd", (32, 48, 24, 40), (20, 10), (0.5, 0.0)),
               ("ir,jr,kr->ijk", (50, 40, 30), (5,), (1.0, 0.0))]


def _split_problem(ms, shape, ranks, seed):
    rng = np.random.default_rng(seed)
    fs = O.factor_shapes(ms, shape, ranks)
    yh = O.contract(ms, [rng.gamma(1.0, 1.0, s) for s in fs])
    Y = rng.poisson(yh / yh.mean() * 3.0).astype(np.float32)
    miss = rng.random(shape) < 0.02
    lab = split_labels(shape, 0.1, 0.05, seed=seed + 1, missing=miss)
    init = [rng.uniform(0.1, 1, s).astype(np.float32) for s in fs]
    return Y, lab, init


@pytest.mark.parametrize("case", SPLIT_CASES, ids=lambda c: "x".join(map(str, c[1])))
def test_split_fit_traces_and_counts(nef, case):
    """Train / validation / heldout loss sums of every sweep from the same streamed pass
    vs the oracle's fit_split; counts exact; factors after one sweep at the factor bar."""
    ms, shape, ranks, (al, be) = case
    Y, lab, init = _split_problem(ms, shape, ranks, 41)
    plan = nef.Plan(ms, shape, ranks)
    spec = nef.loss_spec("ab", al, be)
    ospec = O.make_loss("ab", al, be)
    Yd, Ld = torch.from_numpy(Y).cuda(), torch.from_numpy(lab).cuda()
    for T in (1, 8):
        F = [torch.from_numpy(f.copy()).cuda() for f in init]
        out = plan.fit_split(Yd, Ld, spec, F, max_iters=T, min_rel_decrease=-np.inf, val_patience=0)
        th, traces, counts, t, reason = O.fit_split(ms, Y, lab, init, ospec,
                                                    dict(max_iters=T, min_rel_decrease=-np.inf, val_patience=0))
        assert (out["sweeps"], out["reason"]) == (t, reason) == (T, "max_iters")
        assert out["counts"] == counts
        for q in range(3):
            assert _rel(out["traces"][q], traces[q]) <= TRACE_RTOL, (q, out["traces"][q], traces[q])
        if T == 1:
            errs = [_rel(g.cpu().numpy(), r) for g, r in zip(F, th)]
            assert max(errs) <= FACTOR_RTOL, errs


@pytest.mark.parametrize("case", SPLIT_CASES[::2], ids=lambda c: "x".join(map(str, c[1])))
def test_split_fit_ignores_non_train_values(nef, case):
    """Values at validation / heldout / excluded entries never reach the updates: NaN there leaves
    the factors and the train trace bit-identical."""
    ms, shape, ranks, (al, be) = case
    Y, lab, init = _split_problem(ms, shape, ranks, 43)
    plan = nef.Plan(ms, shape, ranks)
    spec = nef.loss_spec("ab", al, be)
    Ld = torch.from_numpy(lab).cuda()
    outs = []
    for Yv in (Y, np.where(lab == 1, Y, np.float32(np.nan)).astype(np.float32)):
        F = [torch.from_numpy(f.copy()).cuda() for f in init]
        o = plan.fit_split(torch.from_numpy(Yv).cuda(), Ld, spec, F, max_iters=4, min_rel_decrease=-np.inf,
                           val_patience=0)
        outs.append(([f.cpu() for f in F], o))
    for a, b in zip(outs[0][0], outs[1][0]):
        assert torch.equal(a, b)
    assert np.array_equal(outs[0][1]["traces"][0], outs[1][1]["traces"][0])
    # the heldout sums do read the heldout values (they changed)
    assert outs[1][1]["traces"][2][-1] != outs[0][1]["traces"][2][-1]


@pytest.mark.parametrize("case", SPLIT_CASES[::2], ids=lambda c: "x".join(map(str, c[1])))
def test_split_fit_stopping_rules(nef, case):
    """The paper's rules (R30-R32) on an over-parameterised fit: the library's stop sweep and
    reason are exactly the oracle's stop_decision applied to the library's own traces; the traces
    follow the oracle's within 1e-3; the returned factors are the iterate of the stop sweep."""
    ms, shape, ranks, (al, be) = case
    rng = np.random.default_rng(45)
    fs = O.factor_shapes(ms, shape, ranks)
    Y = rng.poisson(2.0 * O.contract(ms, [rng.gamma(1, 1, (s[0], 1)) for s in fs])).astype(np.float32)
    lab = split_labels(shape, 0.1, 0.3, seed=46)
    init = [rng.uniform(0.1, 1, s).astype(np.float32) for s in fs]
    plan = nef.Plan(ms, shape, ranks)
    spec, ospec = nef.loss_spec("ab", al, be), O.make_loss("ab", al, be)
    rule = dict(max_iters=400, min_rel_decrease=1e-6, val_patience=3)
    F = [torch.from_numpy(f.copy()).cuda() for f in init]
    Yd, Ld = torch.from_numpy(Y).cuda(), torch.from_numpy(lab).cuda()
    out = plan.fit_split(Yd, Ld, spec, F, **rule)
    t, tr = out["sweeps"], out["traces"]
    assert 0 < t < 400 and len(tr[0]) == t + 1
    assert out["reason"] == O.stop_decision(tr[0], tr[1], t, rule)
    assert all(O.stop_decision(tr[0], tr[1], k, rule) is None for k in range(t))
    k = min(t, 15)   # the oracle's trajectory over the first sweeps (seconds per sweep on the host)
    _, otr, _, _, _ = O.fit_split(ms, Y, lab, init, ospec, dict(rule, max_iters=k, min_rel_decrease=-np.inf,
                                                                 val_patience=0))
    for q in range(3):
        assert _rel(tr[q][:k + 1], otr[q]) <= TRACE_RTOL, q
    # the returned factors are the iterate after sweep t: a plain fit of t sweeps on the train mask
    G = [torch.from_numpy(f.copy()).cuda() for f in init]
    plan.fit(Yd, (Ld == 1).to(torch.uint8), al, be, G, t)
    for a, b in zip(F, G):
        assert _rel(a.cpu().numpy(), b.cpu().numpy()) <= 1e-5
