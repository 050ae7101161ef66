"""Full-size parity (-m gpu) at BASELINE.json's sizes, in the launch configuration bench.py
times (one nef_fit sweep, device-resident inputs, the sentinel path for masked configs), on
outputs the float64 oracle can compute one by one: after one sweep, sampled rows of every factor
that owns an observed mode are recomputed by the oracle from that row's slab of Y (index fixed
along the factor's mode) with the same inputs the sweep used (factors before ell as updated by
the GPU, factors after ell at their initial values: Gauss-Seidel order).  A row of
factor ell depends only on its slab, so this is the exact per-row update.  The loss trace is
checked for the MM guarantee (non-increasing, Theorem 2) and n_observed exactly against the mask.
"""
import numpy as np
import pytest

from nef_inputs import CONFIGS, generate_torch
from oracle import nef_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FACTOR_RTOL = 1e-4


@pytest.fixture(scope="module")
def nef():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_02759_b200 import nef as n
    return n


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30)))


@pytest.mark.parametrize("name", ["c3", "c5", "c4"])
def test_fullsize_one_sweep_sampled_rows(nef, name):
    cfg = CONFIGS[name]
    dev = torch.device("cuda")
    d = generate_torch(name, dev)
    Y, M = d["Y"], d["mask"]
    init = [f.clone() for f in d["init"]]
    F = [f.clone() for f in d["init"]]
    plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
    tr = plan.fit(Y, M, cfg.alpha, cfg.beta, F, 1)
    torch.cuda.synchronize()
    assert np.all(np.isfinite(tr)) and tr[1] <= tr[0] * (1 + 1e-6), tr
    ops, out = O.parse(cfg.model)
    rng = np.random.default_rng(7)
    checked = 0
    for ell, op in enumerate(ops):
        obs = [c for c in op if c in out]
        if not obs:
            continue                                   # purely contracted factor (c4's kl): no slab
        letter = obs[0]
        mode, axis = out.index(letter), op.index(letter)
        n = cfg.shape[mode]
        rows = sorted(set([0, n - 1] + list(rng.integers(0, n, 2))))
        # inputs of update ell within the sweep: updated factors before ell, initial after
        cur = [(F[k] if k < ell else init[k]).cpu().numpy().astype(np.float64) for k in range(len(ops))]
        got = F[ell].cpu().numpy()
        for i in rows:
            Ys = Y.select(mode, i).unsqueeze(mode).cpu().numpy().astype(np.float64)
            Ms = M.select(mode, i).unsqueeze(mode).cpu().numpy() if M is not None else None
            fs = list(cur)
            fs[ell] = np.take(cur[ell], [i], axis=axis)
            want = O.update_factor(cfg.model, Ys, Ms, fs, ell, cfg.alpha, cfg.beta)
            g = np.take(got, [i], axis=axis)
            assert _rel(g, want) <= FACTOR_RTOL, (name, ell, i, _rel(g, want))
            checked += 1
    assert checked >= 6


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_fullsize_n_observed_exact(nef, name):
    cfg = CONFIGS[name]
    d = generate_torch(name, torch.device("cuda"))
    plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
    loss, n_obs = plan.loss(d["Y"], d["mask"], cfg.alpha, cfg.beta, d["init"])
    assert n_obs == int(d["mask"].sum(dtype=torch.int64).item())
    assert np.isfinite(loss) and loss > 0
