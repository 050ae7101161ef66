"""Parity of the tcgen05 / TMA streaming kernel (-m gpu) on shapes the planner routes to it
(TMA-legal strides, >= 64 rows, >= 32 columns per box), against the float64 oracle.

Shapes are small enough for the oracle yet span several 128-row blocks / 64-column tiles
with ragged tails, every TMA layout (rows-inner 2-D, cols-inner 2-D, 3-D) and both padded
bonds (32, 64).
"""
import numpy as np
import pytest

from oracle import nef_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

# (model, shape, ranks, (alpha, beta), mask, law)
TC_CASES = [
    ("ir,jr,kr->ijk", (160, 144, 96), (32,), (1.0, 0.0), 0.2, "poisson"),         # c3-like, KL
    ("ir,jr,kr->ijk", (144, 80, 112), (64,), (1.0, -0.5), 0.05, "gamma"),         # c5-like
    ("ia,jb,kc,abc->ijk", (96, 80, 64), (16, 16, 16), (1.0, 1.0), 0.1, "absnormal"),  # c2-like
    ("ik,jk,tl,dl,kl->ijtd", (32, 48, 24, 40), (20, 10), (0.5, 0.0), 0.0, "poisson"),  # c4-like
    ("ir,jr,kr->ijk", (130, 96, 64), (40,), (1.0, 0.5), 0.0, "gamma"),            # literal c5 reading, K=40
    ("ir,jr,kr->ijk", (256, 128, 64), (17,), (0.5, 0.5), 0.1, "gamma"),           # Hellinger, odd bond
    # inner column extents divisible by 64: direct-V path (table rows TMA-loaded into the V stage)
    ("ir,jr,kr->ijk", (130, 128, 192), (32,), (1.0, 0.0), 0.2, "poisson"),
    ("ir,jr,kr->ijk", (96, 192, 128), (64,), (1.0, -0.5), 0.05, "gamma"),
    ("ia,jb,kc,abc->ijk", (80, 128, 64), (16, 16, 16), (1.0, 1.0), 0.1, "absnormal"),
    ("ir,jr,kr->ijk", (64, 64, 128), (24,), (0.5, 0.0), 0.0, "poisson"),
    # layout 2 with a ragged 40-column inner block: direct-V runs spanning whole blocks
    ("ia,jb,kc,abc->ijk", (64, 72, 40), (8, 8, 8), (1.0, 1.0), 0.0, "absnormal"),
    # small column space merged into one table (K = 10: padded 16-byte row pitch)
    ("ik,jk,tl,dl,kl->ijtd", (40, 48, 16, 36), (12, 10), (0.5, 0.0), 0.0, "poisson"),
    # layout 1, CI % 32 != 0: two 2-D Y boxes per tile (the 3-D single-box view needs CI % 32 == 0)
    ("ir,jr,kr->ijk", (96, 130, 36), (32,), (1.0, -0.5), 0.05, "gamma"),
    # layout 1, CI % 64 == 32: the last tile's second 32-column half is out of bounds (zero fill)
    ("ir,jr,kr->ijk", (96, 104, 44), (32,), (1.0, 0.0), 0.2, "poisson"),
]


@pytest.fixture(scope="module")
def nef():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_02759_b200 import nef as n
    n.nef_set_kernel_policy(0)
    return n


def _data(ms, shape, ranks, pm, law, seed=11):
    rng = np.random.default_rng(seed)
    fs = O.factor_shapes(ms, shape, ranks)
    truth = [rng.gamma(1.0, 1.0, s) for s in fs]
    yh = O.contract(ms, truth)
    if law == "poisson":
        Y = rng.poisson(yh / yh.mean() * 3.0).astype(np.float32)
    elif law == "absnormal":
        Y = (yh + np.abs(rng.normal(0, 0.1, yh.shape))).astype(np.float32)
    else:
        Y = (yh * rng.gamma(10.0, 0.1, yh.shape)).astype(np.float32)
    M = (rng.random(shape) >= pm).astype(np.uint8) if pm > 0 else None
    init = [rng.uniform(0.1, 1.0, s).astype(np.float32) for s in fs]
    return Y, M, init


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30)))


def _dev(Y, M, init):
    return (torch.from_numpy(Y).cuda(), torch.from_numpy(M).cuda() if M is not None else None,
            [torch.from_numpy(f).cuda() for f in init])


@pytest.mark.parametrize("case", TC_CASES, ids=lambda c: "%s-%s" % (c[0], "x".join(map(str, c[1]))))
def test_routed_to_tcgen05(nef, case):
    ms, shape, ranks = case[:3]
    d = nef.Plan(ms, shape, ranks).describe()
    assert sum(L["tc"] for L in d["lowerings"]) >= 2


@pytest.mark.parametrize("case", TC_CASES, ids=lambda c: "%s-%s" % (c[0], "x".join(map(str, c[1]))))
def test_first_tile_pa(nef, case):
    """P_a = a(Y, Yhat) of CTA (0,0)'s first tile, dumped by the kernel, vs the oracle entry by entry."""
    ms, shape, ranks, (al, be), pm, law = case
    Y, M, init = _data(ms, shape, ranks, pm, law)
    plan = nef.Plan(ms, shape, ranks)
    d = plan.describe()
    Yd, Md, F = _dev(Y, M, init)
    yhat = np.maximum(O.contract(ms, init), O.EPS_Y)
    _, out = O.parse(ms)
    for L in d["lowerings"]:
        if not L["tc"] or (M is not None and not L["tc_mask_ok"]):
            continue   # (num_den streams the uint8 mask: its TMA view needs 16-byte strides)
        buf = torch.full((128 * 64,), -1.0, device="cuda")
        nef.nef_debug_dump(buf)
        try:
            plan.num_den(L["ell"], Yd, Md, al, be, F)
            torch.cuda.synchronize()
        finally:
            nef.nef_debug_dump(None)
        got = buf.cpu().numpy().reshape(128, 64)
        rows, cols = L["row_idx"], L["col_idx"]
        perm = [out.index(c) for c in rows + cols]
        R = L["tc_R"]
        Y2 = np.transpose(Y, perm).reshape(R, -1)
        yh2 = np.transpose(yhat, perm).reshape(R, -1)
        M2 = np.transpose(M, perm).reshape(R, -1) if M is not None else np.ones_like(Y2, dtype=np.uint8)
        # first tile's columns (layout 2: inner block 0 of outer index 0 = the same first 64 linear columns)
        ncol = min(64, L["tc_CI"] if L["tc_layout"] != 0 else L["tc_CO"])
        nrow = min(128, R)
        xs = np.where(M2 != 0, Y2, 1.0)[:nrow, :ncol]
        want = np.where(M2[:nrow, :ncol] != 0, O.a_fn(xs, yh2[:nrow, :ncol], al, be), 0.0)
        g = got[:nrow, :ncol]
        err = np.abs(g - want) / np.maximum(np.abs(want), 1e-6 * np.abs(want).max())
        assert err.max() < 3e-3, (L["ell"], L["tc_layout"], float(err.max()))
        assert np.all(got[nrow:, :] == 0) and np.all(got[:, ncol:] == 0)


@pytest.mark.parametrize("case", TC_CASES, ids=lambda c: "%s-%s" % (c[0], "x".join(map(str, c[1]))))
def test_one_sweep_and_trace(nef, case):
    ms, shape, ranks, (al, be), pm, law = case
    Y, M, init = _data(ms, shape, ranks, pm, law)
    plan = nef.Plan(ms, shape, ranks)
    Yd, Md, F = _dev(Y, M, init)
    tr1 = plan.fit(Yd, Md, al, be, F, 1)
    ref, rtr = O.fit(ms, Y, M, init, al, be, 1)
    for ell, (g, r) in enumerate(zip(F, ref)):
        assert _rel(g.cpu().numpy(), r) <= 1e-4, (ell, _rel(g.cpu().numpy(), r))
    assert _rel(tr1, rtr) <= 1e-3
    # 6 sweeps: trajectory within 1e-3
    Yd, Md, F = _dev(Y, M, init)
    tr = plan.fit(Yd, Md, al, be, F, 6)
    _, rtr = O.fit(ms, Y, M, init, al, be, 6)
    assert _rel(tr, rtr) <= 1e-3, _rel(tr, rtr)


@pytest.mark.parametrize("case", TC_CASES[:3], ids=lambda c: "%s-%s" % (c[0], "x".join(map(str, c[1]))))
def test_tc_matches_ffma_and_n_observed(nef, case):
    ms, shape, ranks, (al, be), pm, law = case
    Y, M, init = _data(ms, shape, ranks, pm, law)
    plan = nef.Plan(ms, shape, ranks)
    Yd, Md, F = _dev(Y, M, init)
    s_tc, n_tc = plan.loss(Yd, Md, al, be, F)
    nef.nef_set_kernel_policy(1)
    try:
        s_ff, n_ff = plan.loss(Yd, Md, al, be, F)
    finally:
        nef.nef_set_kernel_policy(0)
    rs, rn = O.loss(ms, Y, M, init, al, be)
    assert n_tc == n_ff == rn
    assert abs(s_tc - rs) <= 1e-4 * abs(rs) and abs(s_ff - rs) <= 1e-5 * abs(rs)


def test_direct_v_matches_generated_v(nef):
    """The direct-V path (TMA rows scaled in place) and the generated-V path form the same
    TF32-rounded V tiles, hence bit-identical numerators / denominators."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2602_02759_b200 import nef
from tests.test_gpu_tc import TC_CASES, _data, _dev
out = []
for ci in (6, 7, 8):
    ms, shape, ranks, (al, be), pm, law = TC_CASES[ci]
    Y, M, init = _data(ms, shape, ranks, pm, law)
    plan = nef.Plan(ms, shape, ranks)
    Yd, Md, F = _dev(Y, M, init)
    for ell in range(len(F)):
        n, d = plan.num_den(ell, Yd, Md, al, be, F)
        out.append(torch.cat([n.flatten(), d.flatten()]).cpu().numpy())
np.save(sys.argv[1], np.concatenate(out))
'''
    import os
    import tempfile
    res = []
    for flag in ("1", "0"):
        f = tempfile.mktemp(suffix=".npy")
        env = dict(os.environ, NEF_TC_VDIRECT=flag)
        subprocess.run([sys.executable, "-c", code, f], env=env, check=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        res.append(np.load(f))
    assert np.array_equal(res[0], res[1])


@pytest.mark.parametrize("case", [TC_CASES[0], TC_CASES[1], TC_CASES[7]], ids=["c3like", "c5like", "c5direct"])
def test_tc_mask_garbage_and_determinism(nef, case):
    ms, shape, ranks, (al, be), pm, law = case
    Y, M, init = _data(ms, shape, ranks, pm, law)
    plan = nef.Plan(ms, shape, ranks)
    Yd, Md, F0 = _dev(Y, M, init)
    F = [f.clone() for f in F0]
    tr = plan.fit(Yd, Md, al, be, F, 2)
    G = [f.clone() for f in F0]
    tr_again = plan.fit(Yd, Md, al, be, G, 2)
    for a, b in zip(F, G):
        assert torch.equal(a, b)
    assert np.array_equal(tr, tr_again)
    for fill in (float("nan"), float("inf"), 3e38):
        Y2 = torch.where(Md != 0, Yd, torch.full_like(Yd, fill))
        G = [f.clone() for f in F0]
        tr2 = plan.fit(Y2, Md, al, be, G, 2)
        for a, b in zip(F, G):
            assert torch.equal(a, b), fill
        assert np.array_equal(tr, tr2)
