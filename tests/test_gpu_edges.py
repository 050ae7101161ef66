"""Degenerate and edge cases of the CUDA path against the float64 oracle (-m gpu), on shapes
routed to the tcgen05 kernel and to the CUDA-core kernel:

* a factor row / slab with no observed entry: numerator = denominator = 0, multiplier 1
  (R10) - the row must come back bit-identical, everything else at the parity bar;
* an all-missing mask: loss 0, n_observed 0, factors untouched;
* rank 1 (K = 1: padded 16-byte table rows) and unit modes;
* mostly-zero data (x = 0 entries: a = 0, loss terms of the x -> 0 limit).
"""
import os

import numpy as np
import pytest

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


def _problem(ms, shape, ranks, seed, zero_frac=0.0):
    rng = np.random.default_rng(seed)
    fs = O.factor_shapes(ms, shape, ranks)
    truth = [rng.gamma(1.0, 1.0, s) for s in fs]
    Y = rng.poisson(O.contract(ms, truth)).astype(np.float32) + 0.25
    if zero_frac > 0:
        Y[rng.random(shape) < zero_frac] = 0.0
    init = [rng.uniform(0.1, 1, s).astype(np.float32) for s in fs]
    return Y, init


def _fit(nef, ms, shape, ranks, Y, M, init, ab, iters):
    plan = nef.Plan(ms, shape, ranks)
    F = [torch.from_numpy(f.copy()).cuda() for f in init]
    Md = torch.from_numpy(M).cuda() if M is not None else None
    tr = plan.fit(torch.from_numpy(Y).cuda(), Md, ab[0], ab[1], F, iters)
    torch.cuda.synchronize()
    return plan, [f.cpu().numpy() for f in F], tr


# (model, shape, ranks, (alpha, beta)): tcgen05-routed CP shapes and a CUDA-core one
SLAB_CASES = [
    ("ir,jr,kr->ijk", (144, 80, 112), (64,), (1.0, -0.5)),   # c5-like, tcgen05
    ("ir,jr,kr->ijk", (160, 144, 96), (32,), (1.0, 0.0)),    # c3-like, tcgen05
    ("ir,jr,kr->ijk", (50, 40, 30), (5,), (1.0, 0.0)),       # c1 shape, CUDA-core
]


@pytest.mark.parametrize("case", SLAB_CASES, ids=lambda c: "x".join(map(str, c[1])))
def test_unobserved_slabs_keep_their_rows(nef, case):
    ms, shape, ranks, ab = case
    Y, init = _problem(ms, shape, ranks, seed=5)
    rng = np.random.default_rng(6)
    M = (rng.random(shape) > 0.1).astype(np.uint8)
    M[5, :, :] = 0          # factor 0 row 5: no observed entry
    M[:, 7, :] = 0          # factor 1 row 7
    M[:, :, 0] = 0          # factor 2 row 0
    plan, F, tr = _fit(nef, ms, shape, ranks, Y, M, init, ab, 1)
    assert plan.describe()["lowerings"][0]["tc"] == (shape[0] > 64)
    ref, rtr = O.fit(ms, Y, M, init, ab[0], ab[1], 1)
    for ell, (g, r) in enumerate(zip(F, ref)):
        assert _rel(g, r) <= FACTOR_RTOL, (ell, _rel(g, r))
    # R10: multiplier 1 -> bit-identical rows
    assert np.array_equal(F[0][5], init[0][5])
    assert np.array_equal(F[1][7], init[1][7])
    assert np.array_equal(F[2][0], init[2][0])
    assert _rel(tr, rtr) <= TRACE_RTOL


@pytest.mark.parametrize("case", SLAB_CASES, ids=lambda c: "x".join(map(str, c[1])))
def test_all_missing(nef, case):
    ms, shape, ranks, ab = case
    Y, init = _problem(ms, shape, ranks, seed=7)
    M = np.zeros(shape, dtype=np.uint8)
    plan, F, tr = _fit(nef, ms, shape, ranks, Y, M, init, ab, 2)
    assert list(tr) == [0.0, 0.0, 0.0]
    for g, f in zip(F, init):
        assert np.array_equal(g, f)
    s, n = plan.loss(torch.from_numpy(Y).cuda(), torch.from_numpy(M).cuda(), ab[0], ab[1],
                     [torch.from_numpy(f).cuda() for f in init])
    assert s == 0.0 and n == 0


@pytest.mark.parametrize("ms,shape,ranks,ab,pm", [
    ("ir,jr,kr->ijk", (160, 64, 96), (1,), (1.0, -0.5), 0.05),    # rank 1
    ("ir,jr,kr->ijk", (130, 1, 192), (16,), (1.0, 0.0), 0.2),     # unit middle mode
    ("ir,jr,kr->ijk", (1, 96, 128), (8,), (1.0, 1.0), 0.0),       # unit leading mode
])
def test_rank1_and_unit_modes(nef, ms, shape, ranks, ab, pm):
    Y, init = _problem(ms, shape, ranks, seed=9)
    M = (np.random.default_rng(10).random(shape) >= pm).astype(np.uint8) if pm > 0 else None
    _, F, tr = _fit(nef, ms, shape, ranks, Y, M, init, ab, 1)   # the factor bar: after 1 sweep
    ref, rtr = O.fit(ms, Y, M, init, ab[0], ab[1], 1)
    for ell, (g, r) in enumerate(zip(F, ref)):
        assert _rel(g, r) <= FACTOR_RTOL, (ell, _rel(g, r))
    _, _, tr = _fit(nef, ms, shape, ranks, Y, M, init, ab, 4)
    _, rtr = O.fit(ms, Y, M, init, ab[0], ab[1], 4)
    assert _rel(tr, rtr) <= TRACE_RTOL


@pytest.mark.parametrize("ab", [(1.0, 0.0), (1.0, -0.5), (0.5, 0.0), (1.0, 1.0)])
def test_mostly_zero_data(nef, ab):
    ms, shape, ranks = "ir,jr,kr->ijk", (144, 80, 112), (32,)
    Y, init = _problem(ms, shape, ranks, seed=11, zero_frac=0.8)
    M = (np.random.default_rng(12).random(shape) > 0.1).astype(np.uint8)
    _, F, tr = _fit(nef, ms, shape, ranks, Y, M, init, ab, 1)
    ref, rtr = O.fit(ms, Y, M, init, ab[0], ab[1], 1)
    for ell, (g, r) in enumerate(zip(F, ref)):
        assert _rel(g, r) <= FACTOR_RTOL, (ell, _rel(g, r))
    assert _rel(tr, rtr) <= TRACE_RTOL


def test_nccl_path_on_one_rank(nef, monkeypatch):
    """The multi-GPU path with its NCCL calls, on a 1-rank communicator (NEF_NCCL_FORCE=1):
    libnccl loaded, ncclCommInitRank, the all-reduces of the numerator/denominator partials and
    of the loss slots on the workspace - an identity at one rank, so factors and trace must be
    bit-identical to the unsharded fit."""
    from nef_inputs import CONFIGS, generate_numpy
    d = generate_numpy("c5")
    cfg = CONFIGS["c5"]
    Y = torch.from_numpy(d["Y"]).cuda()
    M = torch.from_numpy(d["mask"]).cuda()
    runs = []
    for shard in (False, True):
        plan = nef.Plan(d["model"], d["shape"], d["ranks"])
        if shard:
            monkeypatch.setenv("NEF_NCCL_FORCE", "1")
            plan.shard(0, 1, nef.nef_nccl_unique_id())
            monkeypatch.delenv("NEF_NCCL_FORCE")
            assert plan.info["shard_mode"] == 0
        F = [torch.from_numpy(f.copy()).cuda() for f in d["init"]]
        tr = plan.fit(Y, M, cfg.alpha, cfg.beta, F, 2)
        s, n = plan.loss(Y, M, cfg.alpha, cfg.beta, F)
        torch.cuda.synchronize()
        runs.append(([f.cpu() for f in F], list(tr), s, n))
    (Fa, ta, sa, na), (Fb, tb, sb, nb) = runs
    for a, b in zip(Fa, Fb):
        assert torch.equal(a, b)
    assert ta == tb and sa == sb and na == nb


def _random_cases(n, seed):
    """Seeded random CP / Tucker / 4-way problems that the planner sends to the tcgen05 kernel:
    random bonds 1..64 (KB 32 and 64, K % 4 != 0 padding), ragged row and column tails, random
    (alpha, beta) among the specialised pairs and the generic one, with and without a mask."""
    rng = np.random.default_rng(seed)
    pairs = [(1.0, 0.0), (1.0, -0.5), (0.5, 0.0), (1.0, 1.0), (0.5, 0.5), (1.0, 0.5), (1.3, -0.2)]
    out = []
    while len(out) < n:
        kind = rng.integers(0, 3)
        if kind == 0:
            ms = "ir,jr,kr->ijk"
            shape = tuple(int(x) for x in rng.integers(64, 200, 3))
            ranks = (int(rng.integers(1, 65)),)
        elif kind == 1:
            ms = "ia,jb,kc,abc->ijk"
            shape = tuple(int(x) for x in rng.integers(64, 160, 3))
            ranks = tuple(int(x) for x in rng.integers(2, 17, 3))
        else:
            ms = "ik,jk,tl,dl,kl->ijtd"
            shape = (int(rng.integers(16, 48)), int(rng.integers(16, 48)), int(rng.integers(8, 24)), int(rng.integers(32, 80)))
            ranks = (int(rng.integers(2, 20)), int(rng.integers(2, 12)))
        if rng.random() < 0.7:   # TMA-legal strides (multiples of 4 / 16 bytes) -> tcgen05 path
            shape = tuple(int(x) // 4 * 4 if i > 0 else int(x) for i, x in enumerate(shape))
        ab = pairs[int(rng.integers(0, len(pairs)))]
        pm = float(rng.choice([0.0, 0.05, 0.3]))
        out.append((ms, shape, ranks, ab, pm, int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("case", _random_cases(int(os.environ.get("NEF_RANDOM_CASES", "40")),
                                                int(os.environ.get("NEF_RANDOM_SEED", "2026"))), ids=lambda c: "%s-%s-K%s" % (
    c[0].split("->")[0].count(",") + 1, "x".join(map(str, c[1])), ",".join(map(str, c[2]))))
def test_random_problems(nef, case):
    ms, shape, ranks, ab, pm, seed = case
    rng = np.random.default_rng(seed)
    fs = O.factor_shapes(ms, shape, ranks)
    truth = [rng.gamma(1.0, 1.0, s) for s in fs]
    Y = (rng.poisson(O.contract(ms, truth)) + rng.gamma(2.0, 0.05, shape)).astype(np.float32)
    M = (rng.random(shape) >= pm).astype(np.uint8) if pm > 0 else None
    init = [rng.uniform(0.1, 1, s).astype(np.float32) for s in fs]
    _, F, tr = _fit(nef, ms, shape, ranks, Y, M, init, ab, 1)
    ref, rtr = O.fit(ms, Y, M, init, ab[0], ab[1], 1)
    for ell, (g, r) in enumerate(zip(F, ref)):
        assert _rel(g, r) <= FACTOR_RTOL, (ell, _rel(g, r))
    assert _rel(tr, rtr) <= TRACE_RTOL


@pytest.mark.parametrize("ab", [(1.0, 0.0), (1.0, 1.0), (0.5, 0.0)])
def test_negative_zero_in_unmasked_y(nef, ab):
    """An observed -0.0 is a zero, not a missing entry: unmasked Y is streamed as is
    by the tcgen05 kernel, which must not read 'missing' from its sign bit.  Same factors as the
    oracle (and as the fit on +0.0) with a third of the zeros negated."""
    ms, shape, ranks = "ir,jr,kr->ijk", (144, 80, 112), (32,)
    Y, init = _problem(ms, shape, ranks, seed=21, zero_frac=0.5)
    Yn = Y.copy()
    z = np.argwhere(Yn == 0)
    sel = z[np.random.default_rng(22).random(len(z)) < 0.33]
    Yn[tuple(sel.T)] = -0.0
    assert np.signbit(Yn).sum() > 1000 and not (Yn < 0).any()
    plan, F, tr = _fit(nef, ms, shape, ranks, Yn, None, init, ab, 1)
    assert all(L["tc"] for L in plan.describe()["lowerings"])
    _, F0, tr0 = _fit(nef, ms, shape, ranks, Y, None, init, ab, 1)
    for a, b in zip(F, F0):
        assert np.array_equal(a, b)
    assert np.array_equal(tr, tr0)
    ref, rtr = O.fit(ms, Yn, None, init, ab[0], ab[1], 1)
    errs = [_rel(g, r) for g, r in zip(F, ref)]
    assert max(errs) <= FACTOR_RTOL, errs
    assert _rel(tr, rtr) <= TRACE_RTOL


def test_six_mode_cp_merged_tables(nef):
    """6-mode CP: five column factors per lowering, merged by the planner to <= 4 tables (the
    kernels' limit); parity with the oracle after one sweep."""
    ms, shape, ranks = "ar,br,cr,dr,er,fr->abcdef", (12, 8, 6, 9, 8, 7), (5,)
    Y, init = _problem(ms, shape, ranks, seed=23)
    M = (np.random.default_rng(24).random(shape) > 0.1).astype(np.uint8)
    plan, F, tr = _fit(nef, ms, shape, ranks, Y, M, init, (1.0, 0.0), 1)
    assert all(len(L["tables"]) <= 4 for L in plan.describe()["lowerings"])
    ref, rtr = O.fit(ms, Y, M, init, 1.0, 0.0, 1)
    errs = [_rel(g, r) for g, r in zip(F, ref)]
    assert max(errs) <= FACTOR_RTOL, errs
    assert _rel(tr, rtr) <= TRACE_RTOL


def test_bond_above_64_last_resort(nef):
    """A CP of rank 80 exceeds both kernels' bond limit: the planner's last-resort lowering
    (U = Yhat materialised, K = 1) runs it; parity with the oracle."""
    ms, shape, ranks = "ir,jr,kr->ijk", (20, 24, 16), (80,)
    Y, init = _problem(ms, shape, ranks, seed=25)
    plan, F, tr = _fit(nef, ms, shape, ranks, Y, None, init, (1.0, 0.0), 2)
    assert all(L["K"] == 1 for L in plan.describe()["lowerings"])
    ref, rtr = O.fit(ms, Y, None, init, 1.0, 0.0, 2)
    errs = [_rel(g, r) for g, r in zip(F, ref)]
    assert max(errs) <= 2e-4, errs     # two sweeps
    assert _rel(tr, rtr) <= TRACE_RTOL


GUARD_CASES = [("ir,jr,kr->ijk", (13, 17, 19), (3,), (1.0, 0.0), 0.1),          # CUDA-core, odd primes
               ("ir,jr,kr->ijk", (130, 96, 68), (40,), (1.0, -0.5), 0.05),     # tcgen05, row / column tails
               ("ir,jr,kr->ijk", (96, 104, 44), (32,), (1.0, 0.0), 0.0),       # layout-1 half box out of bounds
               ("ia,jb,kc,abc->ijk", (64, 72, 40), (8, 8, 8), (1.0, 1.0), 0.1),  # layout 2, split P_a
               ("ik,jk,tl,dl,kl->ijtd", (32, 48, 24, 40), (20, 10), (0.5, 0.0), 0.0)]


@pytest.mark.parametrize("case", GUARD_CASES, ids=lambda c: "x".join(map(str, c[1])))
def test_no_out_of_bounds_writes(nef, case):
    """Out-of-bounds write check (compute-sanitizer is closed on this GPU pool): Y, the mask, every
    factor and the workspace sit inside one allocation between guard bands of a NaN bit pattern;
    a fit, a split fit, nef_num_den and nef_loss must leave every guard byte, Y and the mask
    untouched and write only inside the workspace and the factors."""
    ms, shape, ranks, ab, pm = case
    Y, init = _problem(ms, shape, ranks, seed=51)
    M = (np.random.default_rng(52).random(shape) >= pm).astype(np.uint8) if pm > 0 else None
    plan = nef.Plan(ms, shape, ranks)
    G = 1 << 16                                               # guard band, bytes (256-aligned)
    sizes = [Y.nbytes, M.nbytes if M is not None else 0] + [f.nbytes for f in init] + [plan.info["workspace_bytes"]]
    offs, o = [], G
    for n in sizes:
        offs.append(o)
        o += (n + 255) // 256 * 256 + G
    buf = torch.full((o // 4,), 0x7fc0dead, dtype=torch.int32, device="cuda")
    raw = buf.view(torch.uint8)

    def view(i, dtype, shp):
        n = int(np.prod(shp)) * torch.tensor([], dtype=dtype).element_size()
        return raw[offs[i]:offs[i] + n].view(dtype).view(shp)

    Yd = view(0, torch.float32, shape)
    Yd.copy_(torch.from_numpy(Y))
    Md = None
    if M is not None:
        Md = view(1, torch.uint8, shape)
        Md.copy_(torch.from_numpy(M))
    F = [view(2 + l, torch.float32, f.shape) for l, f in enumerate(init)]
    for f, h in zip(F, init):
        f.copy_(torch.from_numpy(h))
    plan._ws = view(len(sizes) - 1, torch.uint8, (sizes[-1],))
    guard = torch.ones(o, dtype=torch.bool, device="cuda")
    for off, n in zip(offs, sizes):
        guard[off:off + n] = False
    before = raw.clone()
    plan.fit(Yd, Md, ab[0], ab[1], F, 2)
    for ell in range(len(F)):
        plan.num_den(ell, Yd, Md, ab[0], ab[1], F)
    plan.loss(Yd, Md, ab[0], ab[1], F)
    if M is not None:
        lab = torch.where(Md != 0, torch.ones_like(Md), torch.full_like(Md, 3))
        plan.fit_split(Yd, lab.contiguous(), nef.loss_spec("ab", ab[0], ab[1]), F, max_iters=2)
    torch.cuda.synchronize()
    assert torch.equal(raw[guard], before[guard]), "guard band written"
    assert torch.equal(Yd.cpu(), torch.from_numpy(Y))
    if M is not None:
        assert torch.equal(Md.cpu(), torch.from_numpy(M))


# models whose sweeps reuse a side operand across updates (planner sweep_reuse): c2's Tucker
# (update 3's U is update 2's table), c4's spatiotemporal model, LR-Tucker and a 6-mode CP
REUSE_CASES = [
    ("ia,jb,kc,abc->ijk", (70, 45, 52), (16, 16, 16), (1.0, 1.0), 0.1),
    ("ik,jk,tl,dl,kl->ijtd", (26, 26, 12, 36), (20, 10), (0.5, 0.0), 0.0),
    ("ia,jb,kc,ar,br,cr->ijk", (40, 36, 44), (4, 5, 6, 3), (1.0, 0.0), 0.05),
    ("ar,br,cr,dr,er,fr->abcdef", (6, 7, 5, 6, 4, 8), (5,), (1.0, 0.0), 0.0),
]


@pytest.mark.parametrize("case", REUSE_CASES, ids=lambda c: c[0].split("->")[0])
def test_sweep_reuse_bit_identical(nef, case):
    """Side-operand reuse inside a sweep skips launches whose results an earlier
    update of the same sweep left in the workspace: the fit must be bit-identical to the fit
    that recomputes every side operand (kernel policy bit 2), through the sweep graph and
    through plain launches, and match the oracle at the parity bar."""
    ms, shape, ranks, ab, pm = case
    Y, init = _problem(ms, shape, ranks, 7)
    M = (np.random.default_rng(8).random(shape) >= pm).astype(np.uint8) if pm > 0 else None
    plan = nef.Plan(ms, shape, ranks)
    assert any(L["reuse_u"] or any(L["reuse_tab"]) for L in plan.describe()["lowerings"])
    runs = {}
    try:
        for pol in (0, 4, 2, 6):
            nef.nef_set_kernel_policy(pol)
            runs[pol] = _fit(nef, ms, shape, ranks, Y, M, init, ab, 3)
    finally:
        nef.nef_set_kernel_policy(0)
    for pol in (4, 2, 6):
        for a, b in zip(runs[0][1], runs[pol][1]):
            assert np.array_equal(a, b), pol
        assert list(runs[0][2]) == list(runs[pol][2]), pol
    ref, rtr = O.fit(ms, Y, M, init, ab[0], ab[1], 3)
    assert _rel(runs[0][2], rtr) <= TRACE_RTOL, _rel(runs[0][2], rtr)
    _, F1, _ = _fit(nef, ms, shape, ranks, Y, M, init, ab, 1)
    ref1, _ = O.fit(ms, Y, M, init, ab[0], ab[1], 1)
    err = max(_rel(g, r) for g, r in zip(F1, ref1))
    assert err <= FACTOR_RTOL, err
