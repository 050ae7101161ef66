"""Batched random restarts (N4) on the GPU (-m gpu): S fits of the same data from
different initialisations, every streamed pass one launch for all restarts (launch z index =
restart, the Y tiles read together).  Each restart must match the float64 oracle's fit from its
own initialisation (factor bar 1e-4 after one sweep, trajectory bar 1e-3) and the library's own
single fit from the same initialisation."""
import numpy as np
import pytest

from nef_inputs import generate_numpy
from oracle import nef_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


CASES = [("c5", (144, 96, 80), 3), ("c3", (160, 144, 96), 2), ("c2", (80, 72, 64), 4), ("c4", (32, 48, 24, 40), 3),
         ("c1", None, 2)]


@pytest.mark.parametrize("name,shape,S", CASES, ids=[c[0] for c in CASES])
def test_restarts_match_oracle_and_single_fits(nef, name, shape, S, record_err):
    d = generate_numpy(name, shape=shape)
    ms, al, be = d["model"], d["alpha"], d["beta"]
    rng = np.random.default_rng(77)
    inits = [d["init"]] + [[rng.uniform(0.1, 1.0, f.shape).astype(np.float32) for f in d["init"]] for _ in range(S - 1)]
    plan = nef.Plan(ms, d["shape"], d["ranks"])
    tc = [L["tc"] for L in plan.describe()["lowerings"]]
    Y = torch.from_numpy(d["Y"]).cuda()
    M = torch.from_numpy(d["mask"]).cuda() if d["mask"] is not None else None
    spec = nef.loss_spec("ab", al, be)
    for iters in (1, 5):
        Fs = [[torch.from_numpy(f.copy()).cuda() for f in init] for init in inits]
        tr = plan.fit_restarts(Y, M, spec, Fs, iters)
        assert tr.shape == (S, iters + 1)
        for r in range(S):
            ref, rtr = O.fit(ms, d["Y"], d["mask"], inits[r], al, be, iters)
            et = _rel(tr[r], rtr)
            assert et <= 1e-3, (r, et)
            G = [torch.from_numpy(f.copy()).cuda() for f in inits[r]]
            gtr = plan.fit(Y, M, al, be, G, iters)
            # the batched launch splits the column range into other chunks than a single fit
            # (fewer CTAs per restart): same arithmetic, other fp32 summation partition
            assert _rel(tr[r], gtr) <= 1e-4, (r, tr[r], gtr)
            es = max(_rel(a.cpu().numpy(), b.cpu().numpy()) for a, b in zip(Fs[r], G))
            assert es <= 1e-4 * iters, (r, es)
            if iters == 1:
                ef = max(_rel(g.cpu().numpy(), x) for g, x in zip(Fs[r], ref))
                record_err(ef, 1e-4, "restart %d of %d factors after 1 sweep (tc %s)" % (r, S, tc))
                assert ef <= 1e-4, (r, ef)
