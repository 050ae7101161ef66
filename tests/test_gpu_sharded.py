"""The sharded CUDA path executed on the GPU (-m gpu).

Virtual ranks on one GPU: for world in {2, 3, 8}, every rank's plan is split with
nef_plan_shard_host(rank, world) and runs the library's own kernels on its local slice of Y
(nef_num_den: side operands, streamed pass, reductions, epilogue on the LOCAL shape); the
partial A|B of factors without the shard mode are summed on the device - the all-reduce the
NCCL path performs - and every rank applies nef_apply_update to its local factors, in
Gauss-Seidel order.  One sweep is compared with the float64 oracle on the whole tensor (factor
bar 1e-4) and with the unsharded GPU fit; per-rank nef_loss partial sums and observed counts
must add up to the global loss / count.  The ranks here never wait on one another (no
collective kernel runs on the single GPU).  A real 2-process NCCL run follows (torchrun, >= 2
GPUs; skipped otherwise)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from nef_inputs import generate_numpy
from oracle import nef_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


def _slice(t, axis, b, n):
    return t.narrow(axis, b, n).clone()   # own allocation: the ABI wants 16-byte aligned Y


# (config, shape): c5 / c3 (tcgen05, masked), c2 (Tucker with the core, tcgen05), c4 (5 factors,
# shard mode d), c1 (CUDA-core)
SHARD_CASES = [("c5", (144, 96, 80)), ("c3", (150, 133, 70)), ("c2", (96, 80, 64)), ("c4", (30, 27, 24, 37)),
               ("c1", None)]


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("name,shape", SHARD_CASES, ids=[c[0] for c in SHARD_CASES])
def test_virtual_ranks_one_sweep(nef, name, shape, world):
    d = generate_numpy(name, shape=shape)
    ms, al, be = d["model"], d["alpha"], d["beta"]
    ops, out = O.parse(ms)
    Y = torch.from_numpy(d["Y"]).cuda()
    M = torch.from_numpy(d["mask"]).cuda() if d["mask"] is not None else None
    plans, loc = [], []
    for r in range(world):
        p = nef.Plan(ms, d["shape"], d["ranks"])
        p.shard_host(r, world)
        plans.append(p)
        i = p.info
        loc.append((i["shard_mode"], i["local_begin"], i["local_len"]))
    sm = loc[0][0]
    letter = out[sm]
    has = plans[0].describe()["factor_has_shard"]
    assert [letter in op for op in ops] == has and any(has)
    assert sum(n for _, _, n in loc) == d["shape"][sm]
    Yl = [_slice(Y, sm, b, n) for _, b, n in loc]
    Ml = [_slice(M, sm, b, n) if M is not None else None for _, b, n in loc]
    F = [[_slice(torch.from_numpy(f).cuda(), op.index(letter), b, n) if letter in op
          else torch.from_numpy(f.copy()).cuda() for f, op in zip(d["init"], ops)] for _, b, n in loc]
    # losses and counts before the sweep: per-rank partials add up to the global values
    parts = [plans[r].loss(Yl[r], Ml[r], al, be, F[r]) for r in range(world)]
    rs, rn = O.loss(ms, d["Y"], d["mask"], d["init"], al, be)
    assert sum(n for _, n in parts) == rn
    assert abs(sum(s for s, _ in parts) - rs) <= 1e-5 * abs(rs)
    # one Gauss-Seidel sweep: local pass on every rank, device sum of the partials, local updates
    for ell, op in enumerate(ops):
        nd = [plans[r].num_den(ell, Yl[r], Ml[r], al, be, F[r]) for r in range(world)]
        if not has[ell]:
            num = torch.stack([x[0] for x in nd]).sum(0)
            den = torch.stack([x[1] for x in nd]).sum(0)
            nd = [(num, den)] * world
        for r in range(world):
            plans[r].apply_update(ell, al, be, F[r], nd[r][0], nd[r][1])
    # replicated factors are identical on every rank; sharded ones reassemble the global factor
    got = []
    for ell, op in enumerate(ops):
        if has[ell]:
            got.append(torch.cat([F[r][ell] for r in range(world)], dim=op.index(letter)).cpu().numpy())
        else:
            for r in range(1, world):
                assert torch.equal(F[r][ell], F[0][ell])
            got.append(F[0][ell].cpu().numpy())
    ref, _ = O.fit(ms, d["Y"], d["mask"], d["init"], al, be, 1)
    errs = [_rel(g, r) for g, r in zip(got, ref)]
    assert max(errs) <= 1e-4, errs
    # and against the unsharded GPU fit of the same sweep
    plan = nef.Plan(ms, d["shape"], d["ranks"])
    G = [torch.from_numpy(f.copy()).cuda() for f in d["init"]]
    plan.fit(Y, M, al, be, G, 1)
    errs = [_rel(g, h.cpu().numpy()) for g, h in zip(got, G)]
    assert max(errs) <= 5e-5, errs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_torchrun_two_ranks_nccl():
    """Two processes, one GPU each, NCCL communicator from nef_nccl_unique_id: the sharded fit
    (A|B and loss all-reduced inside libnef) matches the oracle on the whole tensor."""
    script = os.path.join(ROOT, "tests", "_shard_worker.py")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), script]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "SHARD_OK" in r.stdout
