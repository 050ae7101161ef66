"""Multi-GPU host logic on CPU (world size 2, gloo): the split of Y along its largest mode
 as the library plans it (nef_plan_shard_host: local range and
which factors need their A|B summed over ranks), checked by running the float64 oracle on each
rank's local tensor, all-reducing the partial A|B of the factors that do not contain the shard
mode over gloo, and comparing with the oracle's A|B on the whole tensor.  No GPU: the library is
used for planning only; the arithmetic here is the oracle's (test infrastructure)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
dist = pytest.importorskip("torch.distributed")

from nef_inputs import generate_numpy  # noqa: E402
from oracle import nef_oracle as O  # noqa: E402

CASES = ["c1", "c2", "c4"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _take(a, axis, b, n):
    return np.take(a, np.arange(b, b + n), axis=axis)


def _worker(rank, world, port, name, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_02759_b200 import nef
        d = generate_numpy(name)
        ms, Y, M, F = d["model"], d["Y"].astype(np.float64), d["mask"], [f.astype(np.float64) for f in d["init"]]
        plan = nef.Plan(ms, d["shape"], d["ranks"])
        plan.shard_host(rank, world)
        desc = plan.describe()
        info = plan.info
        sm, b, n = desc["shard_mode"], info["local_begin"], info["local_len"]
        ops, outs = O.parse(ms)
        letter = outs[sm]
        Yl = _take(Y, sm, b, n)
        Ml = _take(M, sm, b, n) if M is not None else None
        Fl = [_take(f, op.index(letter), b, n) if letter in op else f for f, op in zip(F, ops)]
        assert tuple(plan.local_shape) == Yl.shape
        res = {"rank": rank, "range": (b, n), "has_shard": desc["factor_has_shard"], "err": []}
        for ell, op in enumerate(ops):
            A, B = O.numerator_denominator(ms, Yl, Ml, Fl, ell, d["alpha"], d["beta"])
            assert (letter in op) == desc["factor_has_shard"][ell]
            if not desc["factor_has_shard"][ell]:
                t = torch.from_numpy(np.stack([A, B]))
                dist.all_reduce(t)
                A, B = t[0].numpy(), t[1].numpy()
            Ag, Bg = O.numerator_denominator(ms, Y, M, F, ell, d["alpha"], d["beta"])
            if letter in op:
                Ag, Bg = _take(Ag, op.index(letter), b, n), _take(Bg, op.index(letter), b, n)
            res["err"].append(max(float(np.max(np.abs(A - Ag) / np.maximum(np.abs(Ag), 1e-300))),
                                  float(np.max(np.abs(B - Bg) / np.maximum(np.abs(Bg), 1e-300)))))
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", CASES)
def test_world2_partial_sums_match_whole_tensor(name):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0, "worker failed"
    r0, r1 = out[0], out[1]
    # the two local ranges partition the shard mode exactly once
    (b0, n0), (b1, n1) = r0["range"], r1["range"]
    assert b0 == 0 and b1 == n0 and n0 - n1 in (0, 1)
    assert r0["has_shard"] == r1["has_shard"] and any(r0["has_shard"]) and not all(r0["has_shard"])
    for r in (r0, r1):
        assert max(r["err"]) < 1e-12, r["err"]


def test_shard_ranges_cover_every_index():
    from paper_2602_02759_b200 import nef
    for world in (1, 2, 3, 4, 7, 8):
        seen = []
        for rank in range(world):
            p = nef.Plan("ir,jr,kr->ijk", (13, 29, 17), (3,))
            p.shard_host(rank, world)
            i = p.info
            assert i["shard_mode"] == 1
            seen += list(range(i["local_begin"], i["local_begin"] + i["local_len"]))
        assert seen == list(range(29))


def test_host_sharded_plan_refuses_collective_calls_without_gpu():
    from paper_2602_02759_b200 import nef
    p = nef.Plan("ir,jr,kr->ijk", (13, 29, 17), (3,))
    p.shard_host(0, 2)
    with pytest.raises(nef.NefError):
        p.shard_host(1, 2)   # already sharded
    with pytest.raises(nef.NefError):
        nef.Plan("ir,jr,kr->ijk", (3, 2, 2), (3,)).shard_host(0, 4)   # largest mode smaller than world
