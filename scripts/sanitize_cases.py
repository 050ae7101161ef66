"""Small fits for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): c1 on the
CUDA-core kernel, an odd-prime tile-tail shape, and tcgen05 cases over the three TMA layouts with
and without the sentinel copy, the split fit and an App. B loss.  Usage:
    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from nef_inputs import generate_numpy, split_labels  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402


def run(ms, shape, ranks, ab, pm, iters=1, seed=0):
    rng = np.random.default_rng(seed)
    from oracle import nef_oracle as O
    fs = O.factor_shapes(ms, shape, ranks)
    Y = rng.poisson(O.contract(ms, [rng.gamma(1, 1, s) for s in fs])).astype(np.float32) + 0.25
    M = torch.from_numpy((rng.random(shape) >= pm).astype(np.uint8)).cuda() if pm > 0 else None
    F = [torch.from_numpy(rng.uniform(0.1, 1, s).astype(np.float32)).cuda() for s in fs]
    p = nef.Plan(ms, shape, ranks)
    tr = p.fit(torch.from_numpy(Y).cuda(), M, ab[0], ab[1], F, iters)
    torch.cuda.synchronize()
    print(ms, shape, "tc", [L["tc"] for L in p.describe()["lowerings"]], "trace", tr[-1])


def main():
    d = generate_numpy("c1")
    p = nef.Plan(d["model"], d["shape"], d["ranks"])
    F = [torch.from_numpy(f).cuda() for f in d["init"]]
    print("c1", p.fit(torch.from_numpy(d["Y"]).cuda(), None, d["alpha"], d["beta"], F, 2)[-1])
    run("ir,jr,kr->ijk", (13, 17, 19), (3,), (1.0, 0.0), 0.1)                # odd primes, CUDA-core
    run("ir,jr,kr->ijk", (130, 96, 68), (40,), (1.0, -0.5), 0.05)            # tcgen05, tails, sentinel
    run("ir,jr,kr->ijk", (96, 104, 44), (32,), (1.0, 0.0), 0.0)              # layout-1 half box OOB
    run("ia,jb,kc,abc->ijk", (64, 72, 40), (8, 8, 8), (1.0, 1.0), 0.1)      # layout 2, SPA split
    run("ik,jk,tl,dl,kl->ijtd", (32, 48, 24, 40), (20, 10), (0.5, 0.0), 0.0)
    # split fit and an App. B loss on the tcgen05 kernel
    shape = (96, 80, 64)
    rng = np.random.default_rng(3)
    Y = torch.from_numpy(rng.poisson(2.0, shape).astype(np.float32)).cuda()
    lab = torch.from_numpy(split_labels(shape, 0.1, 0.05, seed=4)).cuda()
    p = nef.Plan("ir,jr,kr->ijk", shape, (16,))
    F = [torch.from_numpy(rng.uniform(0.1, 1, (n, 16)).astype(np.float32)).cuda() for n in shape]
    print("split", p.fit_split(Y, lab, nef.loss_spec("ab", 1.0, 0.0), F, max_iters=2)["reason"])
    print("negbin", p.fit_ex(Y, None, nef.loss_spec("negbin", param=2.0), F, 1)[-1])
    torch.cuda.synchronize()
    print("SANITIZE_CASES_DONE")


if __name__ == "__main__":
    main()
