"""Diagnostic: compare tcgen05 numerator / denominator with the oracle and the FFMA path."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import nef_oracle as O  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402
from tests.test_gpu_tc import TC_CASES, _data, _dev  # noqa: E402

np.set_printoptions(precision=4, suppress=True, linewidth=160)
for ci in [int(x) for x in sys.argv[1:]] or [0]:
    ms, shape, ranks, (al, be), pm, law = TC_CASES[ci]
    Y, M, init = _data(ms, shape, ranks, pm, law)
    plan = nef.Plan(ms, shape, ranks)
    Yd, Md, F = _dev(Y, M, init)
    print("case", ci, ms, shape, ranks)
    for ell in range(len(F)):
        A, B = O.numerator_denominator(ms, Y, M, init, ell, al, be)
        nef.nef_set_kernel_policy(0)
        n0, d0 = plan.num_den(ell, Yd, Md, al, be, F)
        nef.nef_set_kernel_policy(1)
        n1, d1 = plan.num_den(ell, Yd, Md, al, be, F)
        nef.nef_set_kernel_policy(0)
        n0 = n0.cpu().numpy().reshape(A.shape[0], -1)
        d0 = d0.cpu().numpy().reshape(A.shape[0], -1)
        n1 = n1.cpu().numpy().reshape(A.shape[0], -1)
        A2 = A.reshape(A.shape[0], -1)
        B2 = B.reshape(B.shape[0], -1)
        print(" ell", ell, "ffma num err %.2e" % np.max(np.abs(n1 - A2) / np.abs(A2)),
              "tc num err %.2e den err %.2e" % (np.max(np.abs(n0 - A2) / np.abs(A2)), np.max(np.abs(d0 - B2) / np.abs(B2))))
        r = n0 / A2
        print("   num ratio rows 0,1,127,128,-1 cols 0..7:\n", r[[0, 1, 127, min(128, r.shape[0] - 1), -1], :8])
        rd = d0 / B2
        print("   den ratio rows 0,1 cols 0..7:\n", rd[[0, 1], :8])
        # does tc num equal oracle num with a bond permutation / mixing?  least squares n0 ~ A2 @ X
        X, *_ = np.linalg.lstsq(A2, n0, rcond=None)
        print("   lstsq mixing diag[:8]", np.diag(X)[:8], "offdiag max %.3f" % np.max(np.abs(X - np.diag(np.diag(X)))))
