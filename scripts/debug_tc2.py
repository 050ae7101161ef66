"""Bisect the numerator MMA: print tc num/oracle for several NEF_TC_* variants (run in subprocesses)."""
import os
import subprocess
import sys

code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import nef_oracle as O
from paper_2602_02759_b200 import nef
from tests.test_gpu_tc import TC_CASES, _data, _dev
ms, shape, ranks, (al, be), pm, law = TC_CASES[int(sys.argv[1])]
Y, M, init = _data(ms, shape, ranks, pm, law)
plan = nef.Plan(ms, shape, ranks)
Yd, Md, F = _dev(Y, M, init)
A, B = O.numerator_denominator(ms, Y, M, init, 0, al, be)
n0, d0 = plan.num_den(0, Yd, Md, al, be, F)
n0 = n0.cpu().numpy()
r = n0 / A
print("ratio[0,:6]", np.round(r[0, :6], 4), "median %.4f  max relerr %.3e" % (np.median(r), np.max(np.abs(r - 1))))
'''
for case in sys.argv[1:] or ["0"]:
    for vt, dbg in [(0, 0), (0, 1), (0, 2), (0, 4), (1, 0), (1, 1)]:
        env = dict(os.environ, NEF_TC_VT=str(vt), NEF_TC_DBG=str(dbg))
        out = subprocess.run([sys.executable, "-c", code, case], env=env, capture_output=True, text=True, timeout=120)
        print("case", case, "vt", vt, "dbg", dbg, "->", (out.stdout.strip() or out.stderr.strip()[-300:]))
