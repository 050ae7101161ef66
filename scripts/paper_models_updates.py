import sys, json, torch
sys.path.insert(0, '.')
from oracle import nef_oracle as O
from paper_2602_02759_b200 import nef
dev = torch.device('cuda')
for name, ms, shape, ranks in [("icews", "ir,jr,ak,kr,tr->ijat", (249, 249, 20, 228), (25, 10)), ("wits", "er,ir,gr,tk,kr->eigt", (196, 196, 96, 29), (25, 10))]:
    g = torch.Generator(device=dev).manual_seed(1)
    fs = O.factor_shapes(ms, shape, ranks)
    truth = [torch._standard_gamma(torch.full(s, 1.0, device=dev), generator=g) * 0.5 for s in fs]
    Y = torch.poisson(torch.einsum(ms, *truth), generator=g).float()
    M = (torch.rand(shape, generator=g, device=dev) >= 0.1).to(torch.uint8)
    F = [torch.rand(s, generator=g, device=dev) * 0.9 + 0.1 for s in fs]
    plan = nef.Plan(ms, shape, ranks)
    for ell in range(len(fs)):
        plan.update(ell, Y, M, 1.0, 0.0, F); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nef.nef_profile_enable(True)
        e0.record()
        for _ in range(3): plan.update(ell, Y, M, 1.0, 0.0, F)
        e1.record(); torch.cuda.synchronize()
        kms, kl, kb = nef.nef_profile_read(); nef.nef_profile_enable(False)
        print(name, ell, "ms/update %.3f" % (e0.elapsed_time(e1) / 3), "fused ms %.3f" % (kms / max(kl, 1)), "launches/update", nef.nef_last_launch_count())
