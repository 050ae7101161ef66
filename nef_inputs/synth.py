"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no a/b/g, no update, no loss).  It
only draws planted data with the value laws BASELINE.json states (DESIGN.md
§Inputs):  true factors from Gamma laws, a planted
mean Yhat_true = einsum(model_str, true factors) (numpy / torch library einsum used
as a data-synthesis primitive), a noise law, a Bernoulli missing-data mask
(nonzero = observed, reading R6) and U(0.1, 1) fp32 initial factors (reading R11).

The paper's datasets (ICEWS P:272, Uber P:274, WITS P:276) are not available; these
draws stand in for them at the configs' shapes.

Two generators:
  * ``generate_numpy``  -- CPU, numpy ``SeedSequence(k-1)`` spawned into
    [true factors, noise, mask, init] (reading R21); used for every size the oracle
    runs on.
  * ``generate_torch``  -- on a CUDA device with torch's Philox generator, for the
    full-size configs (up to 4.3 G entries) that cannot be drawn on the host in
    reasonable time.  Same laws, different stream; the oracle only ever sees slices
    of these tensors copied back to the host.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    model: str
    shape: tuple
    ranks: tuple
    alpha: float          # paper convention
    beta: float           # paper convention: beta_json - 1
    beta_json: float      # the literal BASELINE.json number
    p_missing: float      # P(mask == 0)
    iters: int
    law: str
    small_shape: tuple    # shape the oracle finishes in seconds (several tiles + ragged tail)
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def n_entries(self) -> int:
        return int(math.prod(self.shape))


CONFIGS = {
    "c1": Config("c1", "ir,jr,kr->ijk", (50, 40, 30), (5,), 1.0, 0.0, 1.0, 0.0, 100,
                 "poisson_gamma11", (50, 40, 30)),
    "c2": Config("c2", "ia,jb,kc,abc->ijk", (256, 256, 256), (16, 16, 16), 1.0, 1.0, 2.0, 0.10, 50,
                 "tucker_absnormal", (70, 45, 52)),
    "c3": Config("c3", "ir,jr,kr->ijk", (1024, 1024, 384), (32,), 1.0, 0.0, 1.0, 0.20, 20,
                 "poisson_gamma05_scaled", (150, 133, 70), extra={"scale": 0.10}),
    "c4": Config("c4", "ik,jk,tl,dl,kl->ijtd", (260, 260, 24, 365), (20, 10), 0.5, 0.0, 1.0, 0.0, 20,
                 "negbin_r2", (30, 27, 24, 37)),
    "c5": Config("c5", "ir,jr,kr->ijk", (2048, 2048, 1024), (64,), 1.0, -0.5, 0.5, 0.05, 10,
                 "gamma_noise", (140, 96, 67)),
}

CONFIG_INDEX = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}


def _parse(model):
    lhs, out = model.replace(" ", "").split("->")
    return lhs.split(","), out


def factor_shapes(model, shape, ranks):
    ops, out = _parse(model)
    dims = dict(zip(out, shape))
    con = []
    for op in ops:
        for c in op:
            if c not in dims and c not in con:
                con.append(c)
    dims.update(zip(con, ranks))
    return [tuple(dims[c] for c in op) for op in ops]


def _true_law(cfg):
    return (0.5, 1.0) if cfg.law == "poisson_gamma05_scaled" else (1.0, 1.0)


def generate_numpy(name, shape=None, seed_offset=0, want_truth=False):
    """Draw config ``name`` at ``shape`` (default: its small shape) on the host.

    Returns dict(Y=float32 array, mask=uint8 array or None, init=list[float32],
    alpha, beta, beta_json, model, ranks, iters)."""
    cfg = CONFIGS[name]
    shape = tuple(shape or cfg.small_shape)
    ss = np.random.SeedSequence(CONFIG_INDEX[name] - 1 + 1000 * seed_offset)
    s_true, s_noise, s_mask, s_init = [np.random.default_rng(s) for s in ss.spawn(4)]
    fshapes = factor_shapes(cfg.model, shape, cfg.ranks)
    k, th = _true_law(cfg)
    truth = [s_true.gamma(k, th, size=fs) for fs in fshapes]
    yhat = np.einsum(cfg.model, *truth, optimize="greedy")
    Y = _apply_noise(cfg, yhat, s_noise)
    mask = None
    if cfg.p_missing > 0:
        mask = (s_mask.random(shape) >= cfg.p_missing).astype(np.uint8)
    init = [s_init.uniform(0.1, 1.0, size=fs).astype(np.float32) for fs in fshapes]
    out = dict(Y=Y.astype(np.float32), mask=mask, init=init, alpha=cfg.alpha, beta=cfg.beta,
               beta_json=cfg.beta_json, model=cfg.model, ranks=cfg.ranks, iters=cfg.iters,
               shape=shape)
    if want_truth:
        out["truth"] = truth
    return out


def _apply_noise(cfg, yhat, rng):
    if cfg.law == "poisson_gamma11":
        return rng.poisson(yhat).astype(np.float64)
    if cfg.law == "tucker_absnormal":
        return yhat + np.abs(rng.normal(0.0, 0.1, size=yhat.shape))
    if cfg.law == "poisson_gamma05_scaled":
        return rng.poisson(cfg.extra["scale"] * yhat).astype(np.float64)
    if cfg.law == "negbin_r2":
        r = 2.0
        lam = rng.gamma(r, yhat / r)
        return rng.poisson(lam).astype(np.float64)
    if cfg.law == "gamma_noise":
        return yhat * rng.gamma(10.0, 0.1, size=yhat.shape)
    raise ValueError(cfg.law)


# ------------------------------------------------------------------------------------
# device-side generator for the full-size configs
# ------------------------------------------------------------------------------------
SLAB = 8   # mode-0 rows per independently seeded draw (shard-friendly, reading R21)


def generate_torch(name, device, shape=None, seed_offset=0, mode0_range=None):
    """Draw config ``name`` (default: FULL shape) directly into device memory.

    The planted mean is formed slab-wise along mode 0 with torch.einsum; noise and mask of
    each SLAB-row slab come from their own seeded generator, so the tensor is identical no
    matter how it is split.  ``mode0_range=(b, e)`` returns only rows [b, e) of mode 0 (a
    rank's shard), with the mode-0 factors of ``init`` / ``truth`` sliced accordingly.

    Returns dict(Y=float32 tensor, mask=uint8 tensor or None, init=list[float32 tensor], ...).
    """
    import torch

    cfg = CONFIGS[name]
    shape = tuple(shape or cfg.shape)
    b0, e0 = mode0_range or (0, shape[0])
    base = 7919 * CONFIG_INDEX[name] + 104729 * seed_offset
    g_true = torch.Generator(device=device).manual_seed(base + 1)
    g_init = torch.Generator(device=device).manual_seed(base + 4)
    fshapes = factor_shapes(cfg.model, shape, cfg.ranks)
    k, th = _true_law(cfg)
    truth = []
    for fs in fshapes:
        conc = torch.full(fs, k, dtype=torch.float32, device=device)
        truth.append(torch._standard_gamma(conc, generator=g_true) * th)
    ops, out = _parse(cfg.model)
    lead = out[0]
    for op in ops:
        if lead in op and op[0] != lead:
            raise ValueError("lead index must be first in its operand for slab generation")
    lshape = (e0 - b0,) + shape[1:]
    Y = torch.empty(lshape, dtype=torch.float32, device=device)
    mask = torch.empty(lshape, dtype=torch.uint8, device=device) if cfg.p_missing > 0 else None
    for s0 in range((b0 // SLAB) * SLAB, e0, SLAB):
        s1 = min(shape[0], s0 + SLAB)
        lo, hi = max(s0, b0), min(s1, e0)
        sl = [t[s0:s1] if op[0] == lead else t for t, op in zip(truth, ops)]
        yhat = torch.einsum(cfg.model, *sl)
        g = torch.Generator(device=device).manual_seed(base * 1000003 + 2 * s0 + 11)
        ys = _apply_noise_torch(cfg, yhat, g)
        Y[lo - b0:hi - b0] = ys[lo - s0:hi - s0]
        if mask is not None:
            ms = torch.rand(yhat.shape, generator=g, device=device) >= cfg.p_missing
            mask[lo - b0:hi - b0] = ms[lo - s0:hi - s0].to(torch.uint8)
        del yhat, ys
    init = [torch.rand(fs, generator=g_init, device=device) * 0.9 + 0.1 for fs in fshapes]
    if mode0_range is not None:
        init = [f[b0:e0].contiguous() if op[0] == lead else f for f, op in zip(init, ops)]
        truth = [t[b0:e0].contiguous() if op[0] == lead else t for t, op in zip(truth, ops)]
    return dict(Y=Y, mask=mask, init=init, truth=truth, alpha=cfg.alpha, beta=cfg.beta, beta_json=cfg.beta_json,
                model=cfg.model, ranks=cfg.ranks, iters=cfg.iters, shape=shape, local_shape=lshape)


def _apply_noise_torch(cfg, yhat, g):
    import torch

    if cfg.law == "poisson_gamma11":
        return torch.poisson(yhat, generator=g)
    if cfg.law == "tucker_absnormal":
        return yhat + torch.randn(yhat.shape, generator=g, device=yhat.device).abs_() * 0.1
    if cfg.law == "poisson_gamma05_scaled":
        return torch.poisson(yhat * cfg.extra["scale"], generator=g)
    if cfg.law == "negbin_r2":
        r = 2.0
        lam = torch._standard_gamma(torch.full_like(yhat, r), generator=g) * (yhat / r)
        return torch.poisson(lam, generator=g)
    if cfg.law == "gamma_noise":
        noise = torch._standard_gamma(torch.full_like(yhat, 10.0), generator=g) * 0.1
        return yhat * noise
    raise ValueError(cfg.law)


# ------------------------------------------------------------------------------------
# train / validation / heldout labels: each entry heldout w.p. p_heldout, else
# validation w.p. p_validation, else train; uint8 codes 0 = excluded (missing data), 1 = train,
# 2 = validation, 3 = heldout.  A draw only: no arithmetic of the method.
# ------------------------------------------------------------------------------------
LABEL_EXCLUDED, LABEL_TRAIN, LABEL_VAL, LABEL_HELDOUT = 0, 1, 2, 3


def split_labels(shape, p_heldout=0.1, p_validation=0.05, seed=0, missing=None):
    if not (0 <= p_heldout < 1 and 0 <= p_validation < 1):
        raise ValueError("degenerate split probabilities")
    u = np.random.default_rng(seed).random(tuple(shape))
    lab = np.full(tuple(shape), LABEL_TRAIN, dtype=np.uint8)
    lab[u < p_heldout + (1.0 - p_heldout) * p_validation] = LABEL_VAL
    lab[u < p_heldout] = LABEL_HELDOUT
    if missing is not None:
        lab[np.asarray(missing, dtype=bool)] = LABEL_EXCLUDED
    return lab
