#!/usr/bin/env python
"""Benchmark of the B200-native MU sweep (BASELINE.json metric: tensor entries/s per full MU
sweep, and fraction of the HBM roofline of the streaming kernel).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

A step is one full Gauss-Seidel sweep (every factor update of Algorithm 1, with
the loss of the entering iterate fused into the first factor's pass).  The K timed steps
are ONE nef_fit(iters=K) call (which also runs its single final loss pass), bracketed by
barrier + synchronize, timed with CUDA events on the launch stream, max over ranks.
Inputs are generated on the device (seeded, nef_inputs) and are larger than L2.
N > 1: launched by torchrun; Y is sharded along its largest mode and the small
numerator/denominator partials are all-reduced with NCCL inside libnef.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tensor entries/s per full MU sweep at 1/2/4/8 B200; % of HBM/compute roofline"
UNIT = "entries/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _workload(cfg):
    mask = "%.0f%% missing (uint8)" % (100 * cfg.p_missing) if cfg.p_missing > 0 else "none"
    return {"workload": "%s %s %s R=%s (alpha,beta)=(%g,%g) mask %s" % (cfg.name, cfg.model, "x".join(map(str, cfg.shape)),
                                                                        ",".join(map(str, cfg.ranks)), cfg.alpha, cfg.beta, mask),
            "einsum": cfg.model, "shape": list(cfg.shape), "ranks": list(cfg.ranks),
            "alpha_beta_paper": [cfg.alpha, cfg.beta], "beta_json": cfg.beta_json, "mask_missing": cfg.p_missing,
            "entries": cfg.n_entries}


# ------------------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw,power.limit"
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, pw, lim, reasons = [], [], [], [], set()
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
            try:
                pw.append(float(parts[6]))
                lim.append(float(parts[7]))
            except (ValueError, IndexError):
                pass
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None, "power_limit_w": max(lim) if lim else None}


# ------------------------------------------------------------------------------ oracle timing
def oracle_sample(name, target_s=12.0):
    """Time the float64 oracle (as it stands) for one full sweep + one loss evaluation on a
    bounded sample of the workload: the first s rows of mode 0 drawn with the same laws."""
    import numpy as np
    from nef_inputs import CONFIGS, generate_numpy
    from oracle import nef_oracle as O

    cfg = CONFIGS[name]
    row = math.prod(cfg.shape[1:])

    def run(s, reps=1):
        d = generate_numpy(name, shape=(s,) + tuple(cfg.shape[1:]))
        th = [f.astype(np.float64) for f in d["init"]]
        c0, t0 = os.times(), time.perf_counter()
        for _ in range(reps):
            for ell in range(len(th)):
                th[ell] = O.update_factor(d["model"], d["Y"], d["mask"], th, ell, d["alpha"], d["beta"])
            O.loss(d["model"], d["Y"], d["mask"], th, d["alpha"], d["beta"])
        t, c1 = time.perf_counter() - t0, os.times()
        return t / reps, (c1.user - c0.user) + (c1.system - c0.system), t

    s = 1 if row > 200000 else max(1, min(cfg.shape[0], 200000 // row))
    t, cpu, t_total = run(s)
    # grow the sample to ~target_s: more mode-0 rows, then (whole tensor) repeated sweeps
    s2 = int(max(1, min(cfg.shape[0], s * target_s / max(t, 1e-3))))
    reps = max(1, int(target_s / max(t * s2 / s, 1e-3))) if s2 == cfg.shape[0] else 1
    if s2 > s or reps > 1:
        s = s2
        t, cpu, t_total = run(s, reps)
    # threads actually used: process CPU time over wall time of the timed run (numpy's elementwise
    # work is single-threaded; its einsum contractions may use the BLAS pool)
    n = s * row
    return {"value": n / t, "unit": UNIT, "cores": round(cpu / max(t_total, 1e-9), 2), "kind": "oracle",
            "cores_available": len(os.sched_getaffinity(0)),
            "sample": "%s first %d of %d mode-0 rows (%d entries, %s), %d x (1 sweep + 1 loss), %.2f s" % (
                name, s, cfg.shape[0], n, "x".join(map(str, (s,) + tuple(cfg.shape[1:]))), reps, t_total),
            "seconds": t, "entries": n}, s


def host_info():
    info = {"cores_available": len(os.sched_getaffinity(0))}
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                info["ram_gb"] = round(int(line.split()[1]) / 1048576, 1)
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return info


PRECISION = ("f32 data and factors; tcgen05 kind::tf32 MMAs (reconstruction with the updated factor's side "
             "split hi + lo - for bonds 33-64 the small lo term as kind::f16 BF16 MMAs on BF16 copies of U_lo "
             "and V - numerator / denominator operands TF32 round-to-nearest, Euclidean bond <= 32: "
             "numerator operand split hi + lo); fp32 tensor-core accumulation drained every 256 tiles; fp64 "
             "split-partial, loss and update arithmetic")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    from nef_inputs import CONFIGS, generate_numpy
    from oracle import nef_oracle as O

    cfg = CONFIGS[args.config]
    base, s = oracle_sample(args.config, target_s=4.0)
    d = generate_numpy(args.config, shape=(s,) + tuple(cfg.shape[1:]))
    th = [f.astype(np.float64) for f in d["init"]]

    def step():
        for ell in range(len(th)):
            th[ell] = O.update_factor(d["model"], d["Y"], d["mask"], th, ell, d["alpha"], d["beta"])
        O.loss(d["model"], d["Y"], d["mask"], th, d["alpha"], d["beta"])

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    t = (time.perf_counter() - t0) / max(1, args.steps)
    n = s * math.prod(cfg.shape[1:])
    v = n / t
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": dict(_workload(cfg), sample_rows=s), "host": host_info(),
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": base["cores"], "kind": "oracle",
                            "sample": base["sample"].split(", 1 sweep")[0] + ", each step 1 sweep + 1 loss"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)   # c5's 10 iterations (BASELINE.json)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel-policy", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from nef_inputs import CONFIGS, generate_torch
    from paper_2602_02759_b200 import nef

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    nef.nef_set_kernel_policy(args.kernel_policy)
    plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
    if world > 1:
        uid = [nef.nef_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        plan.shard(rank, world, uid[0])
    info = plan.info
    sm = info["shard_mode"]
    if sm <= 0:
        rng = (info["local_begin"], info["local_begin"] + info["local_len"]) if sm == 0 else None
        data = generate_torch(args.config, dev, mode0_range=rng)
    else:
        data = generate_torch(args.config, dev)
        b, n = info["local_begin"], info["local_len"]
        data["Y"] = data["Y"].narrow(sm, b, n).contiguous()
        if data["mask"] is not None:
            data["mask"] = data["mask"].narrow(sm, b, n).contiguous()
        letter = cfg.model.split("->")[1][sm]
        ops = cfg.model.split("->")[0].split(",")
        data["init"] = [f.narrow(op.index(letter), b, n).contiguous() if letter in op else f
                        for f, op in zip(data["init"], ops)]
    Y, M, F = data["Y"], data["mask"], data["init"]
    assert tuple(Y.shape) == plan.local_shape
    alpha, beta = cfg.alpha, cfg.beta
    ws = plan.workspace(dev)
    torch.cuda.synchronize()

    # warm-up sweeps (untimed)
    plan.fit(Y, M, alpha, beta, F, args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    nef.nef_profile_enable(True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(stream)
    trace = plan.fit(Y, M, alpha, beta, F, args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1)
    kern_ms, kern_launches, algo_bytes = nef.nef_profile_read()
    nef.nef_profile_enable(False)
    launches = nef.nef_last_launch_count()
    t_max = t_ms
    if world > 1:
        tt = torch.tensor([t_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    value = cfg.n_entries * args.steps / (t_max / 1e3)

    peak, peak_src = _peaks()
    achieved = (algo_bytes / max(kern_launches, 1)) / (kern_ms / max(kern_launches, 1) / 1e3) / 1e9 if kern_ms else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.config)
            traffic = tr.get("dram_bytes_per_launch") if tr else None
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "kernel": "fused streaming pass (all factor updates + loss pass)",
                "kernel_share_of_step": kern_ms / t_ms if t_ms else None,
                "algorithmic_bytes_per_launch": algo_bytes / max(kern_launches, 1),
                "launches": kern_launches, "peak_source": peak_src}

    # end to end through the host-buffer C entry point
    e2e = None
    if not args.no_e2e:
        try:
            e2e = _e2e(nef, plan, cfg, data, args, dev, world)
        except Exception as ex:  # report, never hide
            e2e = {"value": None, "unit": UNIT, "error": repr(ex)[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, _ = oracle_sample(args.config)

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f32/tf32/bf16", "precision": PRECISION,
               "data": "synthetic", "host": host_info(),
               "config": dict(_workload(cfg), parallelism=("shard mode %d over %d ranks, NCCL all-reduce of partials"
                                                           % (sm, world)) if world > 1 else "single GPU",
                              l2="inputs (%.1f GB) larger than L2 (126 MB); no flush needed" % (
                                  (Y.numel() * 4 + (M.numel() if M is not None else 0)) * world / 1e9)),
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
               "clocks": clk, "loss_trace_last": float(trace[-1]),
               "entry_visits_per_s": value * len(F)}
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


def _e2e(nef, plan, cfg, data, args, dev, world):
    """Same metric through nef_fit_host: every step copies Y (+mask, factors) from pinned host
    memory and reads the factors + trace back; timed with CUDA events on the stream."""
    import torch
    import torch.distributed as dist

    Y, M, F = data["Y"], data["mask"], data["init"]
    Yh = torch.empty(Y.shape, dtype=Y.dtype, pin_memory=True)
    Yh.copy_(Y)
    Mh = None
    if M is not None:
        Mh = torch.empty(M.shape, dtype=M.dtype, pin_memory=True)
        Mh.copy_(M)
    Fh = [torch.empty(f.shape, dtype=f.dtype, pin_memory=True).copy_(f) for f in F]
    need = nef.nef_host_scratch_bytes(plan.h, M is not None)
    del data
    scratch = torch.empty(need, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    nef.nef_fit_host(plan.h, Yh, Mh, cfg.alpha, cfg.beta, 1e-12, Fh, 1, scratch)   # warm
    torch.cuda.synchronize()
    steps = max(1, args.e2e_steps)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for _ in range(steps):
        nef.nef_fit_host(plan.h, Yh, Mh, cfg.alpha, cfg.beta, 1e-12, Fh, 1, scratch)
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([t], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    h2d = Yh.numel() * 4 + (Mh.numel() if Mh is not None else 0) + sum(f.numel() * 4 for f in Fh)
    d2h = sum(f.numel() * 4 for f in Fh) + 2 * 8
    del scratch
    return {"value": cfg.n_entries * steps / (t / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h * world, "steps": steps,
            "note": "each step = nef_fit_host(iters=1): H2D of Y/mask/factors from pinned memory, 1 sweep + final "
                    "loss pass, D2H of factors and trace"}


if __name__ == "__main__":
    sys.exit(main())
