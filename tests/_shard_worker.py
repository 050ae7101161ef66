"""Worker of tests/test_gpu_sharded.py::test_torchrun_two_ranks_nccl (one rank per GPU)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from nef_inputs import generate_numpy  # noqa: E402
from oracle import nef_oracle as O  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl")
    d = generate_numpy("c5", shape=(144, 96, 80))
    ms, al, be = d["model"], d["alpha"], d["beta"]
    ops, out = O.parse(ms)
    plan = nef.Plan(ms, d["shape"], d["ranks"])
    uid = [nef.nef_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    plan.shard(rank, world, uid[0])
    i = plan.info
    sm, b, n = i["shard_mode"], i["local_begin"], i["local_len"]
    letter = out[sm]
    Y = torch.from_numpy(np.take(d["Y"], np.arange(b, b + n), axis=sm)).cuda()
    M = torch.from_numpy(np.take(d["mask"], np.arange(b, b + n), axis=sm)).cuda()
    F = [torch.from_numpy(np.take(f, np.arange(b, b + n), axis=op.index(letter)) if letter in op else f.copy()).cuda()
         for f, op in zip(d["init"], ops)]
    tr = plan.fit(Y, M, al, be, F, 2)
    ref, rtr = O.fit(ms, d["Y"], d["mask"], d["init"], al, be, 2)
    err_t = float(np.max(np.abs(np.asarray(tr) - rtr) / np.abs(rtr)))
    errs = []
    for f, r, op in zip(F, ref, ops):
        if letter in op:
            r = np.take(r, np.arange(b, b + n), axis=op.index(letter))
        errs.append(float(np.max(np.abs(f.cpu().numpy() - r) / np.abs(r))))
    ok = err_t < 1e-3 and max(errs) < 2e-4
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("rank errors", errs, err_t)
        if flag.item() == 1:
            print("SHARD_OK")
    dist.destroy_process_group()
    return 0 if flag.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
