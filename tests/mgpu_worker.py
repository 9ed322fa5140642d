"""One rank of the real-NCCL multi-GPU parity test (tests/test_multigpu.py),
launched as `python -m torch.distributed.run --nproc-per-node G
tests/mgpu_worker.py OUT.json CONFIG...` -- one process per GPU.

Each rank builds its Morton-range shard plan of every listed BASELINE config
(SURVEY.md §8e), attaches the in-plan NCCL communicator (the 128-byte id
travels over torch.distributed), evaluates through the device path and
through the host-buffer C-ABI path, and rank 0 writes the job totals."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2212_08284_b200 as ankh  # noqa: E402
from paper_2212_08284_b200 import inputs  # noqa: E402


def main():
    out_path, configs = sys.argv[1], [int(c) for c in sys.argv[2:]]
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    results = {}
    for c in configs:
        pos, src, rb, cfg = inputs.make_config(c)
        L = cfg.orders[0] if c != 2 else 5
        ec = ankh.EwaldConfig(order_cheb=L, order_equi=L)
        plan = ankh.Plan(pos.shape[0], rb, ec, device=local, rank=rank, world=world, phase_timing=False)
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(ankh.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        plan.attach_nccl(bytes(uid.cpu().numpy().tobytes()))
        dp, ds = torch.from_numpy(pos).cuda(), torch.from_numpy(src).cuda()
        reps = [plan.energy_device(dp, ds) for _ in range(3)]  # plain, graph capture, replay
        host = plan.energy(pos, src)
        key = lambda r: [r.e_total, r.e_self, r.e_near, r.e_far, r.e_periodic_far]
        results[str(c)] = {"device": [key(r) for r in reps], "host": key(host),
                           "pairs_rank": int(reps[-1].near_pairs)}
        # total near pairs over the ranks (each rank reports its own)
        t = torch.tensor([float(reps[-1].near_pairs)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        results[str(c)]["pairs_total"] = int(t.item())
        plan.close()
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump({"world": world, "results": results}, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
