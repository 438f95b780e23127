"""Worker for the real-rank collective test (torchrun, one process per GPU):
paro_collective(0) of NNN plans (fuse_allreduce = 0) on every world topology,
two calls each, at a bucket large enough that the one-shot all-reduce runs as
reduce-scatter + all-gather (two rounds).  Saves each rank's g_hat slots; the
parent compares them with the oracle."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paro_synth import SEED  # noqa: E402
from graph_worker import _copy  # noqa: E402


def main():
    out = sys.argv[1]
    cfg = json.loads(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_06003_b200 import paro
    M, B, n = cfg["M"], cfg["bucket"], cfg["n"]
    uid = paro.unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    dist.broadcast(t, 0)
    ctx = paro.Context(world, M, mode="real", rank=rank, device=local, uid=bytes(t.tolist()))
    for topo in cfg["topos"]:
        pl = paro.Plan(ctx, "NNN", [n], bucket_elems=B, topology=topo, fuse_allreduce=False,
                       transport="pull", comm_impl=cfg.get("comm_impl", "tma_store"))
        pl.synth_grads(rank, SEED, 1)
        for _ in range(2):
            pl.collective(0)
        torch.cuda.synchronize()
        nb = pl.info()["n_buckets"]
        buf = torch.empty(min(nb, 3) * B, dtype=torch.int16, device="cuda")
        _copy(buf, pl.buffer(rank, 3))
        np.save(os.path.join(out, f"{topo}_r{rank}.npy"), buf.cpu().numpy().view(np.uint16))
        pl.close()
        dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
