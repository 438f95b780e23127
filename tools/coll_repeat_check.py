"""Repeated NNN all-reduces (paro_collective(0)), eager and graph-replayed,
with and without host synchronisation between calls (back-to-back launches
race the device-resident barrier generations if anything is wrong); every
result is compared with the first eager call's.  argv: bucket multiplier,
topology."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from graph_worker import _copy  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_06003_b200 import paro
    M = world // 2 if world >= 4 else 1
    uid = paro.unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    dist.broadcast(t, 0)
    ctx = paro.Context(world, M, mode="real", rank=rank, device=rank, uid=bytes(t.tolist()))
    B = world * 64 * int(sys.argv[1] if len(sys.argv) > 1 else 32)
    s = torch.cuda.Stream()
    topo = sys.argv[2] if len(sys.argv) > 2 else "oneshot"
    pl = paro.Plan(ctx, "NNN", [3 * B], bucket_elems=B, topology=topo, fuse_allreduce=False, stream=s.cuda_stream)
    pl.synth_grads(rank, 1234, 1)
    ghat = pl.buffer(rank, 3)

    def grab():
        torch.cuda.synchronize()
        buf = torch.empty(3 * B, dtype=torch.int16, device="cuda")
        _copy(buf, ghat)
        return buf.cpu().numpy().view(np.uint16).copy()

    with torch.cuda.stream(s):
        pl.collective(0)
    ref = grab()
    out = []

    def check(tag):
        got = grab()
        bad = np.nonzero(got != ref)[0]
        out.append({"rank": rank, "tag": tag, "bad": int(bad.size), "first": bad[:8].tolist(),
                    "got": got[bad[:4]].tolist(), "want": ref[bad[:4]].tolist()})

    for k in range(4):
        with torch.cuda.stream(s):
            pl.collective(0)
        check(f"eager{k}")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            pl.collective(0)
    torch.cuda.synchronize()
    for k in range(4):
        g.replay()
        check(f"replay{k}")
        with torch.cuda.stream(s):
            pl.collective(0)
        check(f"eager_after_replay{k}")
    for k in range(4):                 # no host sync between the replay and the eager call
        g.replay()
        with torch.cuda.stream(s):
            pl.collective(0)
        check(f"replay_then_eager_nosync{k}")
    for k in range(4):
        with torch.cuda.stream(s):
            pl.collective(0)
            pl.collective(0)
        check(f"eager_eager_nosync{k}")
    for k in range(4):
        g.replay()
        g.replay()
        check(f"replay_replay_nosync{k}")
    nbad = sum(o["bad"] > 0 for o in out)
    for o in out:
        if o["bad"]:
            print(json.dumps(o), flush=True)
    print(json.dumps({"rank": rank, "topology": topo, "checks": len(out), "failed": nbad}), flush=True)
    pl.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
