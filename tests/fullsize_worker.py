"""Worker of the full-size sampled parity test (tests/test_gpu_fullsize.py).

Runs bench.py's timed launch configuration (same model list, strategy, group
split, bucket, transport, kernels: `bench.parse` + `bench.plan_kwargs`) for
`steps` real paro_steps on the bench's resident synthetic gradients, then
saves sampled windows of every state the rank holds, with the flat element
ranges the library reports for them (paro_shard_range).  The parent checks
the windows against the oracle element by element.

N = 1: `python tests/fullsize_worker.py OUT CFG`; N > 1 under torchrun.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from devmem import d2h  # noqa: E402
from paro_synth import SEED, llama_param_sizes  # noqa: E402


def windows_of(lo, hi, w):
    """Start, middle and end windows of [lo, hi) (clipped, merged when short)."""
    if hi - lo <= 3 * w:
        return [(lo, hi)]
    mid = lo + ((hi - lo) // 2 // 64) * 64
    return [(lo, lo + w), (mid - w // 2, mid + w // 2), (hi - w, hi)]


def main():
    out = sys.argv[1]
    cfg = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_06003_b200 import paro
    args = bench.parse(cfg.get("bench_args", []) + ["--gpus", str(world)])
    M = args.group_size or bench.default_group(world)
    uid = paro.unique_id() if rank == 0 else bytes(128)
    if world > 1:
        t = torch.tensor(list(uid), dtype=torch.uint8)
        dist.broadcast(t, 0)
        uid = bytes(t.tolist())
    ctx = paro.Context(world, M, mode="real", rank=rank, device=local, uid=uid)
    sizes = llama_param_sizes(args.model)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    slots = cfg.get("grad_slots", 0)          # > 0: streamed gradients (largest models)
    plan = paro.Plan(ctx, args.strategy, sizes, grad_slots=slots, **bench.plan_kwargs(args, stream.cuda_stream))
    info = plan.info()
    st = [torch.empty(info["os_numel"], dtype=torch.float32, device="cuda") for _ in range(3)]
    ptrs = [[x.data_ptr() for x in st]]
    plan.opt_state_init(rank, ptrs[0], seed=SEED)
    if not slots:
        plan.synth_grads(rank, SEED, 1)       # bench: gradients of step 1 stay resident
    steps = cfg.get("steps", 2)
    for s in range(1, steps + 1):
        if slots:
            plan.step_streamed(ptrs, bench.LR, s, seed=SEED, grad_step=1)
        else:
            plan.step(ptrs, bench.LR, s)
    stats = plan.stats()
    torch.cuda.synchronize()

    nb = info["n_buckets"]
    buckets = sorted(set(cfg.get("buckets", [0, nb // 2, nb - 1])))
    W = cfg.get("window", 2048)
    pbuf = plan.buffer(rank, 1)
    res = {"M": M, "strategy": args.strategy, "model": args.model, "bucket_elems": info["bucket_elems"], "n_buckets": nb,
           "psi_pad": info["psi_pad"], "stats": stats, "send": plan.send_bytes(rank), "os": [], "p": [],
           "bucket_ranges": [plan.bucket_range(b) for b in range(nb)],
           "os_ranges": [plan.shard_range("OS", rank, b) for b in range(nb)],
           "p_ranges": [plan.shard_range("P", rank, b) for b in range(nb)]}
    arrays = {}
    for level, key in (("OS", "os"), ("P", "p")):
        off = 0
        for b in range(nb):
            lo, hi = plan.shard_range(level, rank, b)
            if b in buckets:
                for (a, e) in windows_of(lo, hi, W):
                    name = f"{key}_{len(res[key])}"
                    la = off + (a - lo)
                    res[key].append({"bucket": b, "range": [lo, hi], "flat": [a, e], "local": la, "name": name})
                    if level == "OS":
                        for i, nm_ in enumerate(("master", "m", "v")):
                            arrays[f"{name}_{nm_}"] = st[i][la:la + (e - a)].cpu().numpy()
                    else:
                        arrays[f"{name}_param"] = d2h(pbuf + 2 * la, e - a, np.uint16)
            off += hi - lo
    np.savez(os.path.join(out, f"r{rank}.npz"), **arrays)
    with open(os.path.join(out, f"r{rank}.json"), "w") as f:
        json.dump(res, f)
    plan.close()
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
