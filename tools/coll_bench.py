#!/usr/bin/env python
"""All-reduce bus bandwidth sweep (BASELINE config 5): our HO-Ring / flat ring /
two-step / direct all-reduce (paro_collective on an NNN plan: hierarchical
RS + AG with the bf16 hop arithmetic) against torch.distributed.all_reduce
(NCCL) on the same bf16 size.  busbw = S * 2(N-1)/N / t (nccl-tests convention).
Run under torchrun; prints one JSON line per point on rank 0."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # JSON lines only on stdout
if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,4,16,64,256,1024,4096")
    ap.add_argument("--topos", default="ho,flat,two_step,direct")
    ap.add_argument("--group-size", type=int, default=0)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--comm-ctas", type=int, default=0)
    ap.add_argument("--transport", default="pull")
    ap.add_argument("--comm-impl", default="tma_store")
    ap.add_argument("--inter-gbps", type=float, default=0.0, help="emulated inter-group link (0 = off)")
    ap.add_argument("--trace", action="store_true",
                    help="per-launch device trace of the collective (barrier / work / final-barrier us)")
    ap.add_argument("--op", default="ar", choices=["ar", "ag"],
                    help="ar: gradient all-reduce (NNN plan, reduce launches); ag: parameter all-gather "
                         "(NNG plan, gather launches) as in the paper's section 4.4")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("cpu:gloo,cuda:nccl", rank=rank, world_size=world)
    from paper_2310_06003_b200 import paro
    M = a.group_size or (world // 2 if world >= 4 else 1)
    uid = paro.unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    dist.broadcast(t, 0)
    ctx = paro.Context(world, M, mode="real", rank=rank, device=local, uid=bytes(t.tolist()))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    host_us = {}

    def timeit(fn):
        import time
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        for _ in range(a.iters):
            fn()
        host_us["last"] = (time.perf_counter() - t0) * 1e6 / a.iters   # enqueue cost per call (host)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / a.iters], dtype=torch.float64, device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    for mb in [float(x) for x in a.sizes_mb.split(",")]:
        nbytes = int(mb * (1 << 20))
        elems = nbytes // 2
        row = {"bytes": nbytes, "groups": f"{world // M}x{M}", "n_gpus": world, "inter_gbps": a.inter_gbps,
               "comm_ctas": a.comm_ctas, "entry_barrier": os.environ.get("PARO_ENTRY_BARRIER", "1")}
        factor = 2 * (world - 1) / world if a.op == "ar" else (world - 1) / world
        code, what = ("NNN", 0) if a.op == "ar" else ("NNG", 1)
        for name in a.topos.split(","):
            # "<topo>+ce": copy_engine = 3 (the all-gather half of the all-reduce on the copy engines)
            topo, ce = (name[:-3], "tails") if name.endswith("+ce") else (name, False)
            bucket = min(elems, 1 << 28)
            pl = paro.Plan(ctx, code, [elems], bucket_elems=bucket, topology=topo, comm_ctas=a.comm_ctas,
                           stream=stream.cuda_stream, transport="pull" if topo == "oneshot" else a.transport,
                           comm_impl=a.comm_impl, copy_engine=ce,
                           inter_gbps=a.inter_gbps, fuse_gather="never", fuse_allreduce=False)
            pl.synth_grads(rank, 1234, 1)
            ms = timeit(lambda: pl.collective(what))
            row[name] = {"ms": round(ms, 4), "busbw_GBps": round(nbytes * factor / (ms / 1e3) / 1e9, 1),
                         "host_us_per_call": round(host_us["last"], 2)}
            if a.trace:
                pl.profile_start(64)
                for _ in range(4):
                    pl.collective(what)
                torch.cuda.synchronize()
                pr = pl.profile_stop()
                nl = max(1, pr["traced_launches"])
                row[name]["trace_us_per_launch"] = {
                    "event": round(1000 * pr["comm_ms"] / max(1, pr["comm_launches"]), 2),
                    "barrier": round(1000 * pr["traced_barrier_ms"] / nl, 2),
                    "work": round(1000 * pr["traced_work_ms"] / nl, 2),
                    "final": round(1000 * pr["traced_final_ms"] / nl, 2)}
            pl.close()
        if a.no_nccl:
            if rank == 0:
                print(json.dumps(row), flush=True)
            continue
        x = torch.ones(elems, dtype=torch.bfloat16, device="cuda")
        if a.op == "ar":
            ms = timeit(lambda: dist.all_reduce(x))
        else:
            part = x[rank * (elems // world):(rank + 1) * (elems // world)]
            ms = timeit(lambda: dist.all_gather_into_tensor(x, part))
        row["nccl_" + ("allreduce" if a.op == "ar" else "allgather")] = {
            "ms": round(ms, 4), "busbw_GBps": round(nbytes * factor / (ms / 1e3) / 1e9, 1)}
        row["op"] = a.op
        del x
        torch.cuda.empty_cache()
        if rank == 0:
            print(json.dumps(row), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
