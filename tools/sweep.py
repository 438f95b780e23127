#!/usr/bin/env python
"""Diagnostic sweep (not the bench contract): under torchrun, time paro_step for
a grid of (strategy, topology, transport, comm_ctas, bucket) on one job and
print one JSON line per point (rank 0).  Usage:

  torchrun --nproc-per-node 2 tools/sweep.py --model 7B --grid '{"strategy":["IIG"],"comm_ctas":[32,64,148]}'
"""
import argparse
import itertools
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

from paro_synth import SEED, llama_param_sizes  # noqa: E402


def _cudart():
    import ctypes
    import glob
    import nvidia.cuda_runtime as cr
    rt = ctypes.CDLL(glob.glob(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so*"))[0])
    rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    rt.cudaMemcpyAsync.restype = ctypes.c_int
    return rt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7B")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--group-size", type=int, default=0)
    ap.add_argument("--grid", default="{}")
    ap.add_argument("--mem-cap-gb", type=float, default=172.0,
                    help="skip points whose per-rank HBM footprint (from a planning-only plan) exceeds this")
    ap.add_argument("--collective-only", action="store_true",
                    help="time paro_collective(reduce) + paro_collective(gather) per step, no Adam")
    a = ap.parse_args()
    grid = {"strategy": ["IIG"], "topology": ["ho"], "transport": ["pull"], "comm_ctas": [148],
            "bucket": [1 << 26], "depth": [2], "adam_impl": ["auto"], "comm_impl": ["tma_store"], "fuse_gather": ["auto"],
            "copy_engine": [0], "grad_slots": [0], "producer": ["synth"], "fuse_allreduce": [1]}
    grid.update(json.loads(a.grid))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world == 1:
        pass
    if world > 1:
        dist.init_process_group("cpu:gloo,cuda:nccl", rank=rank, world_size=world)
    from paper_2310_06003_b200 import paro
    M = a.group_size or (world // 2 if world >= 4 else 1)
    uid = paro.unique_id() if rank == 0 else bytes(128)
    if world > 1:
        t = torch.tensor(list(uid), dtype=torch.uint8)
        dist.broadcast(t, 0)
        uid = bytes(t.tolist())
    ctx = paro.Context(world, M, mode="real", rank=rank, device=local, uid=uid)
    sizes = llama_param_sizes(a.model)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    keys = list(grid.keys())
    pctx = paro.Context(world, M)     # planning only: memory check before allocating
    for vals in itertools.product(*[grid[k] for k in keys]):
        cfg = dict(zip(keys, vals))
        pp = paro.Plan(pctx, cfg["strategy"], sizes, bucket_elems=cfg["bucket"], topology=cfg["topology"],
                       transport=cfg["transport"], grad_slots=cfg["grad_slots"])
        pi = pp.info()
        pp.close()
        foot = (pi["grad_buffer_bytes"] + pi["mem_p_bytes"] + (pi["mem_g_bytes"] if pi["g_numel"] > 0 else 0)
                + pi["mem_os_bytes"] + pi["workspace_bytes"])
        if foot > a.mem_cap_gb * 1e9:
            if rank == 0:
                print(json.dumps({"cfg": cfg, "groups": f"{world // M}x{M}", "skipped": "OOM",
                                  "footprint_gb": round(foot / 1e9, 1),
                                  "table2_gb": round((pi["mem_p_bytes"] + pi["mem_g_bytes"] + pi["mem_os_bytes"]) / 1e9, 1)}),
                      flush=True)
            continue
        try:
            plan = paro.Plan(ctx, cfg["strategy"], sizes, bucket_elems=cfg["bucket"], topology=cfg["topology"],
                             comm_ctas=cfg["comm_ctas"], pipeline_depth=cfg["depth"], stream=stream.cuda_stream,
                             transport=cfg["transport"], adam_impl=cfg["adam_impl"],
                             comm_impl=cfg["comm_impl"], fuse_gather={1: "always", 0: "never"}.get(cfg["fuse_gather"], cfg["fuse_gather"]),
                             copy_engine=bool(cfg["copy_engine"]), grad_slots=cfg["grad_slots"],
                             fuse_allreduce=bool(cfg["fuse_allreduce"]) and not a.collective_only)
        except Exception as e:  # noqa: BLE001
            if rank == 0:
                print(json.dumps({"cfg": cfg, "error": str(e)}), flush=True)
            continue
        info = plan.info()
        st = [torch.empty(info["os_numel"], dtype=torch.float32, device="cuda") for _ in range(3)]
        ptrs = [[x.data_ptr() for x in st]]
        plan.opt_state_init(rank, ptrs[0], seed=SEED)
        if not cfg["grad_slots"]:
            plan.synth_grads(rank, SEED, 1)
        producer = None
        if cfg["grad_slots"] and cfg["producer"] == "copy":
            # the "backward" hands over each bucket from one resident bucket-sized buffer
            # (2 B read + 2 B written per element, like a real backward's gradient write)
            srcbuf = torch.empty(info["bucket_elems"], dtype=torch.int16, device="cuda").random_(-32768, 32767)
            rt = _cudart()

            def producer(r, b, b0, b1, dst, strm, srcbuf=srcbuf, rt=rt):
                rt.cudaMemcpyAsync(dst, srcbuf.data_ptr(), 2 * (b1 - b0), 3, strm)
        s = 0
        def one_step(s):
            if a.collective_only:
                plan.collective(0)
                plan.collective(1)
            elif cfg["grad_slots"]:   # gradients produced per bucket inside the step (2 B/param written)
                plan.step_streamed(ptrs, 3e-4, s, seed=SEED, grad_step=1, producer=producer)
            else:
                plan.step(ptrs, 3e-4, s)
        for _ in range(a.warmup):
            s += 1
            one_step(s)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        plan.profile_start((info["n_comm_launches"] + info["n_buckets"] + 8) * a.steps + 64)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            s += 1
            one_step(s)
        e1.record(stream)
        torch.cuda.synchronize()
        prof = plan.profile_stop()
        ms = e0.elapsed_time(e1) / a.steps
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(json.dumps({"cfg": cfg, "groups": f"{world // M}x{M}", "ms": round(float(tt.item()), 3),
                              "Gparam_s": round(info["psi"] / float(tt.item()) / 1e6, 1),
                              "adam_ms": round(prof["adam_ms"] / a.steps, 3),
                              "comm_ms": round(prof["comm_ms"] / a.steps, 3),
                              "comm_launch_us": round(1000 * prof["comm_ms"] / max(1, prof["comm_launches"]), 1),
                              "comm_GBps": round(prof["comm_bytes"] / max(1e-9, prof["comm_ms"]) / 1e6, 1),
                              "adam_GBps": round(28 * prof["adam_elems"] / max(1e-9, prof["adam_ms"]) / 1e6, 1),
                              "send_bytes": info["step_send_bytes_intra"] + info["step_send_bytes_inter"],
                              "footprint_gb": round(foot / 1e9, 1),
                              "trace": {k: round(prof[k], 3) for k in ("traced_launches", "traced_barrier_ms",
                                                                      "traced_work_ms", "traced_final_ms")}}),
                  flush=True)
        del st
        plan.close()
        torch.cuda.empty_cache()
    pctx.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
