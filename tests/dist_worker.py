"""Worker for the real multi-GPU parity test (launched by test_gpu_multi.py via
torchrun, one process per GPU).  Each rank runs real-mode paro_step (NCCL
bootstrap, peer-memory collectives) for every strategy / topology requested
and saves its state shards; the parent compares them with the oracle.

Also usable as a standalone smoke: torchrun --nproc-per-node 2 tests/dist_worker.py OUT
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paro_synth import SEED  # noqa: E402


def main():
    out = sys.argv[1]
    cfg = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_06003_b200 import paro
    splits = cfg.get("splits", [world])
    codes = cfg.get("codes", ["NNN", "IIG", "NIG", "IGG", "GGG", "III", "INI", "NNG"])
    topos = cfg.get("topos", ["ho", "two_step", "direct"])
    transports = cfg.get("transports", ["push"])
    comm_impl = cfg.get("comm_impl", "tma_store")
    inter_gbps = cfg.get("inter_gbps", 0.0)
    sizes = cfg.get("sizes", [world * 64 * 40 + 24, 333])
    B = cfg.get("bucket", world * 64 * 12)
    steps = cfg.get("steps", 2)
    accum = cfg.get("accum", 0)          # > 0: that many micro-batches per step (paro_accumulate)
    clip = cfg.get("clip_norm", 0.0)     # > 0: two-phase step with global-norm clipping
    windows = cfg.get("windows", 0)      # > 0: also gather every bucket through paro_gather_window
    adam_impl = cfg.get("adam_impl", "auto")
    fuse_gather = cfg.get("fuse_gather", "auto")
    copy_engine = cfg.get("copy_engine", False)
    mask = cfg.get("mask")               # partial / PEFT training: paro_plan_masked (NEXT-4)
    slots = cfg.get("grad_slots", 0)     # > 0: streamed gradients (paro_step_streamed)
    wire = cfg.get("wire", "bf16")       # wire_dtype (reading A3)
    predivide = cfg.get("predivide", True)
    adam_smem_kb = cfg.get("adam_smem_kb", 0)
    for M in splits:
        uid = paro.unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8)
        dist.broadcast(t, 0)
        ctx = paro.Context(world, M, mode="real", rank=rank, device=local, uid=bytes(t.tolist()))
        for code, topo, tr in [(c, t_, x) for c in codes for t_ in topos for x in transports]:
            if True:
                kw = dict(bucket_elems=B, topology=topo, transport=tr, comm_impl=comm_impl,
                          inter_gbps=inter_gbps, grad_accum=accum > 0, clip_norm=clip,
                          gather_windows=windows, adam_impl=adam_impl, fuse_gather=fuse_gather,
                          copy_engine=copy_engine, grad_slots=slots, wire_dtype=wire, predivide=predivide,
                          adam_smem_kb=adam_smem_kb, bucket_groups=cfg.get("groups"),
                          fuse_allreduce=cfg.get("fuse_allreduce", True))
                fz = None
                if mask:
                    pl, fz = paro.Plan.masked(ctx, code, sizes, mask, **kw)
                    fz.opt_state_init(rank, None, seed=SEED)
                else:
                    pl = paro.Plan(ctx, code, sizes, **kw)
                info = pl.info()
                st = [torch.empty(info["os_numel"], dtype=torch.float32, device="cuda") for _ in range(3)]
                ptrs = [[x.data_ptr() for x in st]]
                pl.opt_state_init(rank, ptrs[0], seed=SEED)
                consumed = None
                if cfg.get("consumer"):   # per-bucket parameter consumer: copies into a side buffer
                    consumed = torch.zeros(info["p_numel"], dtype=torch.int16, device="cuda")
                    rt = _rt()
                    pbase = pl.buffer(rank, 1)

                    def _cons(r, b, b0, b1, src, stream, consumed=consumed, pbase=pbase, rt=rt):
                        assert rt.cudaMemcpyAsync(consumed.data_ptr() + (src - pbase), src, 2 * (b1 - b0), 3,
                                                  stream) == 0
                    pl.set_param_consumer(_cons)
                stats = None
                for s in range(1, steps + 1):
                    if accum:
                        for k in range(accum):
                            pl.synth_grads(rank, SEED, (s << 8) | (k + 1))
                            pl.accumulate()
                    elif slots:
                        pl.step_streamed(ptrs, 3e-4, s, seed=SEED, grad_step=s)
                    else:
                        pl.synth_grads(rank, SEED, s)
                    if not slots:
                        pl.step(ptrs, 3e-4, s)
                    stats = pl.stats()
                torch.cuda.synchronize()
                pbuf = torch.empty(info["p_numel"], dtype=torch.int16, device="cuda")
                _copy(pbuf, pl.buffer(rank, 1))
                tag = f"{M}_{code}_{topo}_{tr}_r{rank}"
                extra = {}
                if windows:
                    parts = []
                    for b in range(info["n_buckets"]):
                        b0, b1 = pl.bucket_range(b)
                        ptr = pl.gather_window(rank, b, slot=b % windows)
                        torch.cuda.synchronize()
                        wb = torch.empty(b1 - b0, dtype=torch.int16, device="cuda")
                        _copy(wb, ptr)
                        parts.append(wb.cpu().numpy().view(np.uint16))
                    extra["full"] = np.concatenate(parts)
                if fz is not None:      # frozen parameters: residency and gathered windows
                    fi = fz.info()
                    fb = torch.empty(fi["p_numel"], dtype=torch.int16, device="cuda")
                    _copy(fb, fz.buffer(rank, 1))
                    extra["frozen_param"] = fb.cpu().numpy().view(np.uint16)
                    parts = []
                    for b in range(fi["n_buckets"]):
                        b0, b1 = fz.bucket_range(b)
                        ptr = fz.gather_window(rank, b, slot=b % max(1, windows))
                        torch.cuda.synchronize()
                        wb = torch.empty(b1 - b0, dtype=torch.int16, device="cuda")
                        _copy(wb, ptr)
                        parts.append(wb.cpu().numpy().view(np.uint16))
                    extra["frozen_full"] = np.concatenate(parts)
                    fz.close()
                if consumed is not None:
                    extra["consumed"] = consumed.cpu().numpy().view(np.uint16)
                np.savez(os.path.join(out, tag + ".npz"), master=st[0].cpu().numpy(), m=st[1].cpu().numpy(),
                         v=st[2].cpu().numpy(), param=pbuf.cpu().numpy().view(np.uint16), **extra)
                with open(os.path.join(out, tag + ".json"), "w") as f:
                    json.dump({"stats": stats, "send": pl.send_bytes(rank)}, f)
                pl.close()
        ctx.close()
        dist.barrier()
    dist.destroy_process_group()


def _rt():
    import ctypes
    import glob
    import nvidia.cuda_runtime as cr
    rt = ctypes.CDLL(glob.glob(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so*"))[0])
    rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    rt.cudaMemcpyAsync.restype = ctypes.c_int
    return rt


def _copy(dst, src_ptr):
    import ctypes
    import glob
    import nvidia.cuda_runtime as cr
    path = glob.glob(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so*"))[0]
    rt = ctypes.CDLL(path)
    rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    assert rt.cudaMemcpy(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src_ptr),
                         dst.numel() * dst.element_size(), 3) == 0


if __name__ == "__main__":
    main()
