"""Worker for the CUDA-graph replay test (torchrun, one process per GPU).

Barrier state lives on the device (launch generation per channel, advanced by
the last CTA of each launch), so collective launches carry no host-side
sequence numbers and a captured graph can be replayed: each rank captures
paro_collective(0) of an NNN plan (HO-Ring and one-shot) into a CUDA graph,
replays it several times interleaved with eager calls, and saves the g_hat
slots after every replay; the parent compares them with the oracle."""
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
    cfg = json.loads(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2310_06003_b200 import paro
    M = cfg["M"]
    uid = paro.unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    dist.broadcast(t, 0)
    ctx = paro.Context(world, M, mode="real", rank=rank, device=local, uid=bytes(t.tolist()))
    B = cfg["bucket"]
    for name in cfg["topos"]:
        # "<topo>+ce": copy_engine = 3 (the all-reduce's all-gather half on the copy engines, second stream)
        topo, ce = (name[:-3], "tails") if name.endswith("+ce") else (name, False)
        s = torch.cuda.Stream()
        pl = paro.Plan(ctx, "NNN", [3 * B], bucket_elems=B, topology=topo, fuse_allreduce=False,
                       stream=s.cuda_stream, copy_engine=ce)
        pl.synth_grads(rank, SEED, 1)
        with torch.cuda.stream(s):
            pl.collective(0)            # eager warm-up (kernel attributes, lazy peer access)
        torch.cuda.synchronize()
        dist.barrier()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(cfg["per_graph"]):
                pl.collective(0)
        torch.cuda.synchronize()
        dist.barrier()
        ghat = pl.buffer(rank, 3)
        for k in range(cfg["replays"]):
            g.replay()
            if k % 2 == 1:
                with torch.cuda.stream(s):
                    pl.collective(0)    # eager calls between replays share the device state
            torch.cuda.synchronize()
            buf = torch.empty(3 * B, dtype=torch.int16, device="cuda")
            _copy(buf, ghat)
            np.save(os.path.join(out, f"{name}_r{rank}_k{k}.npy"), buf.cpu().numpy().view(np.uint16))
        del g
        pl.close()
        dist.barrier()
    ctx.close()
    dist.destroy_process_group()


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
