#!/usr/bin/env python
"""Small N=1 paro_step workload for `ncu --set full` on the fused Adam kernel
(the bench's dominant kernel): 2^28 params in one flat tensor, 3 steps.  The
kernel is a grid-stride streaming kernel, so its per-element DRAM traffic and
stall profile are size-independent; bench.py scales the per-element bytes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paro_synth import SEED  # noqa: E402


def main():
    from paper_2310_06003_b200 import paro
    n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 28)
    ctx = paro.Context(1, 1, mode="real", rank=0, device=0, uid=paro.unique_id())
    pl = paro.Plan(ctx, "NNN", [n], bucket_elems=1 << 26)
    info = pl.info()
    st = [torch.empty(info["os_numel"], dtype=torch.float32, device="cuda") for _ in range(3)]
    ptrs = [[t.data_ptr() for t in st]]
    pl.opt_state_init(0, ptrs[0], seed=SEED)
    pl.synth_grads(0, SEED, 1)
    for s in range(1, 4):
        pl.step(ptrs, 3e-4, s)
    print(pl.stats())
    pl.close()
    ctx.close()


if __name__ == "__main__":
    main()
