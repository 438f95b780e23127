#!/usr/bin/env python
"""Single-GPU workload for `ncu --set full` on the collective rounds kernel
(the dominant kernel of the multi-GPU bench lines).  ncu must not profile a
multi-rank job, so this runs the emulated mode: all ranks of a 2x2 split on
one B200, every round one rounds_tma_kernel launch over every rank's tasks
(local operands instead of NVLink peers).  That captures the kernel's HBM
side (DRAM bytes vs the algorithmic 2 B per task input + 2 B per output
element, which the script prints) and its stall profile; the NVLink side is
measured live by bench.py / tools/coll_bench.py.

  python tools/ncu_rounds.py [elements] [strategy]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paro_synth import SEED  # noqa: E402


def main():
    from paper_2310_06003_b200 import paro
    n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 26)
    code = sys.argv[2] if len(sys.argv) > 2 else "IIG"
    N, M = 4, 2
    ctx = paro.Context(N, M, mode="emulated", device=0)
    pl = paro.Plan(ctx, code, [n], bucket_elems=n, fuse_allreduce=False)   # whole reduction in the rounds kernel
    for r in range(N):
        pl.synth_grads(r, SEED, 1)
    for _ in range(3):
        pl.collective(0)      # gradient reduction (RS_I + RS_E for IIG)
        pl.collective(1)      # parameter restore (AG_E)
    torch.cuda.synchronize()
    pl.profile_start(64)
    pl.collective(0)
    pl.collective(1)
    prof = pl.profile_stop()
    print({"elements": n, "strategy": code, "launches": prof["comm_launches"],
           "algorithmic_hbm_bytes": prof["comm_hbm_bytes"], "comm_ms": prof["comm_ms"],
           "alg_GBps": prof["comm_hbm_bytes"] / max(1e-9, prof["comm_ms"]) / 1e6})
    pl.close()
    ctx.close()


if __name__ == "__main__":
    main()
