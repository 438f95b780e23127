#!/usr/bin/env python
"""CPU baseline per strategy (SURVEY §8(d) "oracle timing"): one full step of
every PaRO code with all N simulated ranks in one process, BASELINE configs[0]
(the 4M-parameter flat model, 8 ranks as 2 groups x 4, 2^18-element buckets),
NumPy single thread.  Prints one JSON line per code: params/s = Psi / t_step.
Test infrastructure (it executes oracle/), not the product path.

  OMP_NUM_THREADS=1 python tools/oracle_timing.py [--psi 4194304] [--N 8] [--M 4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import layout as L  # noqa: E402
from oracle import numerics as nm  # noqa: E402
from oracle import step as ST  # noqa: E402
from oracle import strategy as S  # noqa: E402
from paro_synth import grad_bits, master_f32  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--psi", type=int, default=1 << 22)
    ap.add_argument("--N", type=int, default=8)
    ap.add_argument("--M", type=int, default=4)
    ap.add_argument("--bucket", type=int, default=1 << 18)
    a = ap.parse_args()
    lay = L.Layout([a.psi], a.N, a.M, a.bucket)
    w0 = master_f32(0, lay.psi)
    grads = [grad_bits(r, 1, 0, lay.psi) for r in range(a.N)]
    sc = nm.AdamScalars(3e-4, 1)
    for code in S.paro_strategies():
        state = ST.init_state(w0, lay, code)
        t0 = time.perf_counter()
        ST.strategy_step(code, lay, grads, state, sc)
        dt = time.perf_counter() - t0
        print(json.dumps({"code": code, "psi": lay.psi, "ranks": f"{a.N // a.M}x{a.M}", "bucket": a.bucket,
                          "s_per_step": round(dt, 3), "params_per_s": lay.psi / dt, "cores": 1,
                          "host_cpus": os.cpu_count(), "kind": "oracle"}), flush=True)


if __name__ == "__main__":
    main()
