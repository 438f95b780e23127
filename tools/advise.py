#!/usr/bin/env python
"""Rank the 14 PaRO strategies for a training task with paro_advise (Table 1 +
Table 2 memory + per-mini-batch communication, reading R29).

  python tools/advise.py --model 13B --gpus 8 --group-size 4 --accum 8 --mem-gb 160
  python tools/advise.py --psi 65e9 --gpus 128 --group-size 8 --accum 10 --mem-gb 80 \
      --bw-intra 300 --bw-inter 12.5            # the paper's A100 cluster
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paro_synth import llama_param_sizes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default=None, help="LLaMA list: 7B, 13B, 30B, 65B")
    ap.add_argument("--psi", type=float, default=None, help="parameter count (instead of --model)")
    ap.add_argument("--trainable", type=float, default=None, help="trainable parameters (default: all)")
    ap.add_argument("--peft", action="store_true")
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--group-size", type=int, default=4)
    ap.add_argument("--accum", type=int, default=1)
    ap.add_argument("--mem-gb", type=float, default=160.0, help="model-state budget per GPU")
    ap.add_argument("--bw-intra", type=float, default=770.0, help="GB/s per rank (B200 NVLink measured)")
    ap.add_argument("--bw-inter", type=float, default=770.0, help="GB/s per rank")
    a = ap.parse_args()
    from paper_2310_06003_b200 import paro
    psi = int(a.psi) if a.psi else sum(llama_param_sizes(a.model or "7B"))
    pt = int(a.trainable) if a.trainable else psi
    rows = paro.advise(a.gpus, a.group_size, psi, pt, a.accum, a.mem_gb * 1e9, a.bw_intra, a.bw_inter, a.peft)
    col = paro.paro_table1_column(psi, pt, 1 if a.peft else 0)
    print(f"psi={psi:,} trainable={pt:,} N={a.gpus} M={a.group_size} s={a.accum} "
          f"Table 1 column {col} budget {a.mem_gb} GB")
    print(f"{'code':5} {'rec':>3} {'fits':>4} {'mem GB':>8} {'intra GB':>9} {'inter GB':>9} {'t_comm ms':>10}")
    for r in rows:
        print(f"{r['code']:5} {int(r['recommended']):>3} {int(r['fits']):>4} {r['mem_bytes'] / 1e9:8.1f} "
              f"{r['intra_bytes'] / 1e9:9.2f} {r['inter_bytes'] / 1e9:9.2f} {r['t_s'] * 1e3:10.2f}")


if __name__ == "__main__":
    main()
