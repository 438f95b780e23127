"""Full-size sampled parity: bench.py's timed launch configuration (LLaMA-7B
list, BASELINE.json configs[1] shape, the bench's strategy / split / bucket /
kernels) against the oracle, on sampled outputs the oracle computes one by one.

The step is elementwise once the reduction order is fixed (R2), so
the oracle's value of any flat window needs only that window's inputs:
oracle.step.dp_reduce_window (pinned against dp_reduce) + the canonical Adam.
Checked bit-exact after 2 steps: fp32 master / m / v and bf16 parameters in
windows at the start, middle and end of the rank's residency in the first,
middle and last bucket (the last is ragged); the whole shard map (every
bucket's OS and P range) and the per-rank bytes sent (exact, Table 3 / the
per-strategy closed form).  N = 1 in a subprocess; N = every visible GPU
(2 / 4 / 8) under torchrun when the box has them.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import accounting as A
from oracle import layout as L
from oracle import numerics as nm
from oracle import step as ST
from paro_synth import grad_bits, llama_param_sizes, master_f32

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LR = 3e-4   # bench.LR


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _expected(lay, a, e, steps):
    """Oracle master, m, v, param bits for flat window [a, e) after `steps`
    steps on the resident step-1 gradients (the bench's inputs)."""
    psi = lay.psi

    def grad_of(r, s, n):
        out = np.zeros(n, np.uint16)
        k = max(0, min(n, psi - s))
        if k:
            out[:k] = grad_bits(r, 1, s, k)
        return out

    parts, x = [], a
    while x < e:           # split at global-segment boundaries (the fold order changes there)
        j, p = lay.owner_segment(x)
        y = x
        for (s, n) in lay.buckets:
            if s <= x < s + n:
                c = n // lay.N
                y = min(e, s + ((x - s) // c + 1) * c)
        parts.append(ST.dp_reduce_window(lay, grad_of, x, y))
        x = y
    ghat = np.concatenate(parts)
    w = np.zeros(e - a, np.float32)
    k = max(0, min(e - a, psi - a))
    if k:
        w[:k] = master_f32(a, k)
    m, v = np.zeros_like(w), np.zeros_like(w)
    for t in range(1, steps + 1):
        w, m, v, p = nm.adam_update(w, m, v, ghat, nm.AdamScalars(LR, t))
    return w, m, v, p


def _run(tmp_path, world, cfg):
    worker = os.path.join(ROOT, "tests", "fullsize_worker.py")
    if world == 1:
        cmd = [sys.executable, worker, str(tmp_path), json.dumps(cfg)]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr=127.0.0.1", "--master-port=29523", worker, str(tmp_path), json.dumps(cfg)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    steps = cfg.get("steps", 2)
    for rank in range(world):
        res = json.load(open(tmp_path / f"r{rank}.json"))
        d = np.load(tmp_path / f"r{rank}.npz")
        code, M = res["strategy"], res["M"]
        lay = L.Layout(llama_param_sizes(res["model"]), world, M, res["bucket_elems"])
        # shard map and layout, every bucket, bit-exact
        assert res["psi_pad"] == lay.psi_pad and res["n_buckets"] == len(lay.buckets)
        assert [tuple(x) for x in res["bucket_ranges"]] == [(s, s + n) for (s, n) in lay.buckets]
        assert [tuple(x) for x in res["os_ranges"]] == lay.shard_ranges(code[2], rank)
        assert [tuple(x) for x in res["p_ranges"]] == lay.shard_ranges(code[0], rank)
        # bytes sent by this rank per step: the per-strategy closed form (Table 3 at s = 1)
        ai, ae = A.step_units_per_rank(code, world, M, lay.psi_pad)
        assert tuple(res["send"]) == (2 * ai, 2 * ae)
        assert (res["stats"]["sent_intra"], res["stats"]["sent_inter"]) == (2 * ai, 2 * ae)
        assert res["stats"]["nonfinite"] == 0 and np.isfinite(res["stats"]["grad_norm"])
        n_checked = 0
        for key in ("os", "p"):
            for wdw in res[key]:
                a, e = wdw["flat"]
                w, m, v, p = _expected(lay, a, e, steps)
                tag = (rank, key, wdw["bucket"], a, e)
                if key == "os":
                    for nm_, ref in (("master", w), ("m", m), ("v", v)):
                        got = d[f"{wdw['name']}_{nm_}"]
                        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (tag, nm_)
                else:
                    assert np.array_equal(d[f"{wdw['name']}_param"], p), tag
                n_checked += e - a
        assert n_checked > 0


def test_fullsize_7b_single_gpu(tmp_path):
    """N = 1: the default `python bench.py` configuration."""
    _run(tmp_path, 1, {"steps": 2})


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_fullsize_7b_multi_gpu(tmp_path):
    """Every visible GPU (2x1 / 2x2 / 2x4 at 2 / 4 / 8 GPUs, bench's default split):
    `bench.py --gpus N` under torchrun."""
    _run(tmp_path, _ngpu(), {"steps": 2})


@pytest.mark.skipif(_ngpu() < 4, reason="needs 4 GPUs")
def test_fullsize_30b_streamed_gradients(tmp_path):
    """The largest workload (BASELINE config 4's LLaMA-30B list, OS = G
    strategy GGG at 2 x (N/2): 2x2 on 4 GPUs (136 GB per rank), 2x4 on 8) with
    streamed gradients (4 slots): sampled windows bit-exact, shard map and bytes
    exact."""
    world = _ngpu()
    _run(tmp_path, world, {"steps": 2, "grad_slots": 4,
                           "bench_args": ["--model", "30B", "--strategy", "GGG", "--group-size", str(world // 2)]})
