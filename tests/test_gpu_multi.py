"""Real multi-GPU parity (one process per GPU, NCCL bootstrap, NVLink peer
memory): every rank's state after 2 steps equals the oracle's unsharded-DP
definition bit for bit.  Needs >= 2 GPUs (gpurun --gpus 2 / 4); runs on every
visible GPU and every split M | N (at 8 GPUs: 8x1, 4x2, 2x4, 1x8, the splits of
BASELINE configs 2-5)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import layout as L
from oracle import numerics as nm
from oracle import step as ST
from paro_synth import grad_bits, grad_flat, master_f32, master_flat

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _dp(lay, steps, accum=0, g_level="N", clip=0.0, wire="bf16", predivide=True):
    w = master_flat(lay.psi_pad, lay.real)
    m, v = np.zeros_like(w), np.zeros_like(w)
    for t in range(1, steps + 1):
        if wire != "bf16" or not predivide or lay.groups is not None:
            sc = nm.AdamScalars(3e-4, t, post_div=1 if predivide else lay.N)
            w, m, v, p, gh = ST.dp_step(lay, [grad_flat(r, t, lay.psi_pad, lay.real) for r in range(lay.N)], w, m,
                                        v, sc, wire=wire, predivide=predivide)
            sg = sc.s_g
            continue
        if clip:
            w, m, v, p, gh, nsq = ST.dp_clip_step(lay, [grad_bits(r, t, 0, lay.psi) for r in range(lay.N)],
                                                  w, m, v, 3e-4, t, clip_norm=clip)[:6]
            assert ST.clip_coef(nsq, clip) < 1.0
            sg = np.float32(1.0)
        elif accum:
            mb = [[grad_bits(r, (t << 8) | (k + 1), 0, lay.psi) for r in range(lay.N)] for k in range(accum)]
            w, m, v, p, gh = ST.dp_accum_step(lay, mb, w, m, v, nm.AdamScalars(3e-4, t, accum_steps=accum),
                                              g_level)
            sg = nm.AdamScalars(3e-4, t, accum_steps=accum).s_g
        else:
            w, m, v, p, gh = ST.dp_step(lay, [grad_bits(r, t, 0, lay.psi) for r in range(lay.N)], w, m, v,
                                        nm.AdamScalars(3e-4, t))
            sg = np.float32(1.0)
    return w, m, v, p, nm.grad_sq_sum(gh, sg)


CODES = ["NNN", "NNI", "NNG", "NII", "NIG", "NGG", "INI", "ING", "III", "IIG", "IGG", "GNG", "GIG", "GGG"]


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("variant", ["default", "paced_lsu", "accum", "clip", "copy_engine", "masked", "slots",
                                     "tma_thread_store", "fp32_wire", "predivide_off", "layer_windows", "consumer",
                                     "ce_tails"])
def test_real_ranks_match_oracle(tmp_path, variant):
    world = _ngpu()                  # every visible GPU: 2 (2x1, 1x2), 4 (4x1, 2x2, 1x4), 8 (8x1, 4x2, 2x4, 1x8)
    splits = [m for m in range(1, world + 1) if world % m == 0]
    cfg = {"splits": splits, "steps": 2, "sizes": [world * 64 * 40 + 24, 333], "bucket": world * 64 * 12,
           "codes": CODES, "topos": ["ho", "two_step", "direct"], "transports": ["push", "pull"]}
    if variant == "paced_lsu":   # emulated slow inter link (no fused hop) and the LSU kernels: same bits
        cfg.update({"codes": ["NNN", "IIG", "GGG", "NIG"], "topos": ["ho", "flat"], "transports": ["pull"],
                    "inter_gbps": 50.0, "comm_impl": "lsu"})
    if variant == "accum":       # gradient accumulation, s = 3 micro-batches per step (NEXT-1)
        cfg.update({"accum": 3, "topos": ["ho", "two_step"], "transports": ["pull", "push"], "windows": 2,
                    "adam_impl": "tma_store"})
    if variant == "copy_engine":   # all-gathers on the copy engines (barrier kernel + cudaMemcpyAsync)
        cfg.update({"topos": ["ho", "two_step", "h_ring"], "transports": ["pull"], "fuse_gather": "never",
                    "copy_engine": "all", "windows": 2})
    if variant == "clip":        # two-phase step with an active global-norm clip (NEXT-3)
        cfg.update({"clip_norm": 0.05, "topos": ["ho", "nccl"], "transports": ["pull", "push"],
                    "fuse_gather": "always"})
    if variant == "slots":       # streamed gradients: one bucket slot, reused by every bucket
        cfg.update({"grad_slots": 1, "topos": ["ho", "two_step", "direct"], "transports": ["pull", "push"]})
    if variant == "tma_thread_store":   # rounds kernel with thread stores (comm_impl 0; the default bulk-copies out)
        cfg.update({"topos": ["ho", "two_step", "direct"], "transports": ["push", "pull"], "comm_impl": "tma"})
    if variant == "fp32_wire":   # SURVEY 8(b) wire_dtype = 1; the NCCL comparator is checked at 1e-5 (A24)
        cfg.update({"wire": "fp32", "topos": ["ho", "two_step", "nccl"], "transports": ["pull", "push"]})
    if variant == "predivide_off":   # raw sums, 1/N in Adam; with the co-run Adam budget forced
        cfg.update({"predivide": False, "topos": ["ho", "direct"], "transports": ["pull"], "adam_smem_kb": 120})
    if variant == "layer_windows":   # layer-aligned buckets + per-layer forward/backward gathers (NEXT-2)
        d = world * 8
        cfg.update({"sizes": [d * 3 + 5] + [d * d, d * d + 7, 3 * d * d, d] * 3 + [d * 3 + 5],
                    "groups": [0, 1, 5, 9, 13], "topos": ["ho", "two_step"], "transports": ["pull", "push"],
                    "windows": 2})
    if variant == "consumer":    # per-bucket parameter consumer (incl. fused gathers: channel-3 barrier)
        cfg.update({"consumer": True, "topos": ["ho", "oneshot"], "transports": ["pull"], "fuse_gather": "always",
                    "grad_slots": 2})
    if variant == "ce_tails":    # copy_engine = 3: the all-reduce's all-gather rounds on the copy engines
        cfg.update({"copy_engine": "tails", "fuse_allreduce": False, "topos": ["ho", "two_step", "direct", "oneshot"],
                    "transports": ["pull"], "fuse_gather": "never"})
    if variant == "masked":      # partial / PEFT training: trainable plan + frozen-parameter plan
        cfg.update({"sizes": [world * 64 * 40 + 24, 333, world * 64 * 9 + 5, 4096], "mask": [0, 1, 0, 1],
                    "topos": ["ho", "two_step"], "transports": ["pull"], "windows": 2})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(ROOT, "tests", "dist_worker.py"),
           str(tmp_path), json.dumps(cfg)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=2400, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    mask = cfg.get("mask")
    tsizes = [x for x, t in zip(cfg["sizes"], mask) if t] if mask else cfg["sizes"]
    for M in splits:
        lay = L.Layout(tsizes, world, M, cfg["bucket"], groups=cfg.get("groups"))
        if mask:
            lay_f = L.Layout([x for x, t in zip(cfg["sizes"], mask) if not t], world, M, cfg["bucket"])
            p_frozen = nm.bf16_bits_from_f32(ST.pad_flat(master_f32(0, lay_f.psi), lay_f.psi_pad, np.float32))
        refs = {gl: _dp(lay, 2, cfg.get("accum", 0), gl, cfg.get("clip_norm", 0.0), cfg.get("wire", "bf16"),
                        cfg.get("predivide", True)) for gl in "NIG"}
        for code in cfg["codes"]:
            w, m, v, p, norm = refs[code[1]]
            for topo in cfg["topos"]:
              if topo == "nccl" and cfg.get("wire") == "fp32":
                  # NCCL's reduction order differs; on the fp32 wire that only moves fp32
                  # rounding, so the comparator meets the 1e-5 bar (A24) and bf16 params
                  # are within 1 ulp
                  for tr in cfg["transports"]:
                      for rank in range(world):
                          tag = f"{M}_{code}_{topo}_{tr}_r{rank}"
                          d = np.load(tmp_path / (tag + ".npz"))
                          ref_w = ST.shard_of(w, lay, code[2], rank).astype(np.float64)
                          rel = np.abs(d["master"].astype(np.float64) - ref_w) / np.maximum(np.abs(ref_w), 1e-3)
                          assert rel.max() <= 1e-5, (tag, rel.max())
                          pb = ST.shard_of(p, lay, code[0], rank).astype(np.int32)
                          assert np.abs(d["param"].astype(np.int32) - pb).max() <= 1, tag
                  continue
              if topo in ("flat", "nccl"):   # other reduction orders: flat = the oracle's flat ring,
                  continue                   # nccl = NCCL's (perf comparator; it must only run)
              for tr in cfg["transports"]:
                for rank in range(world):
                    tag = f"{M}_{code}_{topo}_{tr}_r{rank}"
                    d = np.load(tmp_path / (tag + ".npz"))
                    meta = json.load(open(tmp_path / (tag + ".json")))
                    assert np.array_equal(d["master"], ST.shard_of(w, lay, code[2], rank)), tag
                    assert np.array_equal(d["m"], ST.shard_of(m, lay, code[2], rank)), tag
                    assert np.array_equal(d["v"], ST.shard_of(v, lay, code[2], rank)), tag
                    assert np.array_equal(d["param"], ST.shard_of(p, lay, code[0], rank)), tag
                    assert abs(meta["stats"]["grad_norm"] ** 2 - norm) <= 1e-12 * norm, tag
                    # NVLink bytes counted on the device by the kernels that moved them equal the
                    # plan's per-rank transfer list (rank-symmetric schedules; Table 3 accounting;
                    # H-Ring's leaders pull more than they are pulled: its totals are checked below)
                    st_ = meta["stats"]
                    if topo != "h_ring":
                        assert (st_["moved_intra"], st_["moved_inter"]) == (st_["sent_intra"], st_["sent_inter"]), tag
                    if "consumed" in d:  # the consumer saw exactly the final parameters of every bucket
                        assert np.array_equal(d["consumed"], d["param"]), tag
                    if "full" in d:      # forward/backward parameter gather: the full bf16 model
                        assert np.array_equal(d["full"], p), tag
                    if mask:             # frozen tensors: untouched residency, full windows
                        assert np.array_equal(d["frozen_param"], ST.shard_of(p_frozen, lay_f, code[0], rank)), tag
                        assert np.array_equal(d["frozen_full"], p_frozen), tag
                if topo == "h_ring":
                    tot = np.zeros(4, np.int64)
                    for rank in range(world):
                        st_ = json.load(open(tmp_path / f"{M}_{code}_{topo}_{tr}_r{rank}.json"))["stats"]
                        tot += [st_["moved_intra"], st_["moved_inter"], st_["sent_intra"], st_["sent_inter"]]
                    assert (tot[0], tot[1]) == (tot[2], tot[3]), (M, code, topo, tr)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_collective_graph_replay(tmp_path):
    """The peer barriers keep their state on the device (per-channel launch
    generation advanced by each launch's last CTA), so collective launches can
    be captured once in a CUDA graph and replayed, also between eager calls:
    every replay's all-reduce equals the oracle (HO-Ring, one-shot, and HO-Ring
    with its all-gather rounds on the copy engines, copy_engine = 3)."""
    world = _ngpu()
    M = world // 2 if world >= 4 else 1
    B = world * 64 * 32
    cfg = {"M": M, "bucket": B, "topos": ["ho", "oneshot", "ho+ce"], "per_graph": 3, "replays": 4}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29519", os.path.join(ROOT, "tests", "graph_worker.py"),
           str(tmp_path), json.dumps(cfg)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lay = L.Layout([3 * B], world, M, B)
    gh = ST.dp_reduce(lay, [grad_bits(r_, 1, 0, lay.psi) for r_ in range(world)])
    for topo in cfg["topos"]:
        for rank in range(world):
            for k in range(cfg["replays"]):
                got = np.load(tmp_path / f"{topo}_r{rank}_k{k}.npy")
                for b, (s0, n) in enumerate(lay.buckets):   # bucket b's average in slot b % 3
                    assert np.array_equal(got[b * B:b * B + n], gh[s0:s0 + n]), (topo, rank, k, b)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("comm_impl", ["tma_store", "tma"])
def test_collective_allreduce_real_ranks(tmp_path, comm_impl):
    """BASELINE config 5 through real ranks: two back-to-back paro_collective(0)
    all-reduces per topology, at a bucket where the one-shot all-reduce runs as
    reduce-scatter + all-gather, with the bulk-store and thread-store rounds
    kernels, equal the oracle (HO-Ring / two-step / direct / one-shot:
    dp_reduce; flat: the oracle's flat ring), bucket by bucket with a ragged
    last bucket."""
    world = _ngpu()
    M = world // 2 if world >= 4 else 1
    B = world * 64 * 9000                      # one-shot at N >= 3: RS + AG (extra bytes > 6 MiB)
    n = 3 * B - world * 64 * 7                 # 3 buckets, ragged last
    topos = ["ho", "two_step", "direct", "oneshot", "flat"]
    cfg = {"M": M, "bucket": B, "n": n, "topos": topos, "comm_impl": comm_impl}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29521", os.path.join(ROOT, "tests", "coll_worker.py"),
           str(tmp_path), json.dumps(cfg)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lay = L.Layout([n], world, M, B)
    grads = [grad_bits(r_, 1, 0, lay.psi) for r_ in range(world)]
    gh = ST.dp_reduce(lay, grads)
    res = ST.strategy_step("NNN", lay, grads, ST.init_state(master_f32(0, lay.psi), lay, "NNN"),
                           nm.AdamScalars(3e-4, 1), topology="flat")
    for topo in topos:
        for rank in range(world):
            want = res.ghat_os[rank] if topo == "flat" else gh
            got = np.load(tmp_path / f"{topo}_r{rank}.npy")
            for b, (s0, nn) in enumerate(lay.buckets):    # bucket b in slot b % 3 (3 buckets: one each)
                assert np.array_equal(got[b * B:b * B + nn], want[s0:s0 + nn]), (topo, rank, b)
