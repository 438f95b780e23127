"""Pins for the two-phase clipped step of the oracle (NEXT-3, reading R28).

* N = 1: the clipped step is torch.nn.utils.clip_grad_norm_ followed by
  torch.optim.AdamW(foreach=False) (library routines), over several steps;
* the clipping coefficient and reported norm agree with clip_grad_norm_;
* a clip threshold above the norm is the unclipped step, bit for bit;
* after clipping, the norm of the gradient Adam sees is the threshold;
* non-finite gradients with skip leave the state untouched; without skip the
  coefficient is 1 (reported, not clipped).
"""
import math

import numpy as np
import pytest
import torch

from oracle import layout as L
from oracle import numerics as nm
from oracle import step as ST
from paro_synth import edge_grad_bits, grad_bits, master_f32

LR = 3e-4


def test_n1_clipped_matches_torch_clip_then_adamw():
    psi = 5000
    lay = L.Layout([psi], 1, 1, 1 << 12)
    w0 = master_f32(0, psi)
    w = ST.pad_flat(w0, lay.psi_pad, np.float32)
    m, v = np.zeros_like(w), np.zeros_like(w)
    pt = torch.nn.Parameter(torch.tensor(w0.astype(np.float64)).float())
    opt = torch.optim.AdamW([pt], lr=LR, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0, foreach=False)
    clip = 0.05
    for t in range(1, 6):
        g = grad_bits(0, t, 0, psi)
        w, m, v, p, gh, nsq, coef, skipped = ST.dp_clip_step(lay, [g], w, m, v, LR, t, clip_norm=clip)
        assert not skipped and coef < 1.0            # synthetic gradients have norm ~0.07 > 0.05
        pt.grad = torch.tensor(nm.f32_from_bf16_bits(g).copy())
        total = torch.nn.utils.clip_grad_norm_([pt], clip)
        assert math.sqrt(nsq) == pytest.approx(float(total), rel=1e-6)
        opt.step()
        assert np.max(np.abs(w[:psi] - pt.detach().numpy())) < 1e-8


def test_threshold_above_norm_is_the_unclipped_step():
    N, M = 8, 4
    lay = L.Layout([3000, 517, 9000], N, M, bucket_elems=N * 64 * 4)
    grads = [grad_bits(r, 1, 0, lay.psi) for r in range(N)]
    w = ST.pad_flat(master_f32(0, lay.psi), lay.psi_pad, np.float32)
    z = np.zeros_like(w)
    a = ST.dp_step(lay, grads, w, z, z, nm.AdamScalars(LR, 1))
    b = ST.dp_clip_step(lay, grads, w, z, z, LR, 1, clip_norm=1e3)
    assert b[6] == 1.0
    for x, y in zip(a[:5], b[:5]):
        assert np.array_equal(x, y)


def test_clipped_gradient_norm_equals_threshold():
    N, M = 8, 2
    lay = L.Layout([20000], N, M, bucket_elems=N * 64 * 8)
    grads = [grad_bits(r, 2, 0, lay.psi) for r in range(N)]
    w = ST.pad_flat(master_f32(0, lay.psi), lay.psi_pad, np.float32)
    z = np.zeros_like(w)
    for clip, ls, s in [(0.01, 1.0, 1), (0.003, 8.0, 1), (0.002, 1.0, 3)]:
        out = ST.dp_clip_step(lay, grads, w, z, z, LR, 1, clip_norm=clip, loss_scale=ls, accum_steps=s)
        gh, coef = out[4], out[6]
        assert coef < 1.0
        sg = nm.AdamScalars(LR, 1, loss_scale=ls, accum_steps=s, clip_coef=coef).s_g
        seen = math.sqrt(nm.grad_sq_sum(gh, sg))
        n = math.sqrt(out[5])
        assert seen == pytest.approx(clip * n / (n + 1e-6), rel=1e-6)   # the formula's 1e-6 guard


def test_nonfinite_skip_and_flag():
    N, M = 4, 2
    lay = L.Layout([N * 64 * 20], N, M, bucket_elems=N * 64 * 4)
    grads = [edge_grad_bits("specials", lay.psi, rank=r, step=1) for r in range(N)]
    w = ST.pad_flat(master_f32(0, lay.psi), lay.psi_pad, np.float32)
    z = np.zeros_like(w)
    out = ST.dp_clip_step(lay, grads, w, z, z, LR, 1, clip_norm=0.01, skip_nonfinite=True)
    assert out[7] is True
    assert np.array_equal(out[0], w) and np.array_equal(out[1], z) and np.array_equal(out[2], z)
    assert np.array_equal(out[3], nm.bf16_bits_from_f32(w))
    out2 = ST.dp_clip_step(lay, grads, w, z, z, LR, 1, clip_norm=0.01, skip_nonfinite=False)
    assert out2[7] is False and out2[6] == 1.0 and not np.isfinite(out2[5])
    ref = ST.dp_step(lay, grads, w, z, z, nm.AdamScalars(LR, 1))
    assert np.array_equal(np.isnan(out2[0]), np.isnan(ref[0]))
    ok = ~np.isnan(ref[0])
    assert np.array_equal(out2[0][ok], ref[0][ok])
