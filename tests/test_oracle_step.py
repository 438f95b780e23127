"""Pins for oracle/step.py (CPU).

* every PaRO strategy x topology equals the unsharded-DP definition bit for bit
  (R2; the paper's equivalence claim P:549, P:654 in its strongest form);
* at N = 1 the step is torch.optim.AdamW on the local gradient (library routine);
* with small-integer gradients g_hat is the exact mean (brute force);
* parameter residency postcondition and the norm (fsum).
"""
import math

import numpy as np
import pytest
import torch

from oracle import layout as L
from oracle import numerics as nm
from oracle import step as ST
from oracle import strategy as S
from paro_synth import edge_grad_bits, grad_bits, master_f32


def _dp(lay, grads, w0, sc):
    wp = ST.pad_flat(w0, lay.psi_pad, np.float32)
    return ST.dp_step(lay, grads, wp, np.zeros_like(wp), np.zeros_like(wp), sc)


@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (9, 3), (4, 2), (8, 1), (8, 8), (2, 1), (1, 1)])
def test_all_strategies_equal_dp_one_step(N, M):
    sizes = [3000, 517, 64, 9000, 7]
    lay = L.Layout(sizes, N, M, bucket_elems=N * 64 * 4)
    grads = [grad_bits(r, 1, 0, lay.psi) for r in range(N)]
    w0 = master_f32(0, lay.psi)
    sc = nm.AdamScalars(3e-4, 1)
    w, m, v, p, gh = _dp(lay, grads, w0, sc)
    for code in S.paro_strategies():
        for topo in ("ho", "two_step"):
            res = ST.strategy_step(code, lay, grads, ST.init_state(w0, lay, code), sc, topo)
            pl, gl, ol = code
            for r in range(N):
                st = res.state[r]
                assert np.array_equal(st["master"], ST.shard_of(w, lay, ol, r))
                assert np.array_equal(st["m"], ST.shard_of(m, lay, ol, r))
                assert np.array_equal(st["v"], ST.shard_of(v, lay, ol, r))
                assert np.array_equal(st["param"], ST.shard_of(p, lay, pl, r))
                assert np.array_equal(res.ghat_os[r], ST.shard_of(gh, lay, ol, r))
            assert abs(res.norm_sq - nm.grad_sq_sum(gh)) <= 1e-12 * res.norm_sq


@pytest.mark.slow
def test_ten_steps_iig_and_nnn_equal_dp():
    N, M = 8, 4
    lay = L.Layout([N * 64 * 40 + 17], N, M, bucket_elems=N * 64 * 8)
    w0 = master_f32(0, lay.psi)
    wp = ST.pad_flat(w0, lay.psi_pad, np.float32)
    dw, dm, dv = wp, np.zeros_like(wp), np.zeros_like(wp)
    states = {c: ST.init_state(w0, lay, c) for c in ("IIG", "NNN", "GNG")}
    for t in range(1, 11):
        grads = [grad_bits(r, t, 0, lay.psi) for r in range(N)]
        sc = nm.AdamScalars(3e-4, t)
        dw, dm, dv, dp_, _ = ST.dp_step(lay, grads, dw, dm, dv, sc)
        for c in states:
            states[c] = ST.strategy_step(c, lay, grads, states[c], sc).state
    for c, st in states.items():
        for r in range(N):
            assert np.array_equal(st[r]["master"], ST.shard_of(dw, lay, c[2], r))
            assert np.array_equal(st[r]["param"], ST.shard_of(dp_, lay, c[0], r))


def test_n1_equals_torch_adamw():
    n = 5000
    lay = L.Layout([n], 1, 1, bucket_elems=1024)
    w0 = master_f32(0, n)
    wp = ST.pad_flat(w0, lay.psi_pad, np.float32)
    w, m, v = wp, np.zeros_like(wp), np.zeros_like(wp)
    p = torch.nn.Parameter(torch.from_numpy(w0.copy()))
    opt = torch.optim.AdamW([p], lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0,
                            foreach=False, fused=False)
    for t in range(1, 11):
        g = grad_bits(0, t, 0, n)
        w, m, v, pb, _ = ST.dp_step(lay, [g], w, m, v, nm.AdamScalars(3e-4, t))
        p.grad = torch.from_numpy(nm.f32_from_bf16_bits(g).copy())
        opt.step()
    assert np.max(np.abs(w[:n] - p.detach().numpy())) < 1e-8


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (9, 3)])
def test_smallint_grad_hat_is_exact_mean(N, M):
    lay = L.Layout([N * 64 * 3], N, M, bucket_elems=N * 64)
    grads = [edge_grad_bits("smallint", lay.psi, rank=r) for r in range(N)]
    w0 = master_f32(0, lay.psi)
    _, _, _, _, gh = _dp(lay, grads, w0, nm.AdamScalars(1e-3, 1))
    if N & (N - 1) == 0:   # 1/N exact for powers of two
        tot = sum(nm.f32_from_bf16_bits(g).astype(np.float64) for g in grads) / N
        assert np.array_equal(nm.f32_from_bf16_bits(gh).astype(np.float64), tot)
    for code in ("IIG", "NNN", "III"):
        res = ST.strategy_step(code, lay, grads, ST.init_state(w0, lay, code), nm.AdamScalars(1e-3, 1))
        for r in range(N):
            assert np.array_equal(res.ghat_os[r], ST.shard_of(gh, lay, code[2], r))


def test_residency_postcondition_and_specials():
    N, M = 4, 2
    lay = L.Layout([N * 64 * 4], N, M, bucket_elems=N * 64 * 2)
    grads = [edge_grad_bits("specials", lay.psi, rank=r) for r in range(N)]
    w0 = master_f32(0, lay.psi)
    sc = nm.AdamScalars(1e-3, 1)
    w, m, v, p, gh = _dp(lay, grads, w0, sc)
    for code in S.paro_strategies():
        res = ST.strategy_step(code, lay, grads, ST.init_state(w0, lay, code), sc)
        assert res.nonfinite
        for r in range(N):
            assert res.state[r]["param"].size == lay.shard_numel(code[0])
            got = nm.f32_from_bf16_bits(res.state[r]["param"])
            ref = nm.f32_from_bf16_bits(ST.shard_of(p, lay, code[0], r))
            assert np.array_equal(np.isnan(got), np.isnan(ref))
            ok = ~np.isnan(ref)
            assert np.array_equal(got[ok], ref[ok])


def test_norm_matches_fsum():
    N, M = 4, 2
    lay = L.Layout([N * 64 * 4], N, M, bucket_elems=N * 64 * 2)
    grads = [grad_bits(r, 1, 0, lay.psi) for r in range(N)]
    w0 = master_f32(0, lay.psi)
    sc = nm.AdamScalars(1e-3, 1, loss_scale=4.0)
    _, _, _, _, gh = _dp(lay, grads, w0, sc)
    for code in ("NNN", "III", "GGG"):
        res = ST.strategy_step(code, lay, grads, ST.init_state(w0, lay, code), sc)
        ref = math.fsum((float(x) * 0.25) ** 2 for x in nm.f32_from_bf16_bits(gh))
        assert abs(res.norm_sq - ref) <= 1e-12 * ref


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (2, 1), (6, 3)])
def test_reduce_window_equals_full_reduction(N, M):
    """dp_reduce_window (used by the full-size sampled parity tests) is the
    elementwise restriction of dp_reduce: every segment window, and ragged
    sub-windows, give the same bits; a window crossing a segment is refused."""
    sizes = [N * 64 * 5 + 17, 300]
    lay = L.Layout(sizes, N, M, N * 64 * 2)
    grads = [grad_bits(r, 3, 0, lay.psi) for r in range(N)]
    full = ST.dp_reduce(lay, grads)

    def grad_of(r, a, n):
        return ST.pad_flat(grads[r], lay.psi_pad, np.uint16)[a:a + n]

    rng = np.random.default_rng(N * 10 + M)
    for b in range(len(lay.buckets)):
        for k in range(N):
            a, e = lay.segment(b, k)
            assert np.array_equal(ST.dp_reduce_window(lay, grad_of, a, e), full[a:e])
            x = int(rng.integers(a, e - 1))
            y = int(rng.integers(x + 1, e + 1))
            assert np.array_equal(ST.dp_reduce_window(lay, grad_of, x, y), full[x:y])
    a, e = lay.segment(0, 0)
    with pytest.raises(ValueError):
        ST.dp_reduce_window(lay, grad_of, e - 3, e + 3)


def test_reduce_window_smallint_mean_at_llama_scale():
    """At the LLaMA-7B layout (2x4, 2^28 buckets) a window of small-integer
    gradients reduces to the exact mean (the sum is exact in any order)."""
    from paro_synth import edge_grad_bits, llama_param_sizes
    lay = L.Layout(llama_param_sizes("7B"), 8, 4, 1 << 28)
    b = len(lay.buckets) // 2
    a, e = lay.segment(b, 5)
    a, e = a + 1000, a + 1000 + 512

    def grad_of(r, s, n):
        return edge_grad_bits("smallint", n, rank=r, step=s % 97)

    got = nm.f32_from_bf16_bits(ST.dp_reduce_window(lay, grad_of, a, e)).astype(np.float64)
    ints = sum(nm.f32_from_bf16_bits(grad_of(r, a, e - a)).astype(np.float64) for r in range(8))
    assert np.array_equal(got, ints / 8)   # |sum| <= 24: every partial is exact in bf16
