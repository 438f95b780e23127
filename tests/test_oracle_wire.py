"""Pins for the oracle's fp32 wire and pre-division options (CPU).

SURVEY §8(b) `wire_dtype` / `predivide`, reading A3 (wire dtype; G is 2 bytes,
P:225, so bf16 is the default and fp32 the option) and A4 (where 1/N applies).
On the fp32 wire every partial travels and is added in fp32 and g_hat reaches
Adam in fp32, so the result depends on the split only through fp32 summation
order: the cross-split / cross-bucket bar of §8(c-4) (1e-5, A24 metric) holds,
which the bf16 wire cannot meet.  The pins below tie the oracle to torch's own
fp32 arithmetic, to the exact (rational) sum within the textbook error bound of
recursive summation, and to the closed-form identities of pre-division.
"""
import math

import numpy as np
import pytest
import torch

from oracle import layout as L
from oracle import numerics as nm
from oracle import step as ST
from oracle import strategy as S
from paro_synth import grad_bits, master_f32

LR = 3e-4


def _a24(a, b):
    """elementwise |a - b| / max(|b|, 1e-3), max over elements."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-3)))


@pytest.mark.parametrize("N", [2, 3, 6, 8])
def test_pack_f32_and_hop_f32_match_torch(N):
    rng = np.random.default_rng(7 + N)
    bits = rng.integers(0, 1 << 16, size=200_000, dtype=np.uint32).astype(np.uint16)
    bits = bits[(bits & 0x7F80) != 0x7F80]
    g = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).float()
    ref = (g * torch.tensor(np.float32(1.0 / N))).numpy()
    got = nm.pack_f32(bits, 1.0 / N)
    assert got.dtype == np.float32 and np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    a = rng.standard_normal(100_000).astype(np.float32)
    b = (rng.standard_normal(100_000) * 1e-3).astype(np.float32)
    t = (torch.from_numpy(a) + torch.from_numpy(b)).numpy()
    assert np.array_equal(nm.hop_f32(a, b).view(np.uint32), t.view(np.uint32))


@pytest.mark.parametrize("N,M", [(8, 4), (6, 3), (9, 3), (4, 1)])
def test_fp32_wire_reduce_within_recursive_summation_bound(N, M):
    """|g_hat - sum_r g_r / N| <= (N - 1 + 1) u sum_r |g_r / N| (u = 2^-24): one
    rounding per pre-division and per fp32 addition (Higham, recursive
    summation), against the exact sum formed with math.fsum in double."""
    lay = L.Layout([N * 64 * 12 + 5], N, M, N * 64 * 4)
    grads = [grad_bits(r, 1, 0, lay.psi) for r in range(N)]
    gh = ST.dp_reduce(lay, grads, wire="fp32")
    assert gh.dtype == np.float32
    G = np.stack([nm.f32_from_bf16_bits(ST.pad_flat(g, lay.psi_pad, np.uint16)).astype(np.float64) / N
                  for g in grads])
    exact = np.array([math.fsum(G[:, i]) for i in range(lay.psi_pad)])
    bound = N * 2.0 ** -24 * np.abs(G).sum(0)
    assert np.all(np.abs(gh.astype(np.float64) - exact) <= bound)
    # and it is not the bf16 wire: rounding every hop to bf16 violates this bound
    gb = nm.f32_from_bf16_bits(ST.dp_reduce(lay, grads)).astype(np.float64)
    assert np.any(np.abs(gb - exact) > bound)


def test_fp32_wire_small_integers_exact_sum_and_mean():
    """Small integers: every order gives the exact sum (pre-division off) and,
    for N a power of two, the exact mean."""
    for (N, M) in [(8, 2), (8, 4), (6, 2), (4, 4)]:
        lay = L.Layout([N * 64 * 6], N, M, N * 64 * 2)
        rng = np.random.default_rng(N * 10 + M)
        ints = rng.integers(-3, 4, size=(N, lay.psi)).astype(np.float32)
        grads = [nm.bf16_bits_from_f32(x) for x in ints]
        s = ST.dp_reduce(lay, grads, wire="fp32", predivide=False)
        assert np.array_equal(s, ints.sum(0))
        if N & (N - 1) == 0:
            assert np.array_equal(ST.dp_reduce(lay, grads, wire="fp32"), ints.sum(0) / N)


def _ten_steps(N, M, B, wire, psi=1 << 15, steps=10):
    lay = L.Layout([psi], N, M, B)
    w = ST.pad_flat(master_f32(0, lay.psi), lay.psi_pad, np.float32)
    m, v = np.zeros_like(w), np.zeros_like(w)
    for t in range(1, steps + 1):
        w, m, v, p, _ = ST.dp_step(lay, [grad_bits(r, t, 0, lay.psi) for r in range(N)], w, m, v,
                                   nm.AdamScalars(LR, t), wire=wire)
    return w[:psi], p[:psi]


def test_cross_split_and_bucket_within_1e5_only_on_fp32_wire():
    """'Cross-split / cross-bucket: only with wire = fp32, <= 1e-5
    (A24 metric) vs dp_ref of any split'.  10 Adam steps at 8 ranks as 2x4
    (reference), 4x2, 8x1, 1x8 and two bucket sizes; the bf16 wire misses the bar
    (its per-hop roundings depend on the split), the fp32 wire meets it."""
    ref_w, _ = _ten_steps(8, 4, 1 << 12, "fp32")
    worst_f32, worst_bf16 = 0.0, 0.0
    ref_b, _ = _ten_steps(8, 4, 1 << 12, "bf16")
    for (M, B) in [(2, 1 << 12), (1, 1 << 12), (8, 1 << 12), (4, 1 << 10), (2, 3 * 1024)]:
        w, _ = _ten_steps(8, M, B, "fp32")
        worst_f32 = max(worst_f32, _a24(w, ref_w))
        wb, _ = _ten_steps(8, M, B, "bf16")
        worst_bf16 = max(worst_bf16, _a24(wb, ref_b))
    assert worst_f32 <= 1e-5, worst_f32
    assert worst_bf16 > 1e-5, worst_bf16


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (6, 3), (2, 1)])
@pytest.mark.parametrize("topo", ["ho", "two_step"])
def test_fp32_wire_every_strategy_equals_fp32_dp(N, M, topo):
    """On the fp32 wire the strategy simulators (actual rounds, fp32 partials,
    g_hat in fp32 through AG_E / HO-AG) give the fp32-wire DP definition bit for
    bit, like the bf16 wire does (the canonical order is the same)."""
    lay = L.Layout([N * 64 * 5 + 3, 200], N, M, N * 64 * 2)
    grads = [grad_bits(r, 1, 0, lay.psi) for r in range(N)]
    w0 = master_f32(0, lay.psi)
    wp = ST.pad_flat(w0, lay.psi_pad, np.float32)
    sc = nm.AdamScalars(LR, 1)
    w, m, v, p, gh = ST.dp_step(lay, grads, wp, np.zeros_like(wp), np.zeros_like(wp), sc, wire="fp32")
    for code in S.paro_strategies():
        res = ST.strategy_step(code, lay, grads, ST.init_state(w0, lay, code), sc, topology=topo, wire="fp32")
        for r in range(N):
            assert np.array_equal(res.state[r]["master"].view(np.uint32),
                                  ST.shard_of(w, lay, code[2], r).view(np.uint32)), (code, r)
            assert np.array_equal(res.state[r]["param"], ST.shard_of(p, lay, code[0], r)), (code, r)
        assert abs(res.norm_sq - nm.grad_sq_sum(gh)) <= 1e-12 * res.norm_sq


def test_predivide_off_equals_on_at_power_of_two_N():
    """Pre-division by N = 2^k is an exponent shift, which commutes with every
    round-to-nearest in the normal range: summing the raw gradients and
    unscaling by 1/N in Adam (s_g = 1/(loss_scale * N)) gives the same bits as
    dividing first (bf16 and fp32 wires).  For N = 6 the roundings differ, but
    the two stay within the bf16-hop tolerance of each other."""
    for wire in ("bf16", "fp32"):
        for (N, M) in [(8, 4), (4, 2)]:
            lay = L.Layout([N * 64 * 8], N, M, N * 64 * 4)
            grads = [grad_bits(r, 1, 0, lay.psi) for r in range(N)]
            w0 = ST.pad_flat(master_f32(0, lay.psi), lay.psi_pad, np.float32)
            z = np.zeros_like(w0)
            on = ST.dp_step(lay, grads, w0, z, z, nm.AdamScalars(LR, 1), wire=wire)
            off = ST.dp_step(lay, grads, w0, z, z, nm.AdamScalars(LR, 1, post_div=N), wire=wire, predivide=False)
            assert np.array_equal(on[0].view(np.uint32), off[0].view(np.uint32)), (wire, N)
    N, M = 6, 3
    lay = L.Layout([N * 64 * 8], N, M, N * 64 * 4)
    grads = [grad_bits(r, 1, 0, lay.psi) for r in range(N)]
    on = ST.dp_reduce(lay, grads)
    off = ST.dp_reduce(lay, grads, predivide=False)
    a, b = nm.f32_from_bf16_bits(on) * np.float32(6.0), nm.f32_from_bf16_bits(off)
    assert not np.array_equal(a, b)
    # each path: N - 1 hop roundings and N pack roundings of at most half a bf16 ulp
    # (2^-9 relative) of partials bounded by sum_r |g_r|
    gsum = np.sum([np.abs(nm.f32_from_bf16_bits(ST.pad_flat(g, lay.psi_pad, np.uint16))) for g in grads], axis=0)
    assert np.all(np.abs(a - b) <= 2 * N * 2.0 ** -9 * gsum)


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (6, 3)])
def test_fp32_wire_accumulation(N, M):
    """Gradient accumulation on the fp32 wire (R27 + R32): every strategy's
    simulated accumulating step equals dp_accum_step(wire = fp32) bit for bit;
    small integers accumulate to the exact sum; and the three G levels agree
    with each other far closer than on the bf16 wire (only fp32 order differs)."""
    s = 3
    lay = L.Layout([N * 64 * 6 + 5], N, M, N * 64 * 2)
    mb = [[grad_bits(r, (1 << 8) | (k + 1), 0, lay.psi) for r in range(N)] for k in range(s)]
    w0 = master_f32(0, lay.psi)
    wp = ST.pad_flat(w0, lay.psi_pad, np.float32)
    z = np.zeros_like(wp)
    sc = nm.AdamScalars(LR, 1, accum_steps=s)
    refs = {gl: ST.dp_accum_step(lay, mb, wp, z, z, sc, gl, wire="fp32") for gl in "NIG"}
    for code in S.paro_strategies():
        res = ST.strategy_accum_step(code, lay, mb, ST.init_state(w0, lay, code), sc, wire="fp32")
        w = refs[code[1]][0]
        for r in range(N):
            assert np.array_equal(res.state[r]["master"].view(np.uint32),
                                  ST.shard_of(w, lay, code[2], r).view(np.uint32)), (code, r)
    gh = {gl: refs[gl][4].astype(np.float64) for gl in "NIG"}
    scale = np.abs(gh["G"]).max()
    assert max(np.abs(gh["N"] - gh["G"]).max(), np.abs(gh["I"] - gh["G"]).max()) <= 1e-6 * scale
    ints = np.random.default_rng(N).integers(-3, 4, size=(s, N, lay.psi)).astype(np.float32)
    mbi = [[nm.bf16_bits_from_f32(ints[k, r]) for r in range(N)] for k in range(s)]
    for gl in "NIG":
        gi = ST.dp_accum_step(lay, mbi, wp, z, z, sc, gl, wire="fp32")[4]
        if N & (N - 1) == 0:
            assert np.array_equal(gi[:lay.psi], ints.sum((0, 1)) / N), gl
