"""Pins for gradient accumulation in the oracle (s > 1 micro-batches).

* per-rank bytes counted by the round simulator equal Table 3's per-rank
  Backward R-S(G) + Update columns at s > 1 for PaRO-IGG / IIG / NIG (P:488-502,
  readings R12 and R13), and the closed form accum_units_per_rank;
* Eq. 1: the simulated saving of the grouped two-step reduction
  over the world reduction, at equal everything else, is Psi (s-1)(g-1)/N;
* small-integer gradients: g_hat is the exact mean over ranks and micro-batches
  (brute force; every order is exact);
* s = 1 reproduces the s = 1 step bit for bit (a special case);
* every strategy's round simulation equals the plain definition dp_accum_step.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

from oracle import accounting as A
from oracle import layout as L
from oracle import numerics as nm
from oracle import step as ST
from oracle import strategy as S
from paro_synth import edge_grad_bits, grad_bits, master_f32


def _mb(lay, s, t=1):
    return [[grad_bits(r, (t << 8) | k, 0, lay.psi) for r in range(lay.N)] for k in range(s)]


@pytest.mark.parametrize("N,M,s", [(8, 4, 3), (8, 2, 2), (4, 2, 4), (9, 3, 2)])
def test_table3_per_rank_volumes_with_accumulation(N, M, s):
    lay = L.Layout([N * 64 * 6], N, M, bucket_elems=N * 64 * 3)
    psi = lay.psi_pad
    w0 = master_f32(0, lay.psi)
    zero = [[np.zeros(lay.psi, np.uint16) for _ in range(N)] for _ in range(s)]
    sc = nm.AdamScalars(3e-4, 1, accum_steps=s)
    for meth, code in [("PaRO-IGG", "IGG"), ("PaRO-IIG", "IIG"), ("PaRO-NIG", "NIG")]:
        t = A.table3(meth, N, M, s, psi, corrected=True)
        want = [Fr(0), Fr(0)]
        for st in ("bwd_rs_g", "upd_rs_ar_g", "upd_ag_p"):
            want[0] += t[st][0] / N
            want[1] += t[st][1] / N
        assert tuple(want) == A.accum_units_per_rank(code, N, M, psi, s)
        res = ST.strategy_accum_step(code, lay, zero, ST.init_state(w0, lay, code), sc)
        for r in range(N):
            assert tuple(Fr(x) for x in res.sent[r]) == tuple(want), (code, r)


def test_eq1_from_accumulating_step_simulation():
    """NGG reduces every micro-batch globally (HO-RS), NIG groups it (RS_I per
    micro-batch + one RS_E); both then run the same HO-AG.  The per-rank
    difference is Eq. 1 -- 72,000 at the scaled config of S:580."""
    psi, N, M, s = 64000, 8, 2, 4
    lay = L.Layout([psi], N, M, bucket_elems=psi)
    assert lay.psi_pad == psi
    w0 = master_f32(0, psi)
    zero = [[np.zeros(psi, np.uint16) for _ in range(N)] for _ in range(s)]
    sc = nm.AdamScalars(3e-4, 1, accum_steps=s)
    a = ST.strategy_accum_step("NGG", lay, zero, ST.init_state(w0, lay, "NGG"), sc)
    b = ST.strategy_accum_step("NIG", lay, zero, ST.init_state(w0, lay, "NIG"), sc)
    for r in range(N):
        assert sum(a.sent[r]) - sum(b.sent[r]) == A.eq1_delta(psi, N, M, s) == 72000


@pytest.mark.parametrize("N,M", [(8, 4), (4, 1), (4, 4), (2, 2)])   # power-of-2 N: 1/N exact
def test_smallint_accumulation_is_exact_mean(N, M):
    s = 3
    lay = L.Layout([N * 64 * 5 + 3], N, M, bucket_elems=N * 64 * 2)
    mb = [[edge_grad_bits("smallint", lay.psi, rank=r, step=k + 1) for r in range(N)] for k in range(s)]
    exact = np.zeros(lay.psi, np.float64)
    for grads in mb:
        for gr in grads:
            exact += nm.f32_from_bf16_bits(gr).astype(np.float64)
    exact /= N          # mean over ranks; the micro-batch mean is s_g's job
    w0 = master_f32(0, lay.psi)
    sc = nm.AdamScalars(3e-4, 1, accum_steps=s)
    for code in S.paro_strategies():
        res = ST.strategy_accum_step(code, lay, mb, ST.init_state(w0, lay, code), sc)
        ol = code[2]
        for r in range(N):
            got = nm.f32_from_bf16_bits(res.ghat_os[r]).astype(np.float64)
            want = ST.shard_of(ST.pad_flat(exact, lay.psi_pad, np.float64), lay, ol, r)
            assert np.array_equal(got, want), (code, r)
        gr = (exact.astype(np.float32) * sc.s_g).astype(np.float64)   # fp32 unscale, as Adam sees it
        assert res.norm_sq == pytest.approx(float(np.sum(gr ** 2)), rel=1e-12)


def test_single_micro_batch_equals_plain_step():
    N, M = 8, 4
    lay = L.Layout([3000, 517, 9000], N, M, bucket_elems=N * 64 * 4)
    grads = [grad_bits(r, 1, 0, lay.psi) for r in range(N)]
    w0 = master_f32(0, lay.psi)
    sc = nm.AdamScalars(3e-4, 1)
    for code in S.paro_strategies():
        a = ST.strategy_step(code, lay, grads, ST.init_state(w0, lay, code), sc)
        b = ST.strategy_accum_step(code, lay, [grads], ST.init_state(w0, lay, code), sc)
        for r in range(N):
            for k in ("master", "m", "v", "param"):
                assert np.array_equal(a.state[r][k], b.state[r][k]), (code, r, k)
        assert a.sent == b.sent


@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (9, 3), (8, 1), (8, 8)])
def test_every_strategy_equals_accumulated_dp(N, M):
    s = 3
    lay = L.Layout([3000, 517, 64, 2000, 7], N, M, bucket_elems=N * 64 * 4)
    mb = _mb(lay, s)
    w0 = master_f32(0, lay.psi)
    wp = ST.pad_flat(w0, lay.psi_pad, np.float32)
    sc = nm.AdamScalars(3e-4, 1, accum_steps=s)
    ref = {gl: ST.dp_accum_step(lay, mb, wp, np.zeros_like(wp), np.zeros_like(wp), sc, gl) for gl in "NIG"}
    for code in S.paro_strategies():
        for topo in ("ho", "two_step"):
            res = ST.strategy_accum_step(code, lay, mb, ST.init_state(w0, lay, code), sc, topo)
            pl, gl, ol = code
            w, m, v, p, gh = ref[gl]
            for r in range(N):
                st = res.state[r]
                assert np.array_equal(st["master"], ST.shard_of(w, lay, ol, r)), (code, topo, r)
                assert np.array_equal(st["param"], ST.shard_of(p, lay, pl, r))
                assert np.array_equal(res.ghat_os[r], ST.shard_of(gh, lay, ol, r))


def test_g_level_changes_bits_but_not_meaning():
    """Where the micro-batch sum is taken changes bf16 rounding (R27): the three
    G levels give different bits at 2x4 with random gradients, and all stay
    within bf16 accumulation error of the exact mean."""
    N, M, s = 8, 4, 4
    lay = L.Layout([N * 64 * 16], N, M, bucket_elems=N * 64 * 8)
    mb = _mb(lay, s)
    wp = master_f32(0, lay.psi)
    sc = nm.AdamScalars(3e-4, 1, accum_steps=s)
    gh = {gl: ST.dp_accum_step(lay, mb, wp, np.zeros_like(wp), np.zeros_like(wp), sc, gl)[4] for gl in "NIG"}
    assert not np.array_equal(gh["N"], gh["G"]) and not np.array_equal(gh["I"], gh["G"])
    exact = sum(nm.f32_from_bf16_bits(gr).astype(np.float64) for grads in mb for gr in grads) / N
    for gl in "NIG":
        got = nm.f32_from_bf16_bits(gh[gl]).astype(np.float64)
        # each of <= N*s - 1 roundings is at most half an ulp (2^-9 relative) of a partial sum
        bound = (N * s) * 2.0 ** -9 * np.max(np.abs(exact)) + 1e-30
        assert np.max(np.abs(got - exact)) <= bound


def test_accum_scalars():
    sc = nm.AdamScalars(1e-3, 1, loss_scale=2.0, accum_steps=3)
    assert sc.s_g == np.float32(1.0 / 6.0)
    assert nm.AdamScalars(1e-3, 1).s_g == np.float32(1.0)
    with pytest.raises(ValueError):
        nm.AdamScalars(1e-3, 1, accum_steps=0)



# ------------------------------------------------------------- forward/backward parameter gather (NEXT-2)
@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (4, 2), (9, 3)])
def test_param_gather_is_complete_and_matches_table3(N, M):
    """Every rank ends with the full bf16 parameters (brute force), and the
    per-rank bytes equal Table 3's Forward A-G(P) column per micro-batch
    (P:454-490): MiCS / PaRO-IGG / PaRO-IIG gather intra-group (M-1)Psi/M;
    ZeRO-3 gathers (N-1)Psi/N in total over all links (its flat-ring split
    into intra / inter is a different topology, R14)."""
    lay = L.Layout([N * 64 * 20 + 8, 77], N, M, bucket_elems=N * 64 * 4)
    psi = lay.psi_pad
    full = nm.bf16_bits_from_f32(ST.pad_flat(master_f32(0, lay.psi), psi, np.float32))
    for code, meth in [("IGG", "PaRO-IGG"), ("IIG", "PaRO-IIG"), ("III", "MiCS"), ("GGG", "ZeRO-3"),
                       ("GIG", None), ("NNN", None)]:
        params = {r: ST.shard_of(full, lay, code[0], r) for r in range(N)}
        got, sent = ST.param_gather(code, lay, params)
        for r in range(N):
            assert np.array_equal(got[r], full), (code, r)
        if meth is None:
            continue
        t = A.table3(meth, N, M, 1, psi, corrected=True)["fwd_ag_p"]
        for r in range(N):
            if code[0] == "I":
                assert tuple(Fr(x) for x in sent[r]) == (t[0] / N, t[1] / N)
            else:
                assert Fr(sum(sent[r])) == (t[0] + t[1]) / N
