"""N-rank PaRO sync + update step and its unsharded-DP definition (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

`dp_step` is the plain definition (R2): every PaRO strategy is an
exact re-partitioning of data-parallel Adam, so with the canonical reduction
order fixed its result is

    x_r    = RNE_bf16(fp32(grad_r) * (1/N))                 (pack, R4)
    g_hat  = CanonReduce(x_0 .. x_{N-1})                     (R2)
    master, m, v, param = Adam(master, m, v, g_hat)          (R5-R7)

applied to every element.  `strategy_step` simulates one strategy on N ranks
the way the paper schedules it: the actual reduce-scatter /
all-reduce / all-gather rounds with byte counters, Adam only on each rank's
optimizer-state shard, then the parameter all-gathers back to the parameter
residency.  Tests require the two to agree bit for bit (same (N, M, B)).
"""
from __future__ import annotations

import numpy as np

from . import collectives as C
from .accounting import step_ops
from .layout import Layout
from .numerics import (AdamScalars, adam_update, bf16_bits_from_f32, canonical_fold,
                       f32_from_bf16_bits, hop, pack)
from .strategy import validate


def pad_flat(x, psi_pad, dtype):
    out = np.zeros(psi_pad, dtype=dtype)
    out[:x.size] = x
    return out


def shard_of(full, lay: Layout, level, r):
    """Bucket-major concatenation of rank r's residency ranges of a flat array."""
    return np.concatenate([full[a:b] for (a, b) in lay.shard_ranges(level, r)])


def init_state(master_full, lay: Layout, code, ranks=None):
    """Per-rank initial state from a full fp32 master vector (length Psi or Psi_pad).

    master/m/v cover the OS residency, param (bf16 bits) the P residency.
    """
    p, g, o = validate(code)
    mf = pad_flat(np.asarray(master_full, np.float32), lay.psi_pad, np.float32)
    pf = bf16_bits_from_f32(mf)
    out = {}
    for r in (range(lay.N) if ranks is None else ranks):
        ms = shard_of(mf, lay, o, r)
        out[r] = {"master": ms.copy(), "m": np.zeros_like(ms), "v": np.zeros_like(ms),
                  "param": shard_of(pf, lay, p, r)}
    return out


def dp_step(lay: Layout, grads, master, m, v, sc: AdamScalars):
    """Unsharded data parallel with the canonical order (full-length arrays, Psi_pad).

    grads: list of N flat bf16-bit arrays (length Psi or Psi_pad).
    Returns (master, m, v, param_bits, g_hat_bits).
    """
    N = lay.N
    geo = C.Geometry(N, lay.M)
    alpha = 1.0 / N
    X = [pack(pad_flat(gr, lay.psi_pad, np.uint16), alpha) for gr in grads]
    ghat = np.zeros(lay.psi_pad, np.uint16)
    for (s, n) in lay.buckets:
        segn = n // N
        for r in range(N):
            j, p = geo.jp(r)
            k = geo.seg(j, p)
            a, b = s + k * segn, s + (k + 1) * segn
            S = [canonical_fold([X[geo.r(jj, pp)][a:b] for pp in range(lay.M)], p)
                 for jj in range(geo.g)]
            ghat[a:b] = canonical_fold(S, j)
    w2, m2, v2, pb = adam_update(master, m, v, ghat, sc)
    return w2, m2, v2, pb, ghat


class StepResult:
    def __init__(self, N):
        self.state = {}
        self.sent = {r: [0, 0] for r in range(N)}   # units [intra, inter]
        self.rounds = 0
        self.ghat_os = {}          # rank -> bf16 bits over OS residency
        self.grad_shard = {}       # rank -> bf16 bits at the G residency (s = 1 reading)
        self.norm_sq = 0.0
        self.nonfinite = False


def _add_trace(res, tr):
    for r in res.sent:
        a, b = tr.sent(r)
        res.sent[r][0] += a
        res.sent[r][1] += b
    res.rounds += tr.n_rounds()


def strategy_step(code, lay: Layout, grads, state, sc: AdamScalars, topology="ho"):
    """One s = 1 step of strategy `code` on all N ranks.

    grads: list of N flat bf16-bit arrays.  state: from init_state (updated
    copies are returned, inputs untouched).  topology selects the schedule of
    the world-reaching gradient reduce-scatter and parameter all-gather used
    when G in {N, G}: "ho" (HO-Ring), "two_step" or
    "flat" (ring over all ranks, P:399 -- a different, still deterministic
    accumulation order) or "h_ring" (H-Ring all-gather with one leader per
    group, P:401-402 / S:378; its reduce-scatter is two-step).  G = I always runs RS_I then the inter op (Fig 2/3).
    """
    pl, gl, ol = validate(code)
    N, M = lay.N, lay.M
    geo = C.Geometry(N, M)
    alpha = 1.0 / N
    grad_ops, rest_ops = step_ops(code)
    res = StepResult(N)
    X_full = [pack(pad_flat(gr, lay.psi_pad, np.uint16), alpha) for gr in grads]
    new = {r: {"master": [], "m": [], "v": [], "param": []} for r in range(N)}
    ghat_os = {r: [] for r in range(N)}
    gshard = {r: [] for r in range(N)}
    for b, (s, n) in enumerate(lay.buckets):
        segn = n // N
        X = {r: [X_full[r][s + k * segn: s + (k + 1) * segn] for k in range(N)] for r in range(N)}
        # ---- gradient reduction to the OS residency
        if grad_ops[0] == "HO_RS":
            if topology == "ho":
                seg_out, tr, S = C.rs_ho_ring(geo, X, hop)
                grp_partial = None
            elif topology in ("two_step", "h_ring"):   # H-Ring plans reduce two-step
                seg_out, tr, grp_partial = C.rs_two_step(geo, X, hop)
            elif topology == "flat":
                seg_out, tr = C.rs_flat_ring(geo, X, hop)
                grp_partial = None
            else:
                raise ValueError(topology)
            _add_trace(res, tr)
        else:  # RS_I then RS_E / AR_E
            grp_partial, r1 = C.rs_intra(geo, X, hop)
            seg_out, r2 = C.rs_inter(geo, grp_partial, hop)
            t = C.Trace(M)
            t.extend(r1)
            t.extend(r2)
            _add_trace(res, t)
        # per-rank g_hat over the OS residency
        if ol == "G":
            gh = {r: seg_out[r] for r in range(N)}
        elif ol == "I":  # AG_E of the reduced segments (second half of AR_E)
            ch, rounds = C.ag_inter(geo, seg_out)
            t = C.Trace(M)
            t.extend(rounds)
            _add_trace(res, t)
            gh = {r: np.concatenate(ch[r]) for r in range(N)}
        else:  # OS = N: HO-Ring all-gather of g_hat (all-reduce = RS + AG)
            segs, t = _ag(geo, seg_out, topology)
            _add_trace(res, t)
            gh = {r: np.concatenate([segs[r][k] for k in range(N)]) for r in range(N)}
        # G residency (s = 1): the value the strategy keeps as its gradient shard
        for r in range(N):
            if gl == "G":
                gshard[r].append(seg_out[r])
            elif gl == "I":
                gshard[r].append(grp_partial[r])
        # ---- Adam on the OS shard
        adam_out = {}
        for r in range(N):
            a, e = lay.residency(ol, r, b)
            off = _offset_in_shard(lay, ol, r, b)
            st = state[r]
            w2, m2, v2, pb = adam_update(st["master"][off:off + (e - a)], st["m"][off:off + (e - a)],
                                         st["v"][off:off + (e - a)], gh[r], sc)
            new[r]["master"].append(w2)
            new[r]["m"].append(m2)
            new[r]["v"].append(v2)
            adam_out[r] = pb
            ghat_os[r].append(gh[r])
        # ---- parameter restore to the P residency
        if not rest_ops:
            pres = adam_out
        elif rest_ops == ["AG_E"]:
            ch, rounds = C.ag_inter(geo, adam_out)
            t = C.Trace(M)
            t.extend(rounds)
            _add_trace(res, t)
            pres = {r: np.concatenate(ch[r]) for r in range(N)}
        elif rest_ops == ["HO_AG"]:
            segs, t = _ag(geo, adam_out, topology)
            _add_trace(res, t)
            pres = {r: np.concatenate([segs[r][k] for k in range(N)]) for r in range(N)}
        elif rest_ops == ["AG_I"]:
            ch, rounds = C.ag_intra(geo, adam_out)
            t = C.Trace(M)
            t.extend(rounds)
            _add_trace(res, t)
            pres = {r: np.concatenate(ch[r]) for r in range(N)}
        else:
            raise AssertionError(rest_ops)
        for r in range(N):
            new[r]["param"].append(pres[r])
    # norm over unique elements (R8, R23)
    uniq = []
    if ol == "G":
        uniq = [np.concatenate(ghat_os[r]) for r in range(N)]
    elif ol == "I":
        uniq = [np.concatenate(ghat_os[geo.r(0, p)]) for p in range(M)]
    else:
        uniq = [np.concatenate(ghat_os[0])]
    allg = f32_from_bf16_bits(np.concatenate(uniq)) * sc.s_g
    res.norm_sq = float(np.sum(allg.astype(np.float64) ** 2))
    res.nonfinite = bool(not np.all(np.isfinite(allg)))
    for r in range(N):
        res.state[r] = {k: np.concatenate(v) for k, v in new[r].items()}
        res.ghat_os[r] = np.concatenate(ghat_os[r])
        if gshard[r]:
            res.grad_shard[r] = np.concatenate(gshard[r])
    return res


def _ag(geo, Z, topology):
    if topology == "ho":
        return C.ag_ho_ring(geo, Z)
    if topology == "two_step":
        return C.ag_two_step(geo, Z)
    if topology == "flat":
        return C.ag_flat_ring(geo, Z)
    if topology == "h_ring":
        return C.ag_h_ring(geo, Z)
    raise ValueError(topology)


def _offset_in_shard(lay: Layout, level, r, b):
    off = 0
    for bb in range(b):
        a, e = lay.residency(level, r, bb)
        off += e - a
    return off
