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

import math

import numpy as np

from . import collectives as C
from .accounting import step_ops
from .layout import Layout
from .numerics import (F32, AdamScalars, adam_update, bf16_bits_from_f32, canonical_fold,
                       f32_from_bf16_bits, hop, hop_f32, pack, pack_f32)
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


def wire_ops(N, wire="bf16", predivide=True):
    """(pack, hop, dtype) of a wire (readings R2/R4, A3): bf16 wire: x =
    RNE_bf16(g * alpha) and the bf16 hop; fp32 wire: x = fp32(g) * alpha kept in
    fp32 and plain fp32 addition, g_hat in fp32.  alpha = 1/N with pre-division,
    1 without (the average is then taken in Adam's unscale, AdamScalars post_div)."""
    alpha = 1.0 / N if predivide else 1.0
    if wire == "bf16":
        return (lambda g: pack(g, alpha)), hop, np.uint16
    if wire == "fp32":
        return (lambda g: pack_f32(g, alpha)), hop_f32, F32
    raise ValueError(wire)


def dp_reduce(lay: Layout, grads, wire="bf16", predivide=True):
    """g_hat = CanonReduce(pack(grad_r)) over the N ranks (R2, R4): bf16 bits on
    the bf16 wire (pack = RNE_bf16(grad_r / N)), fp32 values on the fp32 wire."""
    N = lay.N
    geo = C.Geometry(N, lay.M)
    pk, op, dt = wire_ops(N, wire, predivide)
    X = [pk(pad_flat(gr, lay.psi_pad, np.uint16)) for gr in grads]
    ghat = np.zeros(lay.psi_pad, dt)
    for (s, n) in lay.buckets:
        segn = n // N
        for r in range(N):
            j, p = geo.jp(r)
            k = geo.seg(j, p)
            a, b = s + k * segn, s + (k + 1) * segn
            S = [canonical_fold([X[geo.r(jj, pp)][a:b] for pp in range(lay.M)], p, op)
                 for jj in range(geo.g)]
            ghat[a:b] = canonical_fold(S, j, op)
    return ghat


def dp_reduce_window(lay: Layout, grad_of, a, b, wire="bf16", predivide=True):
    """dp_reduce restricted to flat elements [a, b) (sampled parity at full size).

    The definition is elementwise, so a window needs only its own inputs:
    grad_of(r, a, n) returns rank r's bf16 gradient bits for [a, a + n).  The
    window must lie inside one global segment (the fold order depends on the
    owner (j, p) of the segment, R1/R2).  Pinned against dp_reduce.
    """
    N = lay.N
    geo = C.Geometry(N, lay.M)
    j, p = lay.owner_segment(a)
    if lay.owner_segment(b - 1) != (j, p):
        raise ValueError("window crosses a segment boundary")
    pk, op, _ = wire_ops(N, wire, predivide)
    X = [pk(np.asarray(grad_of(r, a, b - a), np.uint16)) for r in range(N)]
    S = [canonical_fold([X[geo.r(jj, pp)] for pp in range(lay.M)], p, op) for jj in range(geo.g)]
    return canonical_fold(S, j, op)


def dp_step(lay: Layout, grads, master, m, v, sc: AdamScalars, wire="bf16", predivide=True):
    """Unsharded data parallel with the canonical order (full-length arrays, Psi_pad).

    grads: list of N flat bf16-bit arrays (length Psi or Psi_pad).  wire /
    predivide: see wire_ops (without pre-division sc must carry post_div = N).
    Returns (master, m, v, param_bits, g_hat) -- g_hat as bf16 bits, or fp32
    values on the fp32 wire.
    """
    ghat = dp_reduce(lay, grads, wire, predivide)
    w2, m2, v2, pb = adam_update(master, m, v, ghat, sc)
    return w2, m2, v2, pb, ghat


def clip_coef(norm_sq, clip_norm):
    """Global-norm clipping coefficient (reading R28; the formula of
    torch.nn.utils.clip_grad_norm_): min(1, clip_norm / (||g|| + 1e-6)), in
    double; 1 when clipping is off (clip_norm <= 0)."""
    if clip_norm <= 0.0:
        return 1.0
    return min(1.0, float(F32(clip_norm)) / (math.sqrt(norm_sq) + 1e-6))


def dp_clip_step(lay: Layout, grads, master, m, v, lr, step, clip_norm=0.0, skip_nonfinite=False,
                 accum_steps=1, **adam_kw):
    """Two-phase step with global-norm clipping and non-finite skip (NEXT-3, R28).

    Phase 1 reduces every gradient and takes the norm of the unscaled
    gradient, ||fp32(g_hat) * s_g|| (s_g = 1 / (loss_scale * accum_steps)),
    over all elements; phase 2 runs Adam with the unscale factor
    s_g' = fp32(s_g_double * clip_coef).  With skip_nonfinite and any
    non-finite g_hat the step leaves master, m, v and the parameters unchanged.
    Returns (master, m, v, param_bits, g_hat_bits, norm_sq, coef, skipped).
    """
    ghat = dp_reduce(lay, grads)
    return clip_update(ghat, master, m, v, lr, step, clip_norm, skip_nonfinite, accum_steps, adam_kw)


def clip_update(ghat, master, m, v, lr, step, clip_norm, skip_nonfinite, accum_steps, adam_kw):
    sc0 = AdamScalars(lr, step, accum_steps=accum_steps, **adam_kw)
    g32 = ghat if np.asarray(ghat).dtype == F32 else f32_from_bf16_bits(ghat)   # bf16 bits or fp32 wire
    g = g32 * sc0.s_g
    norm_sq = float(np.sum(g.astype(np.float64) ** 2))
    nonfinite = not bool(np.all(np.isfinite(g32)))   # R9: a non-finite g_hat
    if skip_nonfinite and nonfinite:
        return (np.array(master, np.float32), np.array(m, np.float32), np.array(v, np.float32),
                bf16_bits_from_f32(master), ghat, norm_sq, 1.0, True)
    coef = clip_coef(norm_sq, clip_norm) if np.isfinite(norm_sq) else 1.0
    sc = AdamScalars(lr, step, accum_steps=accum_steps, clip_coef=coef, **adam_kw)
    w2, m2, v2, pb = adam_update(master, m, v, ghat, sc)
    return w2, m2, v2, pb, ghat, norm_sq, coef, False


def dp_accum_step(lay: Layout, grads_mb, master, m, v, sc: AdamScalars, g_level, wire="bf16"):
    """Unsharded data parallel with gradient accumulation (plain definition, R27).

    grads_mb[k][r]: rank r's flat bf16 gradient of micro-batch k (k = 1..s).
    The micro-batch sum is taken where the strategy keeps its gradient shard
    (P:344), so the result depends on the G level only:
      G = G: g_hat = Acc_k CanonReduce(x_k)
      G = I: S_j'  = Acc_k R_M(p; x_(j', 0..M-1), k);  g_hat = R_g(j; S_0..S_{g-1})
      G = N: y_r   = Acc_k x_(r, k);                    g_hat = CanonReduce(y)
    with Acc_k y_k = ((y_1 (+) y_2) (+) ...) (+) y_s and x = RNE_bf16(g / N).
    Then canonical Adam with sc built with accum_steps = s.  wire = "fp32":
    x = fp32(g) / N, every (+) and the accumulator in fp32 (R32).
    """
    N, M = lay.N, lay.M
    geo = C.Geometry(N, M)
    pk, op, dt = wire_ops(N, wire)
    X_mb = [[pk(pad_flat(gr, lay.psi_pad, np.uint16)) for gr in grads] for grads in grads_mb]

    def acc(ys):
        out = ys[0]
        for y in ys[1:]:
            out = op(out, y)
        return out

    if g_level == "N":
        Y = [acc([X[r] for X in X_mb]) for r in range(N)]
    ghat = np.zeros(lay.psi_pad, dt)
    for (s, n) in lay.buckets:
        segn = n // N
        for r in range(N):
            j, p = geo.jp(r)
            k = geo.seg(j, p)
            a, b = s + k * segn, s + (k + 1) * segn
            if g_level == "G":
                per_mb = []
                for X in X_mb:
                    S = [canonical_fold([X[geo.r(jj, pp)][a:b] for pp in range(M)], p, op) for jj in range(geo.g)]
                    per_mb.append(canonical_fold(S, j, op))
                ghat[a:b] = acc(per_mb)
            elif g_level == "I":
                S = [acc([canonical_fold([X[geo.r(jj, pp)][a:b] for pp in range(M)], p, op) for X in X_mb])
                     for jj in range(geo.g)]
                ghat[a:b] = canonical_fold(S, j, op)
            else:
                S = [canonical_fold([Y[geo.r(jj, pp)][a:b] for pp in range(M)], p, op) for jj in range(geo.g)]
                ghat[a:b] = canonical_fold(S, j, op)
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


def strategy_step(code, lay: Layout, grads, state, sc: AdamScalars, topology="ho", wire="bf16",
                  predivide=True):
    """One s = 1 step of strategy `code` on all N ranks.

    grads: list of N flat bf16-bit arrays.  state: from init_state (updated
    copies are returned, inputs untouched).  topology selects the schedule of
    the world-reaching gradient reduce-scatter and parameter all-gather used
    when G in {N, G}: "ho" (HO-Ring), "two_step" or
    "flat" (ring over all ranks, P:399 -- a different, still deterministic
    accumulation order) or "h_ring" (H-Ring all-gather with one leader per
    group, P:401-402 / S:378; its reduce-scatter is two-step).  G = I always runs RS_I then the inter op (Fig 2/3).
    wire / predivide: see wire_ops (fp32 wire: every partial and g_hat in fp32).
    """
    return _simulate(code, lay, [grads], state, sc, topology, accumulate=False, wire=wire, predivide=predivide)


def strategy_accum_step(code, lay: Layout, grads_mb, state, sc: AdamScalars, topology="ho", wire="bf16"):
    """One mini-batch step with gradient accumulation over s = len(grads_mb)
    micro-batches (§3.3; "each GPU maintains a gradient shard
    that accumulates gradients generated by each micro-batch").

    grads_mb[k][r] is rank r's flat bf16 gradient of micro-batch k.  Per
    micro-batch the gradient is reduced only to the G residency and added to
    the rank's accumulator there (reading R27):
      G = G: HO-Ring (or two-step / flat) RS of the micro-batch;
      G = I: intra-group RS_I ("synchronized through the
             intra-group reduce-scatter");
      G = N: nothing is exchanged; each rank accumulates its full gradient.
    Accumulator: acc_1 = r_1, acc_k = acc_{k-1} (+) r_k (the hop operator, G is
    2 bytes).  After the last micro-batch the rest of the reduction runs
    once on the accumulator (G = I: RS_E / AR_E, "performing an
    inter-group reduce-scatter operation only once"; G = N: the s = 1 reduction
    with the accumulator as input), then Adam and the parameter restore as in
    strategy_step.  The mean over micro-batches is folded into the unscale
    factor: pass AdamScalars(..., accum_steps=s).
    """
    return _simulate(code, lay, grads_mb, state, sc, topology, accumulate=True, wire=wire)


def _simulate(code, lay, grads_mb, state, sc, topology, accumulate, wire="bf16", predivide=True):
    pl, gl, ol = validate(code)
    N, M = lay.N, lay.M
    geo = C.Geometry(N, M)
    pk, hop, _ = wire_ops(N, wire, predivide)
    grad_ops, rest_ops = step_ops(code)
    res = StepResult(N)
    X_mb = [[pk(pad_flat(gr, lay.psi_pad, np.uint16)) for gr in grads] for grads in grads_mb]
    new = {r: {"master": [], "m": [], "v": [], "param": []} for r in range(N)}
    ghat_os = {r: [] for r in range(N)}
    gshard = {r: [] for r in range(N)}

    def world_rs(X):
        if topology == "ho":
            seg_out, tr, _S = C.rs_ho_ring(geo, X, hop)
            return seg_out, tr, None
        if topology in ("two_step", "h_ring"):   # H-Ring plans reduce two-step
            return C.rs_two_step(geo, X, hop)
        if topology == "flat":
            seg_out, tr = C.rs_flat_ring(geo, X, hop)
            return seg_out, tr, None
        raise ValueError(topology)

    def intra_rs(X):
        Y, r1 = C.rs_intra(geo, X, hop)
        t = C.Trace(M)
        t.extend(r1)
        return Y, t

    def inter_rs(Y):
        seg_out, r2 = C.rs_inter(geo, Y, hop)
        t = C.Trace(M)
        t.extend(r2)
        return seg_out, t

    for b, (s, n) in enumerate(lay.buckets):
        segn = n // N
        segs = lambda full, r: [full[r][s + k * segn: s + (k + 1) * segn] for k in range(N)]
        grp_partial = None
        if not accumulate:
            (X_full,) = X_mb
            X = {r: segs(X_full, r) for r in range(N)}
            # ---- gradient reduction to the OS residency
            if grad_ops[0] == "HO_RS":
                seg_out, tr, grp_partial = world_rs(X)
                _add_trace(res, tr)
            else:  # RS_I then RS_E / AR_E
                grp_partial, t1 = intra_rs(X)
                seg_out, t2 = inter_rs(grp_partial)
                _add_trace(res, t1)
                _add_trace(res, t2)
        else:
            acc = None
            for X_full in X_mb:
                X = {r: segs(X_full, r) for r in range(N)}
                if gl == "G":
                    red, tr, _ = world_rs(X)
                    _add_trace(res, tr)
                elif gl == "I":
                    red, tr = intra_rs(X)
                    _add_trace(res, tr)
                else:
                    red = {r: np.concatenate(X[r]) for r in range(N)}
                acc = red if acc is None else {r: hop(acc[r], red[r]) for r in range(N)}
            if gl == "G":
                seg_out = acc
            elif gl == "I":
                grp_partial = acc
                seg_out, tr = inter_rs(acc)
                _add_trace(res, tr)
            else:
                seg_out, tr, _ = world_rs({r: [acc[r][k * segn:(k + 1) * segn] for k in range(N)]
                                           for r in range(N)})
                _add_trace(res, tr)
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
            segs_, t = _ag(geo, seg_out, topology)
            _add_trace(res, t)
            gh = {r: np.concatenate([segs_[r][k] for k in range(N)]) for r in range(N)}
        # G residency: the value the strategy keeps as its gradient shard
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
            segs_, t = _ag(geo, adam_out, topology)
            _add_trace(res, t)
            pres = {r: np.concatenate([segs_[r][k] for k in range(N)]) for r in range(N)}
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
    u = np.concatenate(uniq)
    allg = (u if u.dtype == F32 else f32_from_bf16_bits(u)) * sc.s_g
    res.norm_sq = float(np.sum(allg.astype(np.float64) ** 2))
    res.nonfinite = bool(not np.all(np.isfinite(allg)))
    for r in range(N):
        res.state[r] = {k: np.concatenate(v) for k, v in new[r].items()}
        res.ghat_os[r] = np.concatenate(ghat_os[r])
        if gshard[r]:
            res.grad_shard[r] = np.concatenate(gshard[r])
    return res


def param_gather(code, lay: Layout, params, topology="ho"):
    """Forward / backward parameter all-gather of every bucket (P:195-196,
    P:338; Table 3 A-G(P) columns), simulated round by round.

    params[r]: rank r's bf16 parameter residency (bucket-major, as init_state /
    strategy_step keep it).  P = I: intra-group ring AG (AG_I); P = G: the
    world AG on `topology`; P = N: nothing moves.  Returns (full[r] = the
    gathered flat bf16 parameters of rank r, sent[r] = [intra, inter] units).
    """
    pl, _, _ = validate(code)
    N, M = lay.N, lay.M
    geo = C.Geometry(N, M)
    res = StepResult(N)
    full = {r: [] for r in range(N)}
    for b, (s, n) in enumerate(lay.buckets):
        own = {}
        for r in range(N):
            off = _offset_in_shard(lay, pl, r, b)
            a, e = lay.residency(pl, r, b)
            own[r] = params[r][off:off + (e - a)]
        if pl == "N":
            got = own
        elif pl == "I":
            ch, rounds = C.ag_intra(geo, own)
            t = C.Trace(M)
            t.extend(rounds)
            _add_trace(res, t)
            got = {r: np.concatenate(ch[r]) for r in range(N)}
        else:
            segs, t = _ag(geo, own, topology)
            _add_trace(res, t)
            got = {r: np.concatenate([segs[r][k] for k in range(N)]) for r in range(N)}
        for r in range(N):
            full[r].append(got[r])
    return {r: np.concatenate(full[r]) for r in range(N)}, res.sent


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
