"""Closed-form memory and communication accounting (oracle; test infrastructure only).

* Table 2: single-GPU memory of P, G, OS; widths 2Psi, 2Psi', K*Psi'
  with K = 12 for mixed-precision Adam.
* Table 3: cluster-total communication volume per stage, in
  parameter units; dagger entries are inter-group.  Literal cells are kept
  as printed, with the three readings R11-R13 applied only in the
  "corrected" view.
* Eq. 1: Delta_C = Psi (s-1)(g-1) / N.
* Per-strategy op lists and per-rank volumes of the s = 1 sync + update step
  (derived from P:195-202 and P:333-363).

Exact arithmetic: everything is Fraction.
"""
from __future__ import annotations

from fractions import Fraction as Fr

from .strategy import divisor, validate

K_ADAM = 12  # bytes of optimizer state per trainable parameter

NAMED_METHODS = ["ZeRO-1", "ZeRO-2", "ZeRO-3", "MiCS", "ZeRO++", "PaRO-IGG", "PaRO-IIG", "PaRO-NIG"]


# ----------------------------------------------------------------- Table 2
def memory_named(method, N, M, psi, K=K_ADAM):
    """Table 2 row -> (P, G, OS) bytes per GPU."""
    psi = Fr(psi)
    rows = {
        "ZeRO-1": (2 * psi, 2 * psi, K * psi / N),
        "ZeRO-2": (2 * psi, 2 * psi / N, K * psi / N),
        "ZeRO-3": (2 * psi / N, 2 * psi / N, K * psi / N),
        "MiCS": (2 * psi / M, 2 * psi / M, K * psi / M),
        "ZeRO++": (2 * psi / N + 2 * psi / M, 2 * psi / N, K * psi / N),
        "PaRO-IGG": (2 * psi / M, 2 * psi / N, K * psi / N),
        "PaRO-IIG": (2 * psi / M, 2 * psi / M, K * psi / N),
        "PaRO-NIG": (2 * psi, 2 * psi / M, K * psi / N),
    }
    return rows[method]


def memory_strategy(code, N, M, psi, psi_trainable=None, K=K_ADAM):
    """Generic strategy: P = 2Psi/div(P), G = 2Psi'/div(G), OS = K Psi'/div(OS)."""
    p, g, o = validate(code)
    pt = Fr(psi if psi_trainable is None else psi_trainable)
    return (Fr(2 * psi, divisor(p, N, M)), 2 * pt / divisor(g, N, M), K * pt / divisor(o, N, M))


# ----------------------------------------------------------------- Table 3
STAGES = ["fwd_ag_p", "bwd_ag_p", "bwd_rs_g", "upd_rs_ar_g", "upd_ag_p"]


def table3(method, N, M, s, psi, corrected=False):
    """Table 3 cluster totals {stage: (intra, inter)} in parameter units.

    corrected=False returns the cells as printed.  corrected=True applies
    R11 (MiCS update all-reduce read as a ring all-reduce of Psi/M over g ranks
    per position: 2(g-1)Psi/N per rank, all inter), R12 (no s on PaRO-IGG's
    update A-G(P)) and R13 (s on PaRO-NIG's backward R-S(G)).
    """
    g = N // M
    P = Fr(psi)
    z = (Fr(0), Fr(0))
    flat = lambda mult: ((N - g) * mult * P / N * (N - 1), g * mult * P / N * (N - 1))
    grp = lambda mult: (N * mult * P / M * (M - 1), Fr(0))
    if method == "ZeRO-1":
        a = flat(1)
        return {"fwd_ag_p": z, "bwd_ag_p": z, "bwd_rs_g": z,
                "upd_rs_ar_g": (2 * a[0], 2 * a[1]), "upd_ag_p": flat(1)}
    if method == "ZeRO-2":
        return {"fwd_ag_p": z, "bwd_ag_p": z, "bwd_rs_g": flat(s),
                "upd_rs_ar_g": z, "upd_ag_p": flat(1)}
    if method == "ZeRO-3":
        return {"fwd_ag_p": flat(s), "bwd_ag_p": flat(s), "bwd_rs_g": flat(s),
                "upd_rs_ar_g": z, "upd_ag_p": z}
    if method == "MiCS":
        if corrected:
            ar = (Fr(0), N * 2 * (g - 1) * P / N)
        else:
            ar = (2 * (N - g) * P / M * (g - 1), 2 * g * P / M * (g - 1))
        return {"fwd_ag_p": grp(s), "bwd_ag_p": grp(s), "bwd_rs_g": grp(s),
                "upd_rs_ar_g": ar, "upd_ag_p": z}
    if method == "ZeRO++":
        return {"fwd_ag_p": flat(s), "bwd_ag_p": grp(s), "bwd_rs_g": flat(s),
                "upd_rs_ar_g": z, "upd_ag_p": z}
    if method == "PaRO-IGG":
        ag_s = 1 if corrected else s
        return {"fwd_ag_p": grp(s), "bwd_ag_p": grp(s),
                "bwd_rs_g": (N * s * P / M * (M - 1), N * s * P / N * (g - 1)),
                "upd_rs_ar_g": z, "upd_ag_p": (Fr(0), N * ag_s * P / N * (g - 1))}
    if method == "PaRO-IIG":
        return {"fwd_ag_p": grp(s), "bwd_ag_p": grp(s), "bwd_rs_g": grp(s),
                "upd_rs_ar_g": (Fr(0), N * P / N * (g - 1)),
                "upd_ag_p": (Fr(0), N * P / N * (g - 1))}
    if method == "PaRO-NIG":
        rs_s = s if corrected else 1
        return {"fwd_ag_p": z, "bwd_ag_p": z, "bwd_rs_g": grp(rs_s),
                "upd_rs_ar_g": (Fr(0), N * P / N * (g - 1)),
                "upd_ag_p": (N * P / M * (M - 1), N * P / N * (g - 1))}
    raise KeyError(method)


def table3_totals(method, N, M, s, psi, corrected=False):
    t = table3(method, N, M, s, psi, corrected)
    return sum(v[0] for v in t.values()), sum(v[1] for v in t.values())


def eq1_delta(psi, N, M, s):
    """Eq. 1: per-GPU volume saved by the grouped two-step RS."""
    g = N // M
    return Fr(psi) * (s - 1) * (g - 1) / N


def eq1_lhs(psi, N, M, s):
    """Eq. 1 first line, term by term: s*(Psi/N)(N-1) - (s*(Psi/M)(M-1) + (Psi/N)(g-1))."""
    g = N // M
    P = Fr(psi)
    return s * P / N * (N - 1) - (s * P / M * (M - 1) + P / N * (g - 1))


# ----------------------------------------------------------------- step op lists
def step_ops(code):
    """Ordered collective primitives of one s = 1 sync + update step, per bucket.

    Gradient reduction to the OS residency, then Adam, then parameter restore
    to the P residency (Figs 1-3 narrative P:333-363):
      G in {N, G}: HO_RS ("HO-Ring reduce-scatter"); OS = I adds AG_E
                  of g_hat, OS = N adds HO_AG of g_hat (all-reduce).
      G = I:      RS_I, then RS_E if OS = G or AR_E if OS = I
                  (the MiCS partial all-reduce).
      restore:    OS = G, P = I -> AG_E; OS = G, P = N -> HO_AG;
                  OS = I, P = N -> AG_I; OS = P -> nothing.
    Returns (grad_ops, restore_ops).
    """
    p, g, o = validate(code)
    if g == "I":
        grad = ["RS_I", "RS_E"] if o == "G" else ["RS_I", "AR_E"]
    else:
        grad = ["HO_RS"] + ({"G": [], "I": ["AG_E"], "N": ["HO_AG"]}[o])
    if o == p:
        rest = []
    elif o == "G":
        rest = ["AG_E"] if p == "I" else ["HO_AG"]
    else:  # o == "I", p == "N"
        rest = ["AG_I"]
    return grad, rest


def primitive_units(prim, N, M, B):
    """Per-rank (intra, inter) units sent by one primitive on a bucket of B elements."""
    g = N // M
    B = Fr(B)
    return {
        "RS_I": ((M - 1) * B / M, Fr(0)),
        "AG_I": ((M - 1) * B / M, Fr(0)),
        "RS_E": (Fr(0), (g - 1) * B / N),
        "AG_E": (Fr(0), (g - 1) * B / N),
        "AR_E": (Fr(0), 2 * (g - 1) * B / N),
        "HO_RS": ((M - 1) * B / M, (g - 1) * B / N),
        "HO_AG": ((M - 1) * B / M, (g - 1) * B / N),
    }[prim]


def step_units_per_rank(code, N, M, psi):
    """Per-rank (intra, inter) parameter units sent in one s = 1 step."""
    grad, rest = step_ops(code)
    tot = [Fr(0), Fr(0)]
    for prim in grad + rest:
        a, b = primitive_units(prim, N, M, psi)
        tot[0] += a
        tot[1] += b
    return tuple(tot)


# ----------------------------------------------------------------- gradient accumulation
def accum_ops(code):
    """Primitives of a mini-batch step with s > 1 micro-batches (R27).

    Returns (per_micro_batch_ops, once_ops): the G-level reduction each
    micro-batch pays (G = G: HO_RS; G = I: RS_I, P:353/P:369;
    G = N: none, local accumulation), and the rest of the step paid once
    (G = I: RS_E or AR_E; G = N: the whole s = 1 reduction),
    followed by the parameter restore of step_ops.
    """
    p, g, o = validate(code)
    grad, rest = step_ops(code)
    if g == "G":
        return ["HO_RS"], rest
    if g == "I":
        return ["RS_I"], grad[1:] + rest
    return [], grad + rest


def accum_units_per_rank(code, N, M, psi, s):
    """Per-rank (intra, inter) parameter units of one mini-batch step with s micro-batches."""
    per_mb, once = accum_ops(code)
    tot = [Fr(0), Fr(0)]
    for prim, mult in [(x, s) for x in per_mb] + [(x, 1) for x in once]:
        a, b = primitive_units(prim, N, M, psi)
        tot[0] += mult * a
        tot[1] += mult * b
    return tuple(tot)
