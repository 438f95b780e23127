"""Strategy advisor: Table 1 + Table 2 + mini-batch volumes (oracle; test infrastructure only).

NEXT-4 of SURVEY §8(f).  The paper's guideline for picking a strategy is
Table 1 (which of the 14 codes are recommended for each training
type) together with the memory/communication trade-off of §3.1:
finer sharding saves memory (Table 2) and costs communication (Table 3).
The paper gives no selection algorithm, so the advisor is reading R29
(DESIGN.md §3):

  column   Psi' = Psi -> 0, Psi' >= Psi/6 -> 1, Psi' < Psi/6 -> 2, PEFT -> 3
           (PEFT is a training type, passed explicitly: "Psi' << Psi")
  memory   P + G + OS per GPU = 2 Psi/div(P) + 2 Psi'/div(G) + 12 Psi'/div(OS)
           ("2Psi, 2Psi', 12Psi'", Table 2)
  volume   per rank per mini-batch of s micro-batches, parameter units:
             s * 2 * AG(P) over Psi    forward + backward parameter all-gather
                                       (P = I: AG_I,
                                       P = G: HO-AG, P = N: none)
           + accum_units_per_rank over Psi'   gradient reduction + update-stage
                                       ops + parameter restore (R27)
           bytes = 2 * units (bf16 wire, R3)
  time     t = intra_bytes / B_intra + inter_bytes / B_inter   (the per-rank
           link model of §2.2, where inter bandwidth is the bottleneck)
  ranking  recommended-and-fitting codes first, by (t, memory, code); then the
           rest by the same key.

Sizes are padded like the plan (R21: Psi and Psi' each to a multiple of
N * 64) so every byte count is an integer.
"""
from __future__ import annotations

from fractions import Fraction as Fr

from .accounting import K_ADAM, accum_units_per_rank, primitive_units
from .strategy import divisor, paro_strategies, validate

# Table 1, transcribed row by row: 1 = check mark, 0 = cross.
# Columns: Psi' = Psi, Psi' >= Psi/6, Psi' < Psi/6, PEFT.
TABLE1 = {
    "NNN": (1, 1, 1, 1), "NNI": (1, 1, 1, 1), "NNG": (1, 1, 1, 0), "NII": (1, 1, 1, 0),
    "NIG": (1, 1, 1, 0), "NGG": (1, 1, 1, 0), "INI": (0, 0, 0, 1), "ING": (0, 1, 1, 0),
    "III": (0, 0, 1, 0), "IIG": (1, 1, 0, 0), "IGG": (1, 1, 1, 0), "GNG": (0, 1, 1, 1),
    "GIG": (0, 1, 1, 0), "GGG": (1, 1, 1, 0),
}


def pad(x, N):
    unit = N * 64
    return -(-int(x) // unit) * unit


def table1_column(psi, psi_trainable, peft=False):
    """Table 1 column of a training task (P:267 caption, R29)."""
    if peft:
        return 3
    if psi_trainable == psi:
        return 0
    return 1 if 6 * psi_trainable >= psi else 2


def memory_bytes(code, N, M, psi, psi_trainable):
    """Model-state bytes per GPU: 2Psi/div(P) + 2Psi'/div(G) + 12Psi'/div(OS) (Table 2)."""
    p, g, o = validate(code)
    return (2 * pad(psi, N) // divisor(p, N, M) + 2 * pad(psi_trainable, N) // divisor(g, N, M)
            + K_ADAM * pad(psi_trainable, N) // divisor(o, N, M))


def param_gather_units(code, N, M, psi):
    """One forward (or backward) parameter all-gather, per rank (Table 3 A-G(P) columns)."""
    p, _, _ = validate(code)
    if p == "N":
        return Fr(0), Fr(0)
    return primitive_units("AG_I" if p == "I" else "HO_AG", N, M, psi)


def minibatch_units_per_rank(code, N, M, psi, psi_trainable, s):
    """(intra, inter) parameter units one rank sends in a mini-batch of s micro-batches."""
    fa, fe = param_gather_units(code, N, M, pad(psi, N))
    ga, ge = accum_units_per_rank(code, N, M, pad(psi_trainable, N), s)
    return 2 * s * fa + ga, 2 * s * fe + ge


def advise(N, M, psi, psi_trainable, s, mem_budget_bytes, bw_intra_gbs, bw_inter_gbs, peft=False):
    """Every PaRO strategy with its Table 1 mark, memory, volume and modeled time, ranked (R29).

    Returns a list of dicts {code, recommended, fits, mem_bytes, intra_bytes,
    inter_bytes, t_s}, best first.
    """
    col = table1_column(psi, psi_trainable, peft)
    rows = []
    for code in paro_strategies():
        ia, ie = minibatch_units_per_rank(code, N, M, psi, psi_trainable, s)
        assert ia.denominator == 1 and ie.denominator == 1
        intra, inter = 2 * int(ia), 2 * int(ie)
        mem = memory_bytes(code, N, M, psi, psi_trainable)
        t = intra / (bw_intra_gbs * 1e9) + inter / (bw_inter_gbs * 1e9)
        rows.append({"code": code, "recommended": bool(TABLE1[code][col]), "fits": mem <= mem_budget_bytes,
                     "mem_bytes": mem, "intra_bytes": intra, "inter_bytes": inter, "t_s": t})
    rows.sort(key=lambda r: (not (r["recommended"] and r["fits"]), r["t_s"], r["mem_bytes"], r["code"]))
    return rows
