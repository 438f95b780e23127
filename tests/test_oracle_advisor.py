"""Pins of the strategy advisor (oracle/advisor.py, NEXT-4, reading R29)
against what the paper fixes: Table 1, Table 2 rows, Table 3 per-stage
volumes, and the outcomes of the paper's experiments."""
import json
import os
from fractions import Fraction as Fr

import pytest

from oracle import accounting as A
from oracle import advisor as AD
from oracle import strategy as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

NAMED = {"NNG": "ZeRO-1", "NGG": "ZeRO-2", "GGG": "ZeRO-3", "III": "MiCS", "IGG": "PaRO-IGG",
         "IIG": "PaRO-IIG", "NIG": "PaRO-NIG"}


def test_table1_transcription_matches_golden():
    rows = json.load(open(os.path.join(GOLDEN, "table1.json")))["rows"]
    assert {k: tuple(v) for k, v in rows.items()} == AD.TABLE1
    assert sorted(AD.TABLE1) == sorted(S.paro_strategies())


def test_table1_column_selection():
    psi = 6_000_000
    assert AD.table1_column(psi, psi) == 0
    assert AD.table1_column(psi, psi // 6) == 1          # Psi' = Psi/6 is ">= Psi/6"
    assert AD.table1_column(psi, psi // 6 - 1) == 2
    assert AD.table1_column(psi, 10, peft=True) == 3


def test_peft_column_obeys_principle_3():
    """P:254-256 Principle 3: G is not sharded in PEFT -> every PEFT-recommended code has G = N."""
    for code, marks in AD.TABLE1.items():
        if marks[3]:
            assert code[1] == "N", code


@pytest.mark.parametrize("N,M", [(64, 8), (32, 8), (128, 8), (8, 4)])
def test_memory_equals_table2_rows(N, M):
    psi = N * 64 * 1000
    for code, name in NAMED.items():
        assert AD.memory_bytes(code, N, M, psi, psi) == sum(A.memory_named(name, N, M, psi)), code


@pytest.mark.parametrize("s", [1, 4, 8, 10])
@pytest.mark.parametrize("N,M", [(64, 8), (32, 8), (16, 4), (8, 2)])
def test_minibatch_volumes_equal_table3(N, M, s):
    """Per rank = Table 3 cluster total / N (readings R11-R13 applied).  The
    PaRO rows and MiCS match intra and inter exactly; ZeRO-2/3 use a flat ring
    in Table 3 and the HO-Ring here: same total, different intra/inter split."""
    psi = N * 64 * 997
    for code in ("IGG", "IIG", "NIG", "III"):
        a, e = A.table3_totals(NAMED[code], N, M, s, psi, corrected=True)
        assert AD.minibatch_units_per_rank(code, N, M, psi, psi, s) == (a / N, e / N), code
    for code in ("NGG", "GGG"):
        a, e = A.table3_totals(NAMED[code], N, M, s, psi, corrected=True)
        x, y = AD.minibatch_units_per_rank(code, N, M, psi, psi, s)
        assert x + y == (a + e) / N, code
        assert y < e / N          # the hierarchical rings send less across groups


def test_fig5_ordering_of_inter_volume():
    """P:546-548 at Psi = 7B, N = 64, s = 8, g = 8: inter-group volume of
    PaRO-IIG is the lowest of ZeRO-3 / IGG / IIG, and IGG's is below ZeRO-3's."""
    v = {c: AD.minibatch_units_per_rank(c, 64, 8, 7_000_000_000, 7_000_000_000, 8)[1] for c in ("GGG", "IGG", "IIG")}
    assert v["IIG"] < v["IGG"] < v["GGG"]


A100 = dict(bw_intra_gbs=300.0, bw_inter_gbs=100.0 / 8)   # 600 GB/s bidirectional NVLink,
                                                          # > 100 GB/s IB per 8-GPU node


@pytest.mark.parametrize("N", [32, 128])
def test_llama65b_feasible_set_and_order(N):
    """LLaMA-65B on 80 GB A100s, M = 8: only ZeRO-3, ZeRO++, IGG and
    IIG train (MiCS, ZeRO-2, NIG OOM), and IIG > IGG > ZeRO-3 in throughput."""
    psi = 65_285_660_672    # LLaMA-65B
    rows = {r["code"]: r for r in AD.advise(N, 8, psi, psi, 10, 80e9, **A100)}
    for code in ("GGG", "IGG", "IIG"):
        assert rows[code]["fits"], code
    for code in ("III", "NIG", "NGG", "NNG", "NNN"):
        assert not rows[code]["fits"], code
    assert rows["IIG"]["t_s"] < rows["IGG"]["t_s"] < rows["GGG"]["t_s"]


@pytest.mark.parametrize("N", [32, 128])
def test_llama7b_order(N):
    """LLaMA-7B, batch 40 in 4 micro-batches x 10 accumulation
    steps: IIG > IGG > ZeRO-3 and NIG > ZeRO-2; NIG is the fastest of them."""
    psi = 6_738_415_616
    rows = {r["code"]: r for r in AD.advise(N, 8, psi, psi, 10, 80e9, **A100)}
    t = {c: rows[c]["t_s"] for c in ("GGG", "IGG", "IIG", "NIG", "NGG")}
    assert t["IIG"] < t["IGG"] < t["GGG"]
    assert t["NIG"] < t["NGG"]
    assert t["NIG"] == min(t.values())


def test_ranking_is_recommended_and_fitting_first():
    psi = 8 * 64 * 100_000
    rows = AD.advise(8, 4, psi, psi // 10, 4, 40e6, 770.0, 770.0 / 6)
    flags = [r["recommended"] and r["fits"] for r in rows]
    assert flags == sorted(flags, reverse=True)
    k = sum(flags)
    assert k > 0
    ts = [r["t_s"] for r in rows[:k]]
    assert ts == sorted(ts)
    # Psi' < Psi/6: column 2 of Table 1 (IIG and INI not recommended, III is)
    rec = {r["code"] for r in rows if r["recommended"]}
    assert "III" in rec and "IIG" not in rec and "INI" not in rec


def test_peft_memory_is_dominated_by_parameters():
    """with Psi' << Psi the parameters take the most memory."""
    psi, pt = 8 * 64 * 1_000_000, 8 * 64 * 1000
    for code in S.paro_strategies():
        p, g, o = code
        mem_p = 2 * psi // (1 if p == "N" else (4 if p == "I" else 8))
        assert AD.memory_bytes(code, 8, 4, psi, pt) - mem_p < mem_p, code


def test_volumes_are_integral_after_padding():
    for code in S.paro_strategies():
        a, e = AD.minibatch_units_per_rank(code, 12, 3, 1_000_003, 77_777, 3)
        assert isinstance(a, Fr) and a.denominator == 1 and e.denominator == 1
