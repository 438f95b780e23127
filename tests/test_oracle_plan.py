"""Pins for oracle/strategy.py, oracle/layout.py and oracle/accounting.py (CPU).

Strategy set: Table 1 and "27 ... 14".
Shard map: brute force — index-tagged integer payloads pushed through the
round simulators land exactly where the closed-form map says.
Accounting: paper/SPEC worked numbers (tests/golden/cost_examples.json),
Eq. 1's own term-by-term form, Fig 5 orderings, and the
simulator's counted bytes.
"""
import json
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

from oracle import accounting as A
from oracle import collectives as C
from oracle import layout as L
from oracle import strategy as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- strategy
def test_strategy_space_is_table1():
    t1 = _gold("table1.json")
    assert len(S.enumerate_all()) == t1["n_combinations"] == 27
    assert S.enumerate_all()[0] == "NNN" and S.enumerate_all()[-1] == "GGG"
    assert sorted(S.paro_strategies()) == sorted(t1["rows"].keys())
    assert len(S.paro_strategies()) == 14
    assert S.TABLE1_ROWS == list(t1["rows"].keys())
    for code, marks in t1["rows"].items():
        assert list(S.TABLE1_MATRIX[code]) == marks


def test_strategy_errors():
    with pytest.raises(S.StrategyError, match="invalid shard level 'X' at position 1"):
        S.parse("XGG")
    with pytest.raises(S.StrategyError, match="violates Principle 1"):
        S.validate("GGN")
    with pytest.raises(S.StrategyError, match="group_size must divide n_gpus"):
        S.validate_cluster(9, 4)
    assert S.validate_cluster(64, 8) == (64, 8, 8)


# ----------------------------------------------------------------- layout
DIVISORS = lambda n: [m for m in range(1, n + 1) if n % m == 0]


@pytest.mark.parametrize("N", [1, 2, 3, 4, 6, 8, 9, 12, 16, 32])
def test_shard_map_tiles_and_nests(N):
    for M in DIVISORS(N):
        lay = L.Layout([1000, 37, 4096], N, M, bucket_elems=N * 64 * 3)
        assert lay.psi_pad % (N * 64) == 0 and lay.psi_pad >= lay.psi
        assert sum(n for _, n in lay.buckets) == lay.psi_pad
        for b, (s, n) in enumerate(lay.buckets):
            segs = sorted(lay.residency("G", r, b) for r in range(N))
            assert segs[0][0] == s and segs[-1][1] == s + n
            assert all(segs[i][1] == segs[i + 1][0] for i in range(N - 1))
            for j in range(N // M):
                chunks = sorted(lay.residency("I", lay.rank_of(j, p), b) for p in range(M))
                assert chunks[0][0] == s and chunks[-1][1] == s + n
            for r in range(N):
                a, e = lay.residency("G", r, b)
                ca, ce = lay.residency("I", r, b)
                assert ca <= a < e <= ce          # OS=G shard inside P=I shard (R1)
        for lvl in "NIG":
            for r in range(N):
                assert sum(e - a for a, e in lay.shard_ranges(lvl, r)) == lay.shard_numel(lvl)


@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (9, 3), (6, 2), (12, 3), (4, 1), (4, 4)])
def test_shard_map_bruteforce_index_tagged(N, M):
    """Rank r contributes value (r+1) * 2^20 + i at flat index i; after the HO-Ring RS the
    value at rank r must be the brute-force sum of exactly the indices of its segment."""
    lay = L.Layout([5000], N, M, bucket_elems=N * 64 * 2)
    geo = C.Geometry(N, M)
    for b, (s, n) in enumerate(lay.buckets):
        C_ = n // N
        X = {}
        for r in range(N):
            full = (r + 1) * (1 << 20) + np.arange(s, s + n, dtype=np.int64)
            X[r] = [full[k * C_:(k + 1) * C_] for k in range(N)]
        out, _, _ = C.rs_ho_ring(geo, X, lambda a, c: a + c)
        for r in range(N):
            a, e = lay.residency("G", r, b)
            idx = np.arange(a, e, dtype=np.int64)
            expect = sum((q + 1) * (1 << 20) for q in range(N)) + N * idx
            assert np.array_equal(out[r], expect)
            assert lay.owner_segment(a) == geo.jp(r)


# ----------------------------------------------------------------- accounting
def test_table2_worked_examples():
    for ex in _gold("cost_examples.json")["table2"]:
        P, G, OS = A.memory_named(ex["method"], ex["N"], ex["M"], ex["psi"])
        assert P == ex["P"]
        if "G" in ex:
            assert G == ex["G"] and OS == ex["OS"]


def test_table2_named_rows_equal_generic_strategies():
    for (N, M) in [(64, 8), (16, 4), (8, 2)]:
        psi = 7 * 10**9
        for meth, code in [("ZeRO-1", "NNG"), ("ZeRO-2", "NGG"), ("ZeRO-3", "GGG"),
                           ("MiCS", "III"), ("PaRO-IGG", "IGG"), ("PaRO-IIG", "IIG"),
                           ("PaRO-NIG", "NIG")]:
            assert A.memory_named(meth, N, M, psi) == A.memory_strategy(code, N, M, psi)
        assert A.memory_strategy("NNN", N, M, psi) == (2 * psi, 2 * psi, 12 * psi)


def test_table3_worked_examples():
    for ex in _gold("cost_examples.json")["table3"]:
        t = A.table3(ex["method"], ex["N"], ex["M"], ex["s"], ex["psi"])
        assert t[ex["stage"]] == (ex["intra"], ex["inter"])


def test_eq1_examples_and_identity():
    for ex in _gold("cost_examples.json")["eq1"]:
        assert A.eq1_delta(ex["psi"], ex["N"], ex["M"], ex["s"]) == ex["delta"]
    for (psi, N, M, s) in [(7e9, 64, 8, 8), (64000, 8, 2, 4), (123456, 12, 3, 5), (10**6, 9, 3, 2)]:
        assert A.eq1_lhs(int(psi), N, M, s) == A.eq1_delta(int(psi), N, M, s)


def test_eq1_against_simulator_counted_volumes():
    """Per-GPU (global RS x s) - (intra RS x s + inter RS x 1) counted by the ring
    simulators equals Eq. 1 at the scaled config Psi=64000, N=8, M=2, s=4."""
    psi, N, M, s = 64000, 8, 2, 4
    geo = C.Geometry(N, M)
    Cn = psi // N
    X = {r: [np.zeros(Cn, np.int64) for _ in range(N)] for r in range(N)}
    add = lambda a, b: a + b
    _, tr_flat = C.rs_flat_ring(geo, X, add)
    Y, r_i = C.rs_intra(geo, X, add)
    _, r_e = C.rs_inter(geo, Y, add)
    ti, te = C.Trace(M), C.Trace(M)
    ti.extend(r_i)
    te.extend(r_e)
    for r in range(N):
        glob = sum(tr_flat.sent(r))
        grouped = s * sum(ti.sent(r)) + sum(te.sent(r))
        assert s * glob - grouped == A.eq1_delta(psi, N, M, s) == 72000


def test_fig5_orderings():
    cfg = _gold("cost_examples.json")["fig5_config"]
    N, M, s, psi = cfg["N"], cfg["M"], cfg["s"], cfg["psi"]
    mem = {m: sum(A.memory_named(m, N, M, psi)) for m in A.NAMED_METHODS}
    # MiCS memory significantly above IGG, IIG, ZeRO++; ZeRO-3 the smallest
    assert mem["ZeRO-3"] < mem["PaRO-IGG"] < mem["ZeRO++"] < mem["PaRO-IIG"] < mem["MiCS"]
    inter = {m: A.table3_totals(m, N, M, s, psi, corrected=True)[1] for m in A.NAMED_METHODS}
    grouped_min = min(inter[m] for m in ["MiCS", "PaRO-IGG", "PaRO-IIG", "PaRO-NIG", "ZeRO++"])
    assert inter["MiCS"] == inter["PaRO-IIG"] == inter["PaRO-NIG"] == grouped_min == Fr(98 * 10**9)
    # the literal PaRO-NIG cell (no s, R13) contradicts "increases slightly" vs ZeRO-2
    lit = A.table3_totals("PaRO-NIG", N, M, s, psi)[0]
    cor = A.table3_totals("PaRO-NIG", N, M, s, psi, corrected=True)[0]
    z2 = A.table3_totals("ZeRO-2", N, M, s, psi)[0]
    assert lit < z2 < cor


def test_step_units_match_table3_at_s1():
    """Per-rank s=1 step volumes x N equal Table 3's Backward R-S + Update columns
    for the three PaRO rows the paper prints (readings R12/R13)."""
    for (N, M) in [(64, 8), (8, 2), (16, 4)]:
        psi = 7 * 10**9
        for code, meth in [("IGG", "PaRO-IGG"), ("IIG", "PaRO-IIG"), ("NIG", "PaRO-NIG")]:
            t = A.table3(meth, N, M, 1, psi, corrected=True)
            intra = t["bwd_rs_g"][0] + t["upd_rs_ar_g"][0] + t["upd_ag_p"][0]
            inter = t["bwd_rs_g"][1] + t["upd_rs_ar_g"][1] + t["upd_ag_p"][1]
            a, b = A.step_units_per_rank(code, N, M, psi)
            assert (N * a, N * b) == (intra, inter)


def test_step_units_match_simulator_bytes():
    """The simulator's counted sends for a full strategy step equal the closed form."""
    from oracle import step as ST
    from oracle.numerics import AdamScalars
    from paro_synth import grad_bits, master_f32
    for (N, M) in [(8, 4), (4, 2), (9, 3), (8, 1), (4, 4)]:
        lay = L.Layout([N * 64 * 5], N, M, bucket_elems=N * 64 * 2)
        grads = [grad_bits(r, 1, 0, lay.psi) for r in range(N)]
        w0 = master_f32(0, lay.psi)
        for code in S.paro_strategies():
            res = ST.strategy_step(code, lay, grads, ST.init_state(w0, lay, code),
                                   AdamScalars(1e-3, 1), topology="ho")
            a, b = A.step_units_per_rank(code, N, M, lay.psi_pad)
            for r in range(N):
                assert tuple(res.sent[r]) == (a, b), (code, N, M, r)


def _counted(geo, ops, n_seg):
    """Cluster-total [intra, inter] units of a sequence of (collective, multiplier)
    counted message by message by the round simulators (rank-order rings, A14)."""
    N, M = geo.N, geo.M
    add = lambda a, b: a + b
    X = {r: [np.zeros(n_seg, np.int64) for _ in range(N)] for r in range(N)}
    Z = {r: np.zeros(n_seg, np.int64) for r in range(N)}
    tot = [0, 0]
    for op, mult in ops:
        tr = C.Trace(M)
        if op == "flat_rs":
            tr = C.rs_flat_ring(geo, X, add)[1]
        elif op == "flat_ag":
            tr = C.ag_flat_ring(geo, Z)[1]
        elif op == "intra_ag":      # ZeRO++ secondary partition: a Psi/M block per rank, AG inside the group
            tr.extend(C.ag_intra(geo, {r: np.zeros(n_seg * geo.g, np.int64) for r in range(N)})[1])
        else:
            raise ValueError(op)
        a, b = tr.totals()
        tot[0] += mult * a
        tot[1] += mult * b
    return tuple(tot)


@pytest.mark.parametrize("N,M,s", [(8, 2, 1), (8, 4, 3), (12, 3, 2), (16, 4, 4)])
def test_table3_zero_rows_equal_flat_ring_simulator(N, M, s):
    """Table 3's ZeRO-1 / ZeRO-2 / ZeRO-3 / ZeRO++ cells are flat-world
    rings; with rank-order rings (reading A14: rank r = jM + p sends to r + 1, an
    inter link iff r mod M = M - 1) the simulators' counted messages give every
    cell exactly, intra and inter separately, per stage.  ZeRO-1's update
    all-reduce is a flat RS + flat AG; ZeRO++'s backward A-G(P)
    gathers its secondary (intra-group) partition."""
    geo = C.Geometry(N, M)
    n_seg = 64 * 5
    psi = N * n_seg
    plans = {
        "ZeRO-1": {"upd_rs_ar_g": [("flat_rs", 1), ("flat_ag", 1)], "upd_ag_p": [("flat_ag", 1)]},
        "ZeRO-2": {"bwd_rs_g": [("flat_rs", s)], "upd_ag_p": [("flat_ag", 1)]},
        "ZeRO-3": {"fwd_ag_p": [("flat_ag", s)], "bwd_ag_p": [("flat_ag", s)], "bwd_rs_g": [("flat_rs", s)]},
        "ZeRO++": {"fwd_ag_p": [("flat_ag", s)], "bwd_ag_p": [("intra_ag", s)], "bwd_rs_g": [("flat_rs", s)]},
    }
    for meth, stages in plans.items():
        t = A.table3(meth, N, M, s, psi)
        for stage in A.STAGES:
            want = t[stage]
            got = _counted(geo, stages.get(stage, []), n_seg)
            assert (Fr(got[0]), Fr(got[1])) == want, (meth, stage, got, want)
