"""Pins for oracle/collectives.py (CPU): brute force on integer payloads, byte
and round closed forms, HO-RS == two-step bitwise, degenerate splits (S:416-419,
S:383)."""
import numpy as np
import pytest

from oracle import collectives as C
from oracle import numerics as nm

NS = [2, 4, 6, 8, 9, 12, 16, 32]
ADD = lambda a, b: a + b


def _splits():
    for N in NS:
        for M in range(1, N + 1):
            if N % M == 0:
                yield N, M


def _payload(N, Cn, seed):
    rng = np.random.default_rng(seed)
    return {r: [rng.integers(-1000, 1000, Cn).astype(np.int64) for _ in range(N)] for r in range(N)}


@pytest.mark.parametrize("N,M", list(_splits()))
def test_reduce_scatter_variants_equal_bruteforce(N, M):
    geo = C.Geometry(N, M)
    Cn = 3
    X = _payload(N, Cn, N * 100 + M)
    total = [sum(X[r][k] for r in range(N)) for k in range(N)]
    outs = [C.rs_flat_ring(geo, X, ADD)[0], C.rs_two_step(geo, X, ADD)[0],
            C.rs_ho_ring(geo, X, ADD)[0], C.rs_canonical(geo, X, ADD)]
    for out in outs:
        for r in range(N):
            assert np.array_equal(out[r], total[geo.seg(*geo.jp(r))])


@pytest.mark.parametrize("N,M", list(_splits()))
def test_all_gather_variants_complete(N, M):
    geo = C.Geometry(N, M)
    Z = {r: np.array([r * 10 + 1, r * 10 + 2]) for r in range(N)}
    expect = {geo.seg(*geo.jp(r)): Z[r] for r in range(N)}
    for fn in (C.ag_flat_ring, C.ag_two_step, C.ag_ho_ring, C.ag_h_ring):
        have, tr = fn(geo, Z)
        for r in range(N):
            assert set(have[r].keys()) == set(range(N))
            for k in range(N):
                assert np.array_equal(have[r][k], expect[k])


@pytest.mark.parametrize("N,M", list(_splits()))
def test_bytes_and_rounds_closed_forms(N, M):
    geo = C.Geometry(N, M)
    g = N // M
    Cn = 2
    Z = {r: np.zeros(Cn) for r in range(N)}
    X = {r: [np.zeros(Cn, np.int64) for _ in range(N)] for r in range(N)}
    # flat ring AG / RS: (N-1)C per rank
    _, tr = C.ag_flat_ring(geo, Z)
    assert all(sum(tr.sent(r)) == (N - 1) * Cn for r in range(N))
    assert tr.n_rounds() == N - 1
    # HO-Ring AG and RS: per rank [(M-1) g C, (g-1) C]; rounds max(M-1,g-1)+(M-1)[g>1]
    _, tr = C.ag_ho_ring(geo, Z)
    _, tr2, _ = C.rs_ho_ring(geo, X, ADD)
    for t in (tr, tr2):
        for r in range(N):
            assert t.sent(r) == [(M - 1) * g * Cn, (g - 1) * Cn]
        assert t.n_rounds() == C.ho_rounds(N, M)
        tot = t.totals()
        assert sum(tot) == N * (N - 1) * Cn          # conservation of sent units
    # H-Ring: leader inter share (g-1) M C, non-leaders 0
    _, th = C.ag_h_ring(geo, Z)
    for r in range(N):
        j, p = geo.jp(r)
        assert th.sent(r)[1] == ((g - 1) * M * Cn if p == 0 else 0)


def test_fig4_round_structure():
    # N=9, g=3: 2 overlapped rounds + 2 completion rounds
    assert C.ho_rounds(9, 3) == 4
    geo = C.Geometry(9, 3)
    _, tr = C.ag_ho_ring(geo, {r: np.zeros(1) for r in range(9)})
    assert tr.n_rounds() == 4
    assert all(len(tr.rounds[t]) == 9 + 9 for t in range(2))   # intra and inter rings concurrent
    assert all(len(tr.rounds[t]) == 9 for t in range(2, 4))


def test_degenerate_splits_equal_flat_ring():
    rng = np.random.default_rng(7)
    for N, M in [(8, 1), (8, 8), (4, 4), (4, 1)]:
        geo = C.Geometry(N, M)
        X = {r: [nm.bf16_bits_from_f32((rng.standard_normal(16) * 1e-3).astype(np.float32))
                 for _ in range(N)] for r in range(N)}
        a, tra = C.rs_flat_ring(geo, X, nm.hop)
        b, trb, _ = C.rs_ho_ring(geo, X, nm.hop)
        for r in range(N):
            assert np.array_equal(a[r], b[r])
        assert tra.n_rounds() == trb.n_rounds() == N - 1


@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (9, 3), (4, 2), (16, 4), (12, 2)])
def test_ho_rs_equals_two_step_bitwise_and_flat_differs(N, M):
    rng = np.random.default_rng(N * 7 + M)
    geo = C.Geometry(N, M)
    X = {r: [nm.bf16_bits_from_f32((rng.standard_normal(64) * 1e-3).astype(np.float32))
             for _ in range(N)] for r in range(N)}
    ho, _, _ = C.rs_ho_ring(geo, X, nm.hop)
    ts, _, _ = C.rs_two_step(geo, X, nm.hop)
    can = C.rs_canonical(geo, X, nm.hop)
    fl, _ = C.rs_flat_ring(geo, X, nm.hop)
    diff = 0
    for r in range(N):
        assert np.array_equal(ho[r], ts[r]) and np.array_equal(ho[r], can[r])
        diff += int(np.sum(ho[r] != fl[r]))
    assert diff > 0      # the flat ring's order is a different (valid) order when g, M > 1
