"""paro_advise (C ABI, host only) against the oracle advisor and against the
bytes counted from the library's own plans (NEXT-4, reading R29)."""
import numpy as np
import pytest

from oracle import advisor as AD
from oracle import strategy as S
from paper_2310_06003_b200 import paro


@pytest.mark.parametrize("seed", range(6))
def test_advise_equals_oracle(seed):
    rng = np.random.default_rng(seed)
    for _ in range(40):
        M = int(rng.choice([1, 2, 4, 8, 3]))
        g = int(rng.choice([1, 2, 4, 16]))
        N = M * g
        psi = int(rng.integers(1, 10**11))
        pt = psi if rng.random() < 0.3 else int(rng.integers(1, psi + 1))
        s = int(rng.integers(1, 17))
        args = (N, M, psi, pt, s, float(rng.uniform(1e6, 2e11)), float(rng.uniform(50, 900)),
                float(rng.uniform(5, 900)), bool(rng.random() < 0.2))
        assert paro.advise(*args) == AD.advise(*args), args


@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (4, 2), (8, 1), (8, 8), (6, 3)])
def test_advise_volumes_equal_counted_plan_bytes(N, M):
    """The advisor's closed forms are what the kernels send: s x (bytes per
    paro_accumulate) + (bytes of the step after it) + 2 s x (bytes of one
    gather of every bucket through the parameter windows), per rank."""
    psi = N * 64 * 40 + 5
    pt = N * 64 * 12 + 3
    s = 3
    rows = {r["code"]: r for r in paro.advise(N, M, psi, pt, s, 1e12, 100.0, 10.0)}
    ctx = paro.Context(N, M)
    for code in S.paro_strategies():
        pg = paro.Plan(ctx, code, [pt], bucket_elems=N * 64 * 4, grad_accum=True)
        pw = paro.Plan(ctx, code, [psi], bucket_elems=N * 64 * 8, gather_windows=1)
        for r in range(N):
            (ai, ae), (si, se) = pg.accum_send_bytes(r)
            wi, we = pw.gather_send_bytes(r) if code[0] != "N" else (0, 0)
            assert (s * ai + si + 2 * s * wi, s * ae + se + 2 * s * we) == \
                (rows[code]["intra_bytes"], rows[code]["inter_bytes"]), (code, r)
        info_g, info_w = pg.info(), pw.info()
        assert rows[code]["mem_bytes"] == info_w["mem_p_bytes"] + info_g["mem_g_bytes"] + info_g["mem_os_bytes"]
        pg.close()
        pw.close()
    ctx.close()


def test_advise_rejects_bad_input():
    with pytest.raises(paro.ParoError):
        paro.advise(8, 3, 100, 100, 1, 1e9, 1.0, 1.0)
    with pytest.raises(paro.ParoError):
        paro.advise(8, 4, 100, 200, 1, 1e9, 1.0, 1.0)
    with pytest.raises(paro.ParoError):
        paro.advise(8, 4, 100, 100, 0, 1e9, 1.0, 1.0)
    with pytest.raises(paro.ParoError):
        paro.advise(8, 4, 100, 100, 1, 1e9, 0.0, 1.0)


def test_table1_column():
    assert paro.paro_table1_column(600, 600, 0) == 0
    assert paro.paro_table1_column(600, 100, 0) == 1
    assert paro.paro_table1_column(600, 99, 0) == 2
    assert paro.paro_table1_column(600, 600, 1) == 3
