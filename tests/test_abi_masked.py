"""Partial / PEFT training plans (paro_plan_masked, NEXT-4) on a planning-only
context: memory and bytes against the paper's closed forms with Psi' < Psi
("2Psi, 2Psi', 12Psi'"; Table 3 volumes over Psi' for the
update, over Psi for the forward/backward parameter gathers)."""
import pytest

from oracle import accounting as A
from oracle import advisor as AD
from oracle import strategy as S
from paper_2310_06003_b200 import paro


@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (4, 2), (8, 1), (8, 8)])
def test_masked_memory_and_bytes(N, M):
    u = N * 64
    sizes = [u * 7, u * 3, u * 20, u, u * 2]        # unpadded lists: Table 2 holds exactly
    mask = [1, 0, 0, 1, 0]
    psi, pt = sum(sizes), u * 8
    ctx = paro.Context(N, M)
    for code in S.paro_strategies():
        tp, fp = paro.Plan.masked(ctx, code, sizes, mask, bucket_elems=u * 4, gather_windows=1)
        it, ifz = tp.info(), fp.info()
        assert it["psi"] == pt and ifz["psi"] == psi - pt
        mem = it["mem_p_bytes"] + ifz["mem_p_bytes"] + it["mem_g_bytes"] + it["mem_os_bytes"]
        assert (ifz["mem_g_bytes"], ifz["mem_os_bytes"], ifz["os_numel"], ifz["g_numel"]) == (0, 0, 0, 0)
        assert mem == AD.memory_bytes(code, N, M, psi, pt) == sum(A.memory_strategy(code, N, M, psi, pt))
        a, e = A.step_units_per_rank(code, N, M, pt)
        fa, fe = AD.param_gather_units(code, N, M, psi)
        for r in range(N):
            assert tp.send_bytes(r) == (2 * a, 2 * e), code      # the update runs on Psi' only
            assert fp.send_bytes(r) == (0, 0), code               # frozen tensors never sync
            if code[0] != "N":
                wt, wf = tp.gather_send_bytes(r), fp.gather_send_bytes(r)
                assert (wt[0] + wf[0], wt[1] + wf[1]) == (2 * fa, 2 * fe), code
        fp.close()
        tp.close()
    ctx.close()


def test_masked_all_trainable_gives_no_frozen_plan():
    ctx = paro.Context(4, 2)
    tp, fp = paro.Plan.masked(ctx, "IIG", [4 * 64 * 3, 100], [1, 1])
    assert fp is None and tp.info()["psi"] == 4 * 64 * 3 + 100
    tp.close()
    with pytest.raises(paro.ParoError):
        paro.Plan.masked(ctx, "IIG", [10, 20], [0, 0])
    ctx.close()


def test_frozen_plan_rejects_step_calls_on_planner_ctx():
    ctx = paro.Context(4, 2)
    fp = paro.Plan(ctx, "GGG", [4 * 64 * 3], frozen=True)
    info = fp.info()
    assert info["p_numel"] == 4 * 64 * 3 // 4 and info["os_numel"] == 0 and info["n_comm_launches"] == 0
    with pytest.raises(paro.ParoError):
        fp.step([[0, 0, 0]], 1e-3, 1)
    fp.close()
    ctx.close()


# --------------------------------------------------------------------- streamed gradients (grad_slots)
@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (1, 1)])
def test_grad_slots_shrink_the_gradient_buffer_only(N, M):
    """grad_slots = K keeps K bucket slots of raw gradients (2 K B bytes)
    instead of the 2 psi_pad flat buffer; shard map, bytes and Table 2
    accounting are unchanged."""
    u = N * 64
    sizes = [u * 37 + 5, 999, u * 11]
    B = u * 4
    ctx = paro.Context(N, M)
    for code in S.paro_strategies():
        a = paro.Plan(ctx, code, sizes, bucket_elems=B)
        for K in (1, 2, 3):
            b = paro.Plan(ctx, code, sizes, bucket_elems=B, grad_slots=K)
            ia, ib = a.info(), b.info()
            assert ia["grad_buffer_bytes"] == 2 * ia["psi_pad"]
            assert ib["grad_buffer_bytes"] == 2 * min(ia["psi_pad"], K * ib["bucket_elems"])
            for k in ("psi_pad", "p_numel", "g_numel", "os_numel", "mem_p_bytes", "mem_g_bytes", "mem_os_bytes",
                      "step_send_bytes_intra", "step_send_bytes_inter", "n_rounds", "n_comm_launches"):
                assert ia[k] == ib[k], (code, K, k)
            for r in range(N):
                assert a.send_bytes(r) == b.send_bytes(r)
            b.close()
        a.close()
    with pytest.raises(paro.ParoError):
        paro.Plan(ctx, "IIG", sizes, grad_slots=2, grad_accum=True)
    with pytest.raises(paro.ParoError):
        paro.Plan(ctx, "IIG", sizes, grad_slots=-1)
    ctx.close()
    one = paro.Context(1, 1)     # N = 1 two-phase updates from the raw gradients: all must stay resident
    with pytest.raises(paro.ParoError, match="two-phase"):
        paro.Plan(one, "NNN", sizes, bucket_elems=64 * 4, grad_slots=2, clip_norm=1.0)
    paro.Plan(one, "NNN", sizes, bucket_elems=64 * 4, grad_slots=1000, clip_norm=1.0).close()
    one.close()
