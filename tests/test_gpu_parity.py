"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Emulated mode runs all N ranks of a split on one B200 (each collective round
is one kernel over every rank's buffers), so any (N, M) is checked bit for bit.
Bar (BASELINE.json north_star): shard maps / bytes exact; fp32
masters, m, v and bf16 params bit-exact (the 1e-5 relative / 1-ulp fallback
is never needed); NaN compared by isnan; grad norm rel 1e-12.
"""
import numpy as np
import pytest
import torch

from oracle import layout as L
from oracle import numerics as nm
from oracle import step as ST
from oracle import strategy as S
from paro_synth import SEED, edge_grad_bits, grad_bits, master_f32, ragged_param_sizes

from devmem import d2h, h2d

pytestmark = pytest.mark.gpu

LR = 3e-4


def _paro():
    from paper_2310_06003_b200 import paro
    return paro


class EmuRun:
    """All ranks of one split on cuda:0 through the C ABI."""

    def __init__(self, N, M, code, sizes, B, topo="ho", depth=2, wd=0.0, loss_scale=1.0, transport="push",
                 adam_impl="auto", comm_impl="tma_store", grad_accum=False, mode="emulated", clip_norm=0.0,
                 skip_nonfinite=False, fuse_gather="auto", copy_engine=False, fuse_allreduce=True,
                 adam_smem_kb=0, wire="bf16", predivide=True):
        paro = _paro()
        if mode == "emulated":
            self.ctx = paro.Context(N, M, mode="emulated", device=0)
        else:   # one real rank (N = 1): the bench's launch configuration
            self.ctx = paro.Context(1, 1, mode="real", rank=0, device=0, uid=paro.unique_id())
        self.pl = paro.Plan(self.ctx, code, sizes, bucket_elems=B, topology=topo, pipeline_depth=depth,
                            weight_decay=wd, loss_scale=loss_scale, transport=transport, adam_impl=adam_impl,
                            comm_impl=comm_impl, grad_accum=grad_accum, clip_norm=clip_norm,
                            skip_nonfinite=skip_nonfinite, fuse_gather=fuse_gather, copy_engine=copy_engine,
                            fuse_allreduce=fuse_allreduce, adam_smem_kb=adam_smem_kb, wire_dtype=wire,
                            predivide=predivide)
        self.info = self.pl.info()
        self.N, self.code, self.sizes = N, code, sizes
        n = self.info["os_numel"]
        self.st = [tuple(torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(3)) for _ in range(N)]
        for r in range(N):
            self.pl.opt_state_init(r, [t.data_ptr() for t in self.st[r]], seed=SEED)

    def ptrs(self):
        return [[t.data_ptr() for t in s] for s in self.st]

    def set_grads(self, t, kind="synth"):
        for r in range(self.N):
            if kind == "synth":
                self.pl.synth_grads(r, SEED, t)
            else:
                g = np.zeros(self.info["psi_pad"], np.uint16)
                g[:self.info["psi"]] = edge_grad_bits(kind, self.info["psi"], rank=r, step=t)
                h2d(self.pl.buffer(r, 0), g)

    def step(self, t, **kw):
        self.pl.step(self.ptrs(), LR, t, **kw)
        return self.pl.stats()

    def state(self, r):
        torch.cuda.synchronize()
        out = {k: self.st[r][i].cpu().numpy() for i, k in enumerate(("master", "m", "v"))}
        out["param"] = d2h(self.pl.buffer(r, 1), self.info["p_numel"], np.uint16)
        return out

    def close(self):
        self.pl.close()
        self.ctx.close()


def _oracle_grads(N, psi, t, kind="synth"):
    if kind == "synth":
        return [grad_bits(r, t, 0, psi) for r in range(N)]
    return [edge_grad_bits(kind, psi, rank=r, step=t) for r in range(N)]


def _assert_same(got, ref, what):
    if ref.dtype == np.uint16:
        gf, rf = nm.f32_from_bf16_bits(got), nm.f32_from_bf16_bits(ref)
    else:
        gf, rf = got, ref
    nan_g, nan_r = np.isnan(gf), np.isnan(rf)
    assert np.array_equal(nan_g, nan_r), f"{what}: NaN pattern differs"
    ok = ~nan_r
    bad = np.nonzero(gf[ok] != rf[ok])[0]
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first at {bad[0]}: {gf[ok][bad[0]]} vs {rf[ok][bad[0]]}"


def _dp_reference(lay, steps, kind="synth", wd=0.0, loss_scale=1.0, wire="bf16", predivide=True):
    w0 = master_f32(0, lay.psi)
    w = ST.pad_flat(w0, lay.psi_pad, np.float32)
    m, v = np.zeros_like(w), np.zeros_like(w)
    norms = []
    for t in range(1, steps + 1):
        sc = nm.AdamScalars(LR, t, weight_decay=wd, loss_scale=loss_scale, post_div=1 if predivide else lay.N)
        w, m, v, p, gh = ST.dp_step(lay, _oracle_grads(lay.N, lay.psi, t, kind), w, m, v, sc, wire=wire,
                                    predivide=predivide)
        norms.append(nm.grad_sq_sum(gh, sc.s_g))
    return w, m, v, p, norms


def _check_against_dp(run, lay, ref):
    w, m, v, p, _ = ref
    pl_, _, ol = run.code
    for r in range(lay.N):
        st = run.state(r)
        _assert_same(st["master"], ST.shard_of(w, lay, ol, r), f"rank {r} master")
        _assert_same(st["m"], ST.shard_of(m, lay, ol, r), f"rank {r} m")
        _assert_same(st["v"], ST.shard_of(v, lay, ol, r), f"rank {r} v")
        _assert_same(st["param"], ST.shard_of(p, lay, pl_, r), f"rank {r} param")


# --------------------------------------------------------------------- generator
def test_synth_generator_matches_host():
    run = EmuRun(1, 1, "NNN", [100_003], 1 << 16)
    run.set_grads(3)
    g = d2h(run.pl.buffer(0, 0), run.info["psi_pad"], np.uint16)
    assert np.array_equal(g[:100_003], grad_bits(0, 3, 0, 100_003))
    assert not g[100_003:].any()
    st = run.state(0)
    assert np.array_equal(st["master"][:100_003], master_f32(0, 100_003))
    assert np.array_equal(st["param"][:100_003], nm.bf16_bits_from_f32(master_f32(0, 100_003)))
    run.close()


# --------------------------------------------------------------------- N = 1
@pytest.mark.parametrize("adam_impl", ["auto", "lsu", "tma_store"])
@pytest.mark.parametrize("wd,ls", [(0.0, 1.0), (0.1, 4.0)])
def test_n1_ten_steps_bit_exact(wd, ls, adam_impl):
    sizes = [50_000, 4096, 12_345, 3 * 4096 * 148 + 8]   # > one tile per CTA, ragged tail
    lay = L.Layout(sizes, 1, 1, 1 << 14)
    run = EmuRun(1, 1, "NNN", sizes, 1 << 14, wd=wd, loss_scale=ls, adam_impl=adam_impl)
    ref = _dp_reference(lay, 10, wd=wd, loss_scale=ls)
    for t in range(1, 11):
        run.set_grads(t)
        stats = run.step(t)
        assert abs(stats["grad_norm"] ** 2 - ref[4][t - 1]) <= 1e-12 * ref[4][t - 1]
    _check_against_dp(run, lay, ref)
    run.close()


# --------------------------------------------------------------------- all strategies
CONFIG_4M = dict(sizes=[1 << 22], B=1 << 18)   # BASELINE config 1: 2^22 params, 16 buckets


@pytest.mark.parametrize("comm_impl", ["tma", "lsu", "tma_store"])
@pytest.mark.parametrize("transport", ["push", "pull"])
@pytest.mark.parametrize("topo", ["ho", "two_step", "direct", "h_ring"])
def test_4m_2x4_every_strategy_one_step(topo, transport, comm_impl):
    N, M = 8, 4
    lay = L.Layout(CONFIG_4M["sizes"], N, M, CONFIG_4M["B"])
    ref = _dp_reference(lay, 1)
    for code in S.paro_strategies():
        run = EmuRun(N, M, code, CONFIG_4M["sizes"], CONFIG_4M["B"], topo=topo, transport=transport,
                     comm_impl=comm_impl)
        run.set_grads(1)
        stats = run.step(1)
        assert abs(stats["grad_norm"] ** 2 - ref[4][0]) <= 1e-12 * ref[4][0]
        _check_against_dp(run, lay, ref)
        run.close()


@pytest.mark.parametrize("transport", ["push", "pull"])
@pytest.mark.parametrize("N,M", [(8, 2), (4, 2), (8, 1), (8, 8), (6, 3), (2, 2), (2, 1), (9, 3)])
@pytest.mark.parametrize("topo", ["ho", "two_step", "direct"])
def test_splits_every_strategy_ragged(N, M, topo, transport):
    sizes = ragged_param_sizes() + [N * 64 * 7 + 3]
    B = N * 64 * 3
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 2)
    for code in S.paro_strategies():
        run = EmuRun(N, M, code, sizes, B, topo=topo, transport=transport)
        for t in (1, 2):
            run.set_grads(t)
            run.step(t)
        _check_against_dp(run, lay, ref)
        run.close()


@pytest.mark.parametrize("transport", ["push", "pull"])
def test_flat_ring_matches_oracle_flat_simulation(transport):
    N, M = 8, 4
    sizes = [N * 64 * 20]
    B = N * 64 * 6
    lay = L.Layout(sizes, N, M, B)
    grads = _oracle_grads(N, lay.psi, 1)
    w0 = master_f32(0, lay.psi)
    for code in ("NNN", "NNG", "GGG", "IGG"):
        res = ST.strategy_step(code, lay, grads, ST.init_state(w0, lay, code), nm.AdamScalars(LR, 1),
                               topology="flat")
        run = EmuRun(N, M, code, sizes, B, topo="flat", transport=transport)
        run.set_grads(1)
        run.step(1)
        for r in range(N):
            st = run.state(r)
            for k in ("master", "m", "v", "param"):
                _assert_same(st[k], res.state[r][k], f"{code} rank {r} {k}")
        run.close()


# Adam kernels selected by (adam_impl, adam_smem_kb); emulated "auto" = TMA
# stores.  g_hat inputs per element at 2x4: NNN 1, III 2 (AR_E folded into
# Adam, R31), IIG / GGG 3 (HO-Ring final hop fused).  120 KB is the co-run
# budget real N > 1 steps use; 60 KB forces 2048-element thread-store tiles.
ADAM_CASES = [("auto", 0), ("lsu", 0), ("tma_store", 0), ("tma", 0), ("tma", 120), ("tma_store", 120),
              ("tma", 60), ("tma_ws", 0), ("tma_ws", 120)]


@pytest.mark.parametrize("adam_impl,smem", ADAM_CASES)
@pytest.mark.parametrize("code", ["IIG", "NNN", "III", "GGG"])
def test_4m_2x4_ten_steps(code, adam_impl, smem):
    N, M = 8, 4
    lay = L.Layout(CONFIG_4M["sizes"], N, M, CONFIG_4M["B"])
    ref = _dp_reference(lay, 10)
    run = EmuRun(N, M, code, CONFIG_4M["sizes"], CONFIG_4M["B"], adam_impl=adam_impl, adam_smem_kb=smem)
    for t in range(1, 11):
        run.set_grads(t)
        if t == 10:
            run.pl.profile_start(4096)
        run.step(t)
    prof = run.pl.profile_stop()
    _check_against_dp(run, lay, ref)
    v = _paro().ADAM_VARIANTS[prof["adam_variant"]]
    if adam_impl == "lsu":
        assert v == "adam_kernel"
    elif adam_impl == "tma":
        assert v in ("adam_tma_kernel<false,512>", "adam_tma_kernel<false,256>")
        if smem == 60:
            assert v == "adam_tma_kernel<false,256>"
    elif adam_impl == "tma_ws":   # 4096- or 2048-element tiles, by the stages that fit the budget
        assert v in ("adam_tma_ws_kernel<512>", "adam_tma_ws_kernel<256>")
        if smem == 120:
            assert v == "adam_tma_ws_kernel<256>"
    else:
        assert v.startswith("adam_tma_kernel<true,") or v.startswith("adam_tma_ws_kernel")
    run.close()


def test_adam_variant_selection_covers_corun_kernels():
    """The co-run budget (120 KB) selects the kernels real N > 1 steps run:
    thread stores with 4096-element tiles at 2 stages when they fit, 2048-element
    tiles when two 4096-element stages of a 3-input fused hop do not; TMA stores
    at 2048-element tiles.  Each is bit-exact vs the DP definition."""
    N, M = 8, 4
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 2)
    seen = set()
    for code, impl, kb in (("NNN", "tma", 120), ("IIG", "tma", 120), ("GGG", "tma", 120), ("III", "tma", 120),
                           ("IIG", "tma_store", 120), ("NIG", "tma", 0), ("IIG", "tma_ws", 0), ("GGG", "tma_ws", 120)):
        run = EmuRun(N, M, code, sizes, B, adam_impl=impl, adam_smem_kb=kb, transport="pull")
        run.pl.profile_start(1024)
        for t in (1, 2):
            run.set_grads(t)
            run.step(t)
        prof = run.pl.profile_stop()
        seen.add((_paro().ADAM_VARIANTS[prof["adam_variant"]], prof["adam_stages"]))
        _check_against_dp(run, lay, ref)
        run.close()
    names = {v for v, _ in seen}
    assert {"adam_tma_kernel<false,512>", "adam_tma_kernel<false,256>", "adam_tma_kernel<true,256>"} <= names, seen
    assert ("adam_tma_kernel<false,512>", 2) in seen, seen


@pytest.mark.parametrize("fuse", [True, False])
@pytest.mark.parametrize("topo", ["ho", "two_step", "direct"])
@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (6, 3), (2, 1)])
def test_fused_inter_allreduce_os_i(N, M, topo, fuse):
    """OS = I at g = 2 (R31): AR_E folded into Adam (the peer's intra partial
    pulled beside the own one) gives the ring's bits, 3 steps (g_hat slots of
    G = N reused), ragged, depth 1 and 2."""
    sizes = ragged_param_sizes() + [N * 64 * 7 + 3]
    B = N * 64 * 3
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 3)
    for code in ("III", "NII", "INI", "NNI") + (("NNN",) if M == 1 else ()):
        for adam_impl, depth, kb in (("auto", 1, 0), ("lsu", 2, 0), ("tma", 1, 120)):
            run = EmuRun(N, M, code, sizes, B, topo=topo, depth=depth, transport="pull", adam_impl=adam_impl,
                         fuse_allreduce=fuse, adam_smem_kb=kb)
            for t in (1, 2, 3):
                run.set_grads(t)
                stats = run.step(t)
            assert abs(stats["grad_norm"] ** 2 - ref[4][2]) <= 1e-12 * ref[4][2]
            _check_against_dp(run, lay, ref)
            run.close()


@pytest.mark.parametrize("N,M", [(4, 2), (2, 1)])
@pytest.mark.parametrize("kind", ["specials", "nearmax", "smallint"])
def test_fused_inter_allreduce_edge_inputs(kind, N, M):
    sizes = [N * 64 * 10 + 5]
    B = N * 64 * 4
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 1, kind=kind)
    gh = ST.dp_step(lay, _oracle_grads(N, lay.psi, 1, kind), *ref[:3], nm.AdamScalars(LR, 1))[4]
    expect_nonfinite = int(not np.all(np.isfinite(nm.f32_from_bf16_bits(gh))))
    for code in ("III", "NII", "INI", "NNI", "NNN"):
        run = EmuRun(N, M, code, sizes, B, transport="pull")
        run.set_grads(1, kind=kind)
        stats = run.step(1)
        assert stats["nonfinite"] == expect_nonfinite
        _check_against_dp(run, lay, ref)
        run.close()


@pytest.mark.parametrize("kind", ["zeros", "smallint", "specials", "nearmax"])
def test_edge_inputs(kind):
    N, M = 4, 2
    sizes = [N * 64 * 10 + 5]
    B = N * 64 * 4
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 1, kind=kind)
    gh = ST.dp_step(lay, _oracle_grads(N, lay.psi, 1, kind), *ref[:3], nm.AdamScalars(LR, 1))[4]
    expect_nonfinite = int(not np.all(np.isfinite(nm.f32_from_bf16_bits(gh))))
    if kind == "specials":
        assert expect_nonfinite == 1
    for code in ("NNN", "IIG", "INI", "GGG"):
        run = EmuRun(N, M, code, sizes, B)
        run.set_grads(1, kind=kind)
        stats = run.step(1)
        assert stats["nonfinite"] == expect_nonfinite
        _check_against_dp(run, lay, ref)
        run.close()


def test_pack_and_unpack_paths_and_depth_determinism():
    """Per-parameter gradient pointers (pack) and per-parameter outputs (unpack)
    give the same bits as the zero-copy path; pipeline depth 1 vs 4 identical."""
    N, M = 4, 2
    sizes = [1000, 64, 4096 + 8, 777]
    B = N * 64 * 4
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 1)
    grads = _oracle_grads(N, lay.psi, 1)
    for code in ("NNN", "NIG", "IGG"):
        outs = []
        for depth, use_ptrs in ((1, False), (4, True)):
            run = EmuRun(N, M, code, sizes, B, depth=depth)
            gkeep, gptrs, pkeep, pptrs = [], [], [], []
            for r in range(N):
                for i, s in enumerate(sizes):
                    o = lay.param_offsets[i]
                    tg = torch.from_numpy(grads[r][o:o + s].view(np.int16).copy()).cuda()
                    gkeep.append(tg)
                    gptrs.append(tg.data_ptr())
                if code[0] == "N":
                    for s in sizes:
                        tp = torch.zeros(s, dtype=torch.int16, device="cuda")
                        pkeep.append(tp)
                        pptrs.append(tp.data_ptr())
                else:
                    tp = torch.zeros(run.info["p_numel"], dtype=torch.int16, device="cuda")
                    pkeep.append(tp)
                    pptrs.append(tp.data_ptr())
            if use_ptrs:
                run.step(1, grads=gptrs, params=pptrs)
            else:
                run.set_grads(1)
                run.step(1)
            _check_against_dp(run, lay, ref)
            if use_ptrs:
                torch.cuda.synchronize()
                for r in range(N):
                    st = run.state(r)
                    if code[0] == "N":
                        got = np.concatenate([t.cpu().numpy().view(np.uint16)
                                              for t in pkeep[r * len(sizes):(r + 1) * len(sizes)]])
                        assert np.array_equal(got, st["param"][:lay.psi])
                    else:
                        assert np.array_equal(pkeep[r].cpu().numpy().view(np.uint16), st["param"])
            outs.append([run.state(r)["master"] for r in range(N)])
            run.close()
        for a, b in zip(*outs):
            assert np.array_equal(a, b)



# --------------------------------------------------------------------- gradient accumulation (NEXT-1)
def _mb_id(t, k):
    return (t << 8) | (k + 1)     # synthetic-gradient counter of micro-batch k of step t


def _accum_reference(lay, steps, s, g_level, loss_scale=1.0, wire="bf16"):
    w = ST.pad_flat(master_f32(0, lay.psi), lay.psi_pad, np.float32)
    m, v = np.zeros_like(w), np.zeros_like(w)
    norms = []
    for t in range(1, steps + 1):
        mb = [[grad_bits(r, _mb_id(t, k), 0, lay.psi) for r in range(lay.N)] for k in range(s)]
        sc = nm.AdamScalars(LR, t, loss_scale=loss_scale, accum_steps=s)
        w, m, v, p, gh = ST.dp_accum_step(lay, mb, w, m, v, sc, g_level, wire=wire)
        norms.append(nm.grad_sq_sum(gh, sc.s_g))
    return w, m, v, p, norms


def _run_accum(run, steps, s):
    stats = []
    for t in range(1, steps + 1):
        for k in range(s):
            for r in range(run.N):
                run.pl.synth_grads(r, SEED, _mb_id(t, k))
            run.pl.accumulate()
        stats.append(run.step(t))
    return stats


@pytest.mark.parametrize("topo,transport", [("ho", "pull"), ("ho", "push"), ("two_step", "pull"),
                                            ("direct", "pull"), ("ho", "ce")])
def test_accumulation_every_strategy_2x4(topo, transport):
    """BASELINE config 1 shape (2 groups x 4, 16 buckets) with s = 3 micro-batches,
    two mini-batch steps: every strategy bit-exact vs dp_accum_step (R27)."""
    N, M, s = 8, 4, 3
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    refs = {gl: _accum_reference(lay, 2, s, gl) for gl in "NIG"}
    for code in S.paro_strategies():
        ce = transport == "ce"
        run = EmuRun(N, M, code, sizes, B, topo=topo, transport="pull" if ce else transport, grad_accum=True,
                     copy_engine="all" if ce else False)
        stats = _run_accum(run, 2, s)
        ref = refs[code[1]]
        _check_against_dp(run, lay, ref)
        assert abs(stats[-1]["grad_norm"] ** 2 - ref[4][-1]) <= 1e-12 * ref[4][-1]
        (ai, ae), (si, se) = run.pl.accum_send_bytes(0)
        assert (stats[-1]["sent_intra"], stats[-1]["sent_inter"]) == (si, se)
        run.close()


@pytest.mark.parametrize("N,M", [(8, 2), (8, 1), (8, 8), (9, 3), (2, 1)])
def test_accumulation_splits(N, M):
    s = 2
    sizes = ragged_param_sizes() + [N * 64 * 9]
    B = N * 64 * 4
    lay = L.Layout(sizes, N, M, B)
    refs = {gl: _accum_reference(lay, 1, s, gl) for gl in "NIG"}
    for code in ("NNN", "NIG", "IIG", "IGG", "III", "GGG", "NNI"):
        run = EmuRun(N, M, code, sizes, B, grad_accum=True, transport="pull")
        _run_accum(run, 1, s)
        _check_against_dp(run, lay, refs[code[1]])
        run.close()


def test_accumulation_single_gpu_real_mode():
    """N = 1 in the bench's configuration (one real rank): local accumulation,
    loss scale 4, s = 4, three steps."""
    sizes = [1 << 16, 3 * 4096 + 8, 517]
    B = 1 << 14
    lay = L.Layout(sizes, 1, 1, B)
    ref = _accum_reference(lay, 3, 4, "N", loss_scale=4.0)
    for code in ("IIG", "NNN"):
        run = EmuRun(1, 1, code, sizes, B, grad_accum=True, loss_scale=4.0, mode="real")
        stats = _run_accum(run, 3, 4)
        _check_against_dp(run, lay, ref)
        assert abs(stats[-1]["grad_norm"] ** 2 - ref[4][-1]) <= 1e-12 * ref[4][-1]
        run.close()


def test_accumulation_with_one_micro_batch_is_the_plain_step():
    N, M = 8, 4
    sizes = [N * 64 * 24]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 1)
    for code in ("IIG", "NIG", "GGG", "NNN"):
        run = EmuRun(N, M, code, sizes, B, grad_accum=True, transport="pull")
        run.set_grads(1)
        run.pl.accumulate()
        run.step(1)
        _check_against_dp(run, lay, ref)
        run.close()


def test_step_after_accumulate_rejects_grads():
    run = EmuRun(2, 1, "IIG", [4096], 1024, grad_accum=True)
    run.set_grads(1)
    run.pl.accumulate()
    paro = _paro()
    with pytest.raises(paro.ParoError, match="grads must be NULL"):
        run.pl.step(run.ptrs(), LR, 1, grads=[run.pl.buffer(0, 0)] * 2)
    run.close()
    plain = EmuRun(2, 1, "IIG", [4096], 1024)
    with pytest.raises(paro.ParoError, match="grad_accum"):
        plain.pl.accumulate()
    plain.close()


# --------------------------------------------------------------------- clipping / skip (NEXT-3)
def _clip_reference(lay, steps, clip, skip=False, kind="synth", accum=0):
    w = ST.pad_flat(master_f32(0, lay.psi), lay.psi_pad, np.float32)
    m, v = np.zeros_like(w), np.zeros_like(w)
    out = []
    for t in range(1, steps + 1):
        if accum:
            mb = [[grad_bits(r, _mb_id(t, k), 0, lay.psi) for r in range(lay.N)] for k in range(accum)]
            gh = ST.dp_accum_step(lay, mb, w, m, v, nm.AdamScalars(LR, t, accum_steps=accum), accum_glevel)[4]
            res = ST.clip_update(gh, w, m, v, LR, t, clip, skip, accum, {})
        else:
            res = ST.dp_clip_step(lay, _oracle_grads(lay.N, lay.psi, t, kind), w, m, v, LR, t, clip_norm=clip,
                                  skip_nonfinite=skip)
        w, m, v = res[0], res[1], res[2]
        out.append(res)
    last = out[-1]
    return (w, m, v, last[3], [r[5] for r in out]), out


accum_glevel = "G"


@pytest.mark.parametrize("topo,transport", [("ho", "pull"), ("ho", "push"), ("two_step", "pull")])
def test_clipping_every_strategy_2x4(topo, transport):
    N, M = 8, 4
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    clip = 0.05                       # below the synthetic gradient norm: the coefficient is active
    ref, per = _clip_reference(lay, 3, clip)
    assert all(r[6] < 1.0 for r in per)
    for code in S.paro_strategies():
        run = EmuRun(N, M, code, sizes, B, topo=topo, transport=transport, clip_norm=clip)
        for t in range(1, 4):
            run.set_grads(t)
            st = run.step(t)
            assert abs(st["grad_norm"] ** 2 - per[t - 1][5]) <= 1e-12 * per[t - 1][5]
        _check_against_dp(run, lay, ref)
        run.close()


def test_clipping_single_gpu_real_mode_and_accumulation():
    sizes = [1 << 16, 3 * 4096 + 8]
    B = 1 << 14
    lay = L.Layout(sizes, 1, 1, B)
    ref, per = _clip_reference(lay, 3, 0.02)
    assert per[0][6] < 1.0
    run = EmuRun(1, 1, "NNN", sizes, B, clip_norm=0.02, mode="real")
    for t in range(1, 4):
        run.set_grads(t)
        run.step(t)
    _check_against_dp(run, lay, ref)
    run.close()
    # accumulation + clipping, 2x4 emulated, G = G strategy
    N, M = 8, 4
    sizes = [N * 64 * 24]
    lay = L.Layout(sizes, N, M, N * 64 * 8)
    ref, per = _clip_reference(lay, 2, 0.01, accum=3)
    assert per[0][6] < 1.0
    for code in ("IGG", "GGG"):
        run = EmuRun(N, M, code, sizes, N * 64 * 8, clip_norm=0.01, grad_accum=True, transport="pull")
        _run_accum(run, 2, 3)
        _check_against_dp(run, lay, ref)
        run.close()


def test_nonfinite_skip_leaves_state_unchanged():
    N, M = 8, 2
    sizes = [N * 64 * 30]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    for code in ("NNN", "IIG", "NIG", "GGG"):
        run = EmuRun(N, M, code, sizes, B, skip_nonfinite=True, transport="pull")
        run.set_grads(1)
        run.step(1)
        before = [run.state(r) for r in range(N)]
        run.set_grads(2, kind="specials")
        st = run.step(2)
        assert st["nonfinite"] == 1
        for r in range(N):
            after = run.state(r)
            for k in ("master", "m", "v", "param"):
                assert np.array_equal(after[k], before[r][k]), (code, r, k)
        run.set_grads(3)       # a finite step afterwards updates again: t = 3 over t = 1's state
        run.step(3)
        w = ST.pad_flat(master_f32(0, lay.psi), lay.psi_pad, np.float32)
        z = np.zeros_like(w)
        w1, m1, v1 = ST.dp_step(lay, _oracle_grads(N, lay.psi, 1), w, z, z, nm.AdamScalars(LR, 1))[:3]
        ref = ST.dp_step(lay, _oracle_grads(N, lay.psi, 3), w1, m1, v1, nm.AdamScalars(LR, 3))
        _check_against_dp(run, lay, ref)
        run.close()


# --------------------------------------------------------------------- forward/backward parameter gather (NEXT-2)
@pytest.mark.parametrize("topo,transport", [("ho", "pull"), ("ho", "push"), ("two_step", "pull"),
                                            ("flat", "pull"), ("h_ring", "push")])
def test_gather_windows_return_full_parameters(topo, transport):
    """After a step, gathering every bucket into alternating windows gives each
    rank the bucket slice of the full model's bf16 parameters, bit for bit."""
    N, M = 8, 4
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    p_full = _dp_reference(lay, 1)[3]
    for code in S.paro_strategies():
        run = EmuRun(N, M, code, sizes, B, topo=topo, transport=transport)
        run.pl.close()
        paro = _paro()
        run.pl = paro.Plan(run.ctx, code, sizes, bucket_elems=B, topology=topo, transport=transport,
                           gather_windows=2)
        for r in range(N):
            run.pl.opt_state_init(r, [t.data_ptr() for t in run.st[r]], seed=SEED)
        run.set_grads(1)
        run.step(1)
        # the full model assembled from every rank's parameter residency (bit copies)
        assembled = np.zeros(lay.psi_pad, np.uint16)
        for r in range(N):
            mine = run.state(r)["param"]
            off = 0
            for (a, e) in lay.shard_ranges(code[0], r):
                assembled[a:e] = mine[off:off + e - a]
                off += e - a
        if topo != "flat":               # flat ring: another (deterministic) reduction order
            assert np.array_equal(assembled, p_full), code
        for b in range(len(lay.buckets)):
            s0, n = lay.buckets[b]
            out = run.pl.gather_window(0, b, slot=b % 2)
            for r in range(N):
                if code[0] == "N":
                    ptr = run.pl.buffer(r, 1) + 2 * s0
                else:
                    ptr = run.pl.buffer(r, 5) + 2 * (b % 2) * B
                if r == 0:
                    assert ptr == out
                got = d2h(ptr, n, np.uint16)
                assert np.array_equal(got, assembled[s0:s0 + n]), (code, b, r)
        run.close()



# --------------------------------------------------------------------- fused parameter all-gather
@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (8, 1), (4, 4), (6, 3)])
@pytest.mark.parametrize("transport,adam_impl", [("pull", "auto"), ("push", "lsu"), ("pull", "tma_store")])
def test_fused_gather_every_strategy(N, M, transport, adam_impl):
    """fuse_gather = always: the Adam kernel stores the bf16 parameters into the
    consumers' buffers (AG_E / AG_I / one world ring); bits equal the DP definition
    and the bytes per link class stay those of the ring."""
    sizes = ragged_param_sizes() + [N * 64 * 20]
    B = N * 64 * 6
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 2)
    for code in S.paro_strategies():
        run = EmuRun(N, M, code, sizes, B, transport=transport, adam_impl=adam_impl, fuse_gather="always")
        plain = _paro().Plan(run.ctx, code, sizes, bucket_elems=B, transport=transport, fuse_gather="never")
        for r in range(N):
            assert run.pl.send_bytes(r) == plain.send_bytes(r), (code, r)
        plain.close()
        for t in (1, 2):
            run.set_grads(t)
            run.step(t)
        _check_against_dp(run, lay, ref)
        run.close()



# --------------------------------------------------------------------- copy-engine all-gathers
@pytest.mark.parametrize("ce", ["gathers", "all"])
@pytest.mark.parametrize("topo", ["ho", "two_step", "h_ring", "flat"])
def test_copy_engine_gathers_every_strategy(topo, ce):
    N, M = 8, 4
    sizes = ragged_param_sizes() + [N * 64 * 20]
    B = N * 64 * 6
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 2)
    for code in S.paro_strategies():
        run = EmuRun(N, M, code, sizes, B, topo=topo, transport="pull", fuse_gather="never", copy_engine=ce)
        for t in (1, 2):
            run.set_grads(t)
            run.step(t)
        if topo == "flat":
            run.close()
            continue
        _check_against_dp(run, lay, ref)
        run.close()


# --------------------------------------------------------------------- partial / PEFT training (NEXT-4)
@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (8, 1), (1, 1)])
def test_masked_plans_peft(N, M):
    """paro_plan_masked: the trainable plan equals unsharded-DP Adam over the
    trainable tensors alone (their own flat layout), the frozen tensors keep
    their initial bf16 parameters bit for bit, and the parameter gathers of
    both plans return the full bf16 model."""
    paro = _paro()
    u = N * 64
    sizes = [u * 5 + 3, 1000, u * 9 + 17, 77, 4096, u * 2]
    mask = [0, 1, 0, 1, 1, 0]
    B = u * 4
    tr = [s for s, t in zip(sizes, mask) if t]
    fr = [s for s, t in zip(sizes, mask) if not t]
    lay_t, lay_f = L.Layout(tr, N, M, B), L.Layout(fr, N, M, B)
    w, m, v, p, _ = _dp_reference(lay_t, 3)
    p_frozen = nm.bf16_bits_from_f32(ST.pad_flat(master_f32(0, lay_f.psi), lay_f.psi_pad, np.float32))
    for code in S.paro_strategies():
        ctx = paro.Context(N, M, mode="emulated", device=0) if N > 1 else \
            paro.Context(1, 1, mode="real", rank=0, device=0, uid=paro.unique_id())
        tp, fp = paro.Plan.masked(ctx, code, sizes, mask, bucket_elems=B, gather_windows=2)
        n = tp.info()["os_numel"]
        st = [tuple(torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(3)) for _ in range(N)]
        for r in range(N):
            tp.opt_state_init(r, [x.data_ptr() for x in st[r]], seed=SEED)
            fp.opt_state_init(r, None, seed=SEED)
        for t in range(1, 4):
            for r in range(N):
                tp.synth_grads(r, SEED, t)
            tp.step([[x.data_ptr() for x in s] for s in st], LR, t)
        torch.cuda.synchronize()
        for r in range(N):
            _assert_same(st[r][0].cpu().numpy(), ST.shard_of(w, lay_t, code[2], r), f"{code} r{r} master")
            _assert_same(st[r][1].cpu().numpy(), ST.shard_of(m, lay_t, code[2], r), f"{code} r{r} m")
            _assert_same(st[r][2].cpu().numpy(), ST.shard_of(v, lay_t, code[2], r), f"{code} r{r} v")
            pt = d2h(tp.buffer(r, 1), tp.info()["p_numel"], np.uint16)
            assert np.array_equal(pt, ST.shard_of(p, lay_t, code[0], r)), (code, r)
            pf = d2h(fp.buffer(r, 1), fp.info()["p_numel"], np.uint16)
            assert np.array_equal(pf, ST.shard_of(p_frozen, lay_f, code[0], r)), (code, r)
        for plan, lay, full in ((tp, lay_t, p), (fp, lay_f, p_frozen)):
            for b, (s0, nb) in enumerate(lay.buckets):
                out = plan.gather_window(0, b, slot=b % 2)
                assert np.array_equal(d2h(out, nb, np.uint16), full[s0:s0 + nb]), (code, b)
        with pytest.raises(paro.ParoError):
            fp.step([[x.data_ptr() for x in s] for s in st], LR, 4)
        fp.close()
        tp.close()
        ctx.close()


# --------------------------------------------------------------------- streamed gradients (grad_slots)
@pytest.mark.parametrize("N,M,K", [(8, 4, 1), (8, 4, 2), (4, 2, 3), (8, 1, 1), (1, 1, 1), (1, 1, 3)])
def test_streamed_step_every_strategy(N, M, K):
    """paro_step_streamed with K gradient slots (the library's synthetic
    producer) gives the same bits as the resident-gradient step: unsharded-DP
    Adam over 3 steps, every strategy (K = 1: every bucket reuses the slot)."""
    paro = _paro()
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 3)
    for code in S.paro_strategies():
        mode = "emulated" if N > 1 else "real"
        run = EmuRun(N, M, code, sizes, B, mode=mode)
        run.pl.close()
        run.pl = paro.Plan(run.ctx, code, sizes, bucket_elems=B, grad_slots=K)
        run.info = run.pl.info()
        assert run.info["grad_buffer_bytes"] == 2 * min(lay.psi_pad, K * B)
        for r in range(N):
            run.pl.opt_state_init(r, [t.data_ptr() for t in run.st[r]], seed=SEED)
        with pytest.raises(paro.ParoError):
            run.pl.synth_grads(0, SEED, 1)
        for t in range(1, 4):
            run.pl.step_streamed(run.ptrs(), LR, t, seed=SEED, grad_step=t)
        _check_against_dp(run, lay, ref)
        st = run.pl.stats()
        assert abs(st["grad_norm"] ** 2 - ref[4][-1]) <= 1e-12 * ref[4][-1]
        run.close()


def test_streamed_step_python_producer():
    """A caller-supplied producer (here: device-to-device copies of the bucket
    from a torch tensor, on the library's stream) drives the streamed step."""
    import ctypes
    paro = _paro()
    N, M, K = 4, 2, 2
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 2)
    from devmem import _cudart
    rt = _cudart()
    rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    rt.cudaMemcpyAsync.restype = ctypes.c_int
    run = EmuRun(N, M, "IIG", sizes, B)
    run.pl.close()
    run.pl = paro.Plan(run.ctx, "IIG", sizes, bucket_elems=B, grad_slots=K)
    run.info = run.pl.info()
    for r in range(N):
        run.pl.opt_state_init(r, [t.data_ptr() for t in run.st[r]], seed=SEED)
    calls = []
    for t in range(1, 3):
        full = [torch.from_numpy(ST.pad_flat(grad_bits(r, t, 0, lay.psi), lay.psi_pad, np.uint16).view(np.int16)).cuda()
                for r in range(N)]
        torch.cuda.synchronize()

        def producer(r, b, b0, b1, dst, stream):
            calls.append((r, b))
            assert rt.cudaMemcpyAsync(dst, full[r].data_ptr() + 2 * b0, 2 * (b1 - b0), 3, stream) == 0

        run.pl.step_streamed(run.ptrs(), LR, t, producer=producer)
        torch.cuda.synchronize()
    assert len(calls) == 2 * N * len(lay.buckets)
    _check_against_dp(run, lay, ref)
    run.close()


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2)])
def test_streamed_step_with_clipping(N, M):
    """Two-phase step (global-norm clipping) with one gradient slot: phase 1
    reduces every bucket as it is produced, the slot is reused once the
    reduction read it (no Adam reads raw slots in two-phase mode at N > 1)."""
    paro = _paro()
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    clip = 0.05
    ref, per = _clip_reference(lay, 3, clip)
    for code in S.paro_strategies():
        run = EmuRun(N, M, code, sizes, B)
        run.pl.close()
        run.pl = paro.Plan(run.ctx, code, sizes, bucket_elems=B, grad_slots=1, clip_norm=clip)
        run.info = run.pl.info()
        for r in range(N):
            run.pl.opt_state_init(r, [t.data_ptr() for t in run.st[r]], seed=SEED)
        for t in range(1, 4):
            run.pl.step_streamed(run.ptrs(), LR, t, seed=SEED, grad_step=t)
            st = run.pl.stats()
            assert abs(st["grad_norm"] ** 2 - per[t - 1][5]) <= 1e-12 * per[t - 1][5]
        _check_against_dp(run, lay, ref)
        run.close()


# --------------------------------------------------------------------- empty / zero-size inputs
@pytest.mark.parametrize("sizes", [[], [0], [0, 5, 0, 77, 0]])
def test_empty_model_and_zero_size_tensors(sizes):
    """An empty parameter list or zero-size tensors: the plan and step run
    (nothing to do for psi = 0; zero-size tensors take no room and may have
    NULL pointers), and the rest still matches unsharded DP."""
    paro = _paro()
    N, M, B = 8, 4, 8 * 64 * 2
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 2) if lay.psi else None
    for code in ("NNN", "IIG", "GGG", "NIG"):
        run = EmuRun(N, M, code, sizes, B)
        assert run.info["psi"] == sum(sizes)
        for t in range(1, 3):
            if lay.psi:
                run.set_grads(t)
                st = run.step(t)
            else:
                run.pl.step([[0, 0, 0]] * N, LR, t)
                st = run.pl.stats()
                assert st["grad_norm"] == 0.0 and st["nonfinite"] == 0
        if lay.psi:
            _check_against_dp(run, lay, ref)
            # per-tensor pointers with NULL for the zero-size tensors (pack path)
            ptrs = []
            for r in range(N):
                g = torch.from_numpy(grad_bits(r, 3, 0, lay.psi).view(np.int16)).cuda()
                o = 0
                for s in sizes:
                    ptrs.append(g.data_ptr() + 2 * o if s else 0)
                    o += s
                run.__dict__.setdefault("_keep", []).append(g)
            run.pl.step(run.ptrs(), LR, 3, grads=ptrs)
            torch.cuda.synchronize()
        run.close()


# --------------------------------------------------------------------- collective only (BASELINE config 5)
@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (2, 1), (8, 1)])
@pytest.mark.parametrize("topo", ["ho", "two_step", "flat"])
def test_collective_allreduce_matches_oracle(N, M, topo):
    """paro_collective(0) of an NNN plan made with fuse_allreduce = 0 is the bf16
    gradient all-reduce the bench sweeps (config 5): every rank's g_hat slot holds
    the canonical-order average (HO-Ring / two-step: dp_reduce; flat ring: the
    oracle's flat-ring simulation), bucket by bucket; a plan that folds part of
    the reduction into Adam is refused."""
    paro = _paro()
    B = N * 64 * 16
    sizes = [3 * B - N * 64 * 5]          # 3 buckets (ragged last): every slot of depth 2 holds one
    lay = L.Layout(sizes, N, M, B)
    grads = _oracle_grads(N, lay.psi, 1)
    if topo == "flat":
        res = ST.strategy_step("NNN", lay, grads, ST.init_state(master_f32(0, lay.psi), lay, "NNN"),
                               nm.AdamScalars(LR, 1), topology="flat")
        want = {r: res.ghat_os[r] for r in range(N)}
    else:
        gh = ST.dp_reduce(lay, grads)
        want = {r: gh for r in range(N)}
    ctx = paro.Context(N, M, mode="emulated", device=0)
    pl = paro.Plan(ctx, "NNN", sizes, bucket_elems=B, topology=topo, fuse_allreduce=False, transport="pull")
    for r in range(N):
        pl.synth_grads(r, SEED, 1)
    pl.collective(0)
    torch.cuda.synchronize()
    for r in range(N):
        for b, (s0, n) in enumerate(lay.buckets):
            got = d2h(pl.buffer(r, 3) + 2 * (b % 3) * B, n, np.uint16)
            assert np.array_equal(got, want[r][s0:s0 + n]), (topo, r, b)
    pl.close()
    fused = paro.Plan(ctx, "GGG", sizes, bucket_elems=B, topology=topo, transport="pull")   # final hop in Adam
    with pytest.raises(paro.ParoError, match="fuse_allreduce = 0"):
        fused.collective(0)
    fused.close()
    ctx.close()


# --------------------------------------------------------------------- fp32 wire / predivide
@pytest.mark.parametrize("topo,transport", [("ho", "pull"), ("ho", "push"), ("two_step", "pull"), ("direct", "pull"),
                                            ("direct", "push")])
def test_fp32_wire_every_strategy_2x4(topo, transport):
    """wire_dtype = 1: fp32 partials and fp32 g_hat through every strategy's
    schedule (fused final hop, fused inter all-reduce, AG of fp32 g_hat) equal
    the oracle's fp32-wire DP definition bit for bit (same split), 3 steps, with
    the default Adam, the LSU Adam and the co-run thread-store Adam."""
    N, M = 8, 4
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 3, wire="fp32")
    for i, code in enumerate(S.paro_strategies()):
        impl, kb = (("auto", 0), ("lsu", 0), ("tma", 120))[i % 3]
        run = EmuRun(N, M, code, sizes, B, topo=topo, transport=transport, wire="fp32", adam_impl=impl,
                     adam_smem_kb=kb)
        for t in (1, 2, 3):
            run.set_grads(t)
            st = run.step(t)
        assert abs(st["grad_norm"] ** 2 - ref[4][-1]) <= 1e-12 * ref[4][-1]
        _check_against_dp(run, lay, ref)
        run.close()


def _a24(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-3)))


def test_fp32_wire_cross_split_within_1e5():
    """SURVEY 8(c-4) cross-split / cross-bucket pin: on the fp32 wire, 10 steps
    at 8 ranks as 2x4, 4x2, 8x1, 1x8 and two bucket sizes each equal their own
    split's oracle bit for bit and agree with the 2x4 reference within 1e-5
    (A24 metric); fp32 masters and bf16 parameters both compared."""
    N = 8
    sizes = [1 << 16]
    lay_ref = L.Layout(sizes, N, 4, 1 << 13)
    w_ref = _dp_reference(lay_ref, 10, wire="fp32")[0][:sizes[0]]
    worst = 0.0
    for (M, B, code) in [(4, 1 << 13, "IIG"), (2, 1 << 13, "NIG"), (1, 1 << 13, "GGG"), (8, 1 << 13, "III"),
                         (4, 1 << 11, "NNN"), (2, 3 * 1024, "IGG")]:
        lay = L.Layout(sizes, N, M, B)
        ref = _dp_reference(lay, 10, wire="fp32")
        run = EmuRun(N, M, code, sizes, B, wire="fp32", transport="pull")
        for t in range(1, 11):
            run.set_grads(t)
            run.step(t)
        _check_against_dp(run, lay, ref)
        full = np.zeros(lay.psi_pad, np.float32)
        for r in range(N):
            off = 0
            st = run.state(r)
            for (a, e) in lay.shard_ranges(code[2], r):
                full[a:e] = st["master"][off:off + e - a]
                off += e - a
        worst = max(worst, _a24(full[:sizes[0]], w_ref))
        run.close()
    assert worst <= 1e-5, worst


@pytest.mark.parametrize("wire", ["bf16", "fp32"])
@pytest.mark.parametrize("N,M", [(8, 4), (6, 3), (4, 1)])
def test_predivide_off_every_strategy(wire, N, M):
    """predivide = 0: the raw gradients are summed and Adam takes the 1/N average
    (s_g = 1/(loss_scale * N)), bit for bit the oracle with post_div = N."""
    sizes = ragged_param_sizes() + [N * 64 * 7 + 3]
    B = N * 64 * 3
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 2, wire=wire, predivide=False, loss_scale=2.0)
    for code in S.paro_strategies():
        run = EmuRun(N, M, code, sizes, B, transport="pull", wire=wire, predivide=False, loss_scale=2.0)
        for t in (1, 2):
            run.set_grads(t)
            st = run.step(t)
        assert abs(st["grad_norm"] ** 2 - ref[4][-1]) <= 1e-12 * ref[4][-1]
        _check_against_dp(run, lay, ref)
        run.close()


@pytest.mark.parametrize("code,kw", [("IIG", {}), ("NNN", {"clip_norm": 0.05}), ("GGG", {"fuse_gather": "always"}),
                                     ("IGG", {"copy_engine": "gathers"})])
def test_fp32_wire_with_options(code, kw):
    """fp32 wire with the two-phase clipped step, fused parameter gathers and
    copy-engine all-gathers (4x2, 2 steps)."""
    N, M = 4, 2
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    if "clip_norm" in kw:
        w = ST.pad_flat(master_f32(0, lay.psi), lay.psi_pad, np.float32)
        m, v = np.zeros_like(w), np.zeros_like(w)
        for t in (1, 2):
            gh = ST.dp_reduce(lay, _oracle_grads(N, lay.psi, t), wire="fp32")
            w, m, v, p = ST.clip_update(gh, w, m, v, LR, t, kw["clip_norm"], False, 1, {})[:4]
        ref = (w, m, v, p, None)
    else:
        ref = _dp_reference(lay, 2, wire="fp32")
    run = EmuRun(N, M, code, sizes, B, transport="pull", wire="fp32", **kw)
    for t in (1, 2):
        run.set_grads(t)
        run.step(t)
    _check_against_dp(run, lay, ref)
    run.close()


# --------------------------------------------------------------------- layer-aligned buckets (NEXT-2 per layer)
LAYERS = lambda d, f, L: [d * 3 + 5] + [d * d, d * d + 7, f * d, d] * L + [d * 3 + 5]


@pytest.mark.parametrize("N,M,topo", [(8, 4, "ho"), (4, 2, "two_step"), (8, 1, "ho"), (6, 3, "flat")])
def test_layer_windows_every_strategy(N, M, topo):
    """bucket_groups: every bucket is one layer group (parameters
    gathered layer by layer for the forward / backward pass).  After 2 steps the
    state equals unsharded DP over the padded layer layout, and gathering layer
    b + 1 on a side stream (prefetch) while layer b's window is read returns
    each layer's full bf16 parameters, bit for bit, on every rank."""
    from paro_synth import grad_flat, master_flat
    paro = _paro()
    sizes = LAYERS(64, 176, 3)
    groups = [0, 1, 5, 9, 13]
    lay = L.Layout(sizes, N, M, 0, groups=groups)
    w = master_flat(lay.psi_pad, lay.real)
    m, v = np.zeros_like(w), np.zeros_like(w)
    for t in (1, 2):
        w, m, v, p, _ = ST.dp_step(lay, [grad_flat(r, t, lay.psi_pad, lay.real) for r in range(N)], w, m, v,
                                   nm.AdamScalars(LR, t))
    ref = (w, m, v, p, None)
    side = torch.cuda.Stream()
    for code in S.paro_strategies():
        ctx = paro.Context(N, M, mode="emulated", device=0)
        pl = paro.Plan(ctx, code, sizes, bucket_groups=groups, topology=topo, gather_windows=2, transport="pull")
        info = pl.info()
        assert info["n_buckets"] == len(lay.buckets) and info["psi_pad"] == lay.psi_pad
        st = [tuple(torch.empty(info["os_numel"], dtype=torch.float32, device="cuda") for _ in range(3))
              for _ in range(N)]
        run = type("R", (), {})()
        run.N, run.code, run.pl, run.st, run.info = N, code, pl, st, info
        run.state = lambda r, run=run: EmuRun.state(run, r)
        for r in range(N):
            pl.opt_state_init(r, [x.data_ptr() for x in st[r]], seed=SEED)
        for t in (1, 2):
            for r in range(N):
                pl.synth_grads(r, SEED, t)
            pl.step([[x.data_ptr() for x in s] for s in st], LR, t)
        if topo != "flat":
            _check_against_dp(run, lay, ref)
        full = np.zeros(lay.psi_pad, np.uint16)
        for r in range(N):       # the full model assembled from every rank's P shards (bit copies)
            mine, off = run.state(r)["param"], 0
            for (a, e) in lay.shard_ranges(code[0], r):
                full[a:e] = mine[off:off + e - a]
                off += e - a
        if topo != "flat":
            assert np.array_equal(full, p), code
        nb = len(lay.buckets)
        pl.gather_window(0, 0, slot=0)
        for b in range(nb):
            if b + 1 < nb:       # prefetch the next layer on a side stream
                pl.gather_window(0, b + 1, slot=(b + 1) % 2, stream=side.cuda_stream)
            s0, n = lay.buckets[b]
            for r in range(N):
                resident = info["p_numel"] == lay.psi_pad      # P = N (or I with groups of one GPU)
                ptr = pl.buffer(r, 1) + 2 * s0 if resident else pl.buffer(r, 5) + 2 * (b % 2) * lay.B
                got = d2h(ptr, n, np.uint16)
                assert np.array_equal(got, full[s0:s0 + n]), (code, b, r)
            torch.cuda.current_stream().wait_stream(side)
        pl.close()
        ctx.close()


# --------------------------------------------------------------------- one-shot topology
@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (8, 1), (6, 3), (2, 1), (9, 3), (4, 4)])
def test_oneshot_every_strategy_ragged(N, M):
    """PARO_TOPO_ONESHOT: one round per collective, nested N-input folds in the
    owner's canonical order: every strategy bit-exact vs unsharded DP (same
    bits as HO-Ring), 2 steps, ragged sizes; with and without the folds fused
    into Adam; the fp32 wire too."""
    sizes = ragged_param_sizes() + [N * 64 * 7 + 3]
    B = N * 64 * 3
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 2)
    ref32 = _dp_reference(lay, 2, wire="fp32")
    for i, code in enumerate(S.paro_strategies()):
        for fuse, wire in ((True, "bf16"), (False, "bf16"), (True, "fp32")):
            if wire == "fp32" and i % 2:
                continue
            run = EmuRun(N, M, code, sizes, B, topo="oneshot", transport="pull", fuse_allreduce=fuse, wire=wire)
            for t in (1, 2):
                run.set_grads(t)
                run.step(t)
            _check_against_dp(run, lay, ref if wire == "bf16" else ref32)
            run.close()


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2)])
def test_oneshot_accumulation_and_collective(N, M):
    """One-shot schedules with gradient accumulation (s = 3, the accumulator
    hopped after the nested fold) and the NNN all-reduce through paro_collective."""
    s = 3
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    refs = {gl: _accum_reference(lay, 2, s, gl) for gl in "NIG"}
    for code in S.paro_strategies():
        run = EmuRun(N, M, code, sizes, B, topo="oneshot", transport="pull", grad_accum=True)
        _run_accum(run, 2, s)
        _check_against_dp(run, lay, refs[code[1]])
        run.close()
    paro = _paro()
    ctx = paro.Context(N, M, mode="emulated", device=0)
    pl = paro.Plan(ctx, "NNN", [3 * B], bucket_elems=B, topology="oneshot", fuse_allreduce=False)
    lay3 = L.Layout([3 * B], N, M, B)
    gh = ST.dp_reduce(lay3, _oracle_grads(N, lay3.psi, 1))
    for r in range(N):
        pl.synth_grads(r, SEED, 1)
    pl.collective(0)
    torch.cuda.synchronize()
    for r in range(N):
        for b, (s0, n) in enumerate(lay3.buckets):
            assert np.array_equal(d2h(pl.buffer(r, 3) + 2 * (b % 3) * B, n, np.uint16), gh[s0:s0 + n]), (r, b)
    pl.close()
    ctx.close()


# --------------------------------------------------------------------- parameter consumer
@pytest.mark.parametrize("N,M,slots", [(8, 4, 0), (4, 2, 2), (2, 1, 0), (1, 1, 2)])
def test_param_consumer_every_strategy(N, M, slots):
    """paro_set_param_consumer: each bucket's updated bf16 parameters (the rank's
    P residency) are handed over on a side stream as soon as they are final; a
    consumer that copies them out gets exactly the parameter buffer after the
    step (= unsharded DP), every bucket once per step, in bucket order; also in
    streamed steps (grad_slots) and at N = 1."""
    import ctypes
    from devmem import _cudart
    paro = _paro()
    rt = _cudart()
    rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    rt.cudaMemcpyAsync.restype = ctypes.c_int
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    ref = _dp_reference(lay, 2)
    for code in S.paro_strategies():
        mode = "emulated" if N > 1 else "real"
        run = EmuRun(N, M, code, sizes, B, mode=mode, transport="pull")
        if slots:
            run.pl.close()
            run.pl = paro.Plan(run.ctx, code, sizes, bucket_elems=B, grad_slots=slots, transport="pull")
            run.info = run.pl.info()
            for r in range(N):
                run.pl.opt_state_init(r, [t.data_ptr() for t in run.st[r]], seed=SEED)
        out = [torch.zeros(run.info["p_numel"], dtype=torch.int16, device="cuda") for _ in range(N)]
        calls = []

        def consumer(r, b, b0, b1, src, stream, out=out, calls=calls, run=run):
            calls.append((r, b))
            off = src - run.pl.buffer(r, 1)
            assert rt.cudaMemcpyAsync(out[r].data_ptr() + off, src, 2 * (b1 - b0), 3, stream) == 0

        run.pl.set_param_consumer(consumer)
        for t in (1, 2):
            if slots:
                run.pl.step_streamed(run.ptrs(), LR, t, seed=SEED, grad_step=t)
            else:
                run.set_grads(t)
                run.step(t)
        torch.cuda.synchronize()
        _check_against_dp(run, lay, ref)
        nb = len(lay.buckets)
        assert calls == [(r, b) for _ in range(2) for b in range(nb) for r in range(N)]
        for r in range(N):
            assert np.array_equal(out[r].cpu().numpy().view(np.uint16), run.state(r)["param"]), (code, r)
        run.pl.set_param_consumer(None)
        run.close()


@pytest.mark.parametrize("N,M,topo", [(8, 4, "ho"), (4, 2, "two_step"), (2, 1, "ho"), (8, 4, "oneshot")])
def test_fp32_wire_accumulation_every_strategy(N, M, topo):
    """Gradient accumulation on the fp32 wire: fp32 accumulators at the G
    residency (s = 3 micro-batches, 2 steps), every strategy bit-exact vs
    dp_accum_step(wire = fp32)."""
    s = 3
    sizes = [N * 64 * 40 + 24, 1000]
    B = N * 64 * 8
    lay = L.Layout(sizes, N, M, B)
    refs = {gl: _accum_reference(lay, 2, s, gl, wire="fp32") for gl in "NIG"}
    for code in S.paro_strategies():
        run = EmuRun(N, M, code, sizes, B, topo=topo, transport="pull", grad_accum=True, wire="fp32")
        stats = _run_accum(run, 2, s)
        _check_against_dp(run, lay, refs[code[1]])
        assert abs(stats[-1]["grad_norm"] ** 2 - refs[code[1]][4][-1]) <= 1e-12 * refs[code[1]][4][-1]
        run.close()
