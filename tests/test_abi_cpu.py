"""C-ABI tests that need no GPU: the library loads, exports every symbol
include/paro.h declares, and its host planner agrees bit-exactly with the
oracle (shard maps, per-rank bytes counted from the transfer lists, memory
accounting, error strings)."""
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import accounting as A
from oracle import layout as L
from oracle import numerics as nm
from oracle import step as ST
from oracle import strategy as S
from paper_2310_06003_b200 import paro
from paro_synth import grad_bits, llama_param_sizes, master_f32

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "paro.h")).read()
    declared = set(re.findall(r"\b(paro_[a-z0-9_]+)\s*\(", hdr))
    out = subprocess.run(["nm", "-D", "--defined-only", paro.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (paro_[a-z0-9_]+)$", out, re.M))
    assert declared, "no declarations parsed"
    assert declared <= exported, declared - exported
    assert set(paro.EXPORTED) == declared


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", paro.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_strings():
    ctx = paro.Context(8, 4)
    for code, msg in [("XGG", "invalid shard level 'X' at position 1"),
                      ("GGN", "strategy 'GGN' violates Principle 1 (S_P>=S_OS and S_G>=S_OS)"),
                      ("IG", "strategy code must have 3 characters")]:
        with pytest.raises(paro.ParoError, match=re.escape(msg)):
            paro.Plan(ctx, code, [1024])
    with pytest.raises(paro.ParoError, match="group_size must divide n_gpus"):
        paro.Context(9, 4)
    ctx.close()


def test_all_27_codes_accept_exactly_table1():
    ctx = paro.Context(4, 2)
    ok = []
    for code in S.enumerate_all():
        try:
            paro.Plan(ctx, code, [4096]).close()
            ok.append(code)
        except paro.ParoError:
            pass
    assert sorted(ok) == sorted(S.TABLE1_ROWS)
    ctx.close()


SPLITS = [(8, 4), (8, 2), (4, 2), (9, 3), (8, 1), (8, 8), (2, 1), (1, 1), (12, 3), (6, 2), (16, 4)]


@pytest.mark.parametrize("N,M", SPLITS)
def test_shard_ranges_and_memory_match_oracle(N, M):
    sizes = [3000, 517, 64, 9000, 7]
    B = N * 64 * 4
    lay = L.Layout(sizes, N, M, B)
    ctx = paro.Context(N, M)
    for code in S.paro_strategies():
        pl = paro.Plan(ctx, code, sizes, bucket_elems=B)
        info = pl.info()
        assert info["psi"] == lay.psi and info["psi_pad"] == lay.psi_pad
        assert info["n_buckets"] == len(lay.buckets) and info["bucket_elems"] == lay.B
        for b in range(len(lay.buckets)):
            assert pl.bucket_range(b) == (lay.buckets[b][0], sum(lay.buckets[b]))
            for r in range(N):
                for st, lvl in zip(("P", "G", "OS"), code):
                    assert pl.shard_range(st, r, b) == lay.residency(lvl, r, b)
        mp, mg, mo = A.memory_strategy(code, N, M, lay.psi_pad)
        assert (info["mem_p_bytes"], info["mem_g_bytes"], info["mem_os_bytes"]) == (mp, mg, mo)
        assert info["p_numel"] == lay.shard_numel(code[0])
        assert info["os_numel"] == lay.shard_numel(code[2])
        pl.close()
    ctx.close()


@pytest.mark.parametrize("N,M", SPLITS)
def test_send_bytes_match_oracle_simulator(N, M):
    """Bytes counted from the library's transfer lists == the oracle's round
    simulator (HO-Ring, two-step and flat topologies), bit-exact."""
    sizes = [3000, 517, 64, 9000, 7]
    B = N * 64 * 4
    lay = L.Layout(sizes, N, M, B)
    grads = [grad_bits(r, 1, 0, lay.psi) for r in range(N)]
    w0 = master_f32(0, lay.psi)
    ctx = paro.Context(N, M)
    for code in S.paro_strategies():
        for topo, tr, ce in [(a, b, c) for a in ("ho", "two_step", "flat", "h_ring") for b in ("push", "pull")
                             for c in (False, "gathers", "all", "tails")]:
            pl = paro.Plan(ctx, code, sizes, bucket_elems=B, topology=topo, transport=tr, copy_engine=ce)
            res = ST.strategy_step(code, lay, grads, ST.init_state(w0, lay, code), nm.AdamScalars(1e-3, 1),
                                   topology=topo)
            for r in range(N):
                assert pl.send_bytes(r) == (2 * res.sent[r][0], 2 * res.sent[r][1]), (code, topo, r)
            pl.close()
    ctx.close()


@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (4, 2), (8, 1), (8, 8), (16, 4)])
def test_direct_topology_bytes_equal_closed_form(N, M):
    ctx = paro.Context(N, M)
    for code in S.paro_strategies():
        for tr in ("push", "pull"):
            pl = paro.Plan(ctx, code, [N * 64 * 16], bucket_elems=N * 64 * 4, topology="direct", transport=tr)
            a, b = A.step_units_per_rank(code, N, M, N * 64 * 16)
            for r in range(N):
                assert pl.send_bytes(r) == (2 * a, 2 * b), code
            pl.close()
    ctx.close()


def test_llama7b_plan_accounting():
    sizes = llama_param_sizes("7B")
    assert len(sizes) == 291 and sum(sizes) == 6_738_415_616
    ctx = paro.Context(8, 4)
    for code in S.paro_strategies():
        pl = paro.Plan(ctx, code, sizes, bucket_elems=1 << 26)
        info = pl.info()
        assert info["psi_pad"] == 6_738_415_616 and info["n_buckets"] == 101
        a, b = A.step_units_per_rank(code, 8, 4, info["psi_pad"])
        for r in range(8):
            assert pl.send_bytes(r) == (2 * a, 2 * b)
        pl.close()
    ctx.close()


@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (4, 2), (9, 3), (8, 1), (8, 8), (1, 1)])
def test_accumulation_bytes_match_oracle_simulator(N, M):
    """grad_accum plans: s * (bytes per paro_accumulate) + (bytes of the step
    after it) == the oracle's simulated mini-batch with s micro-batches, for
    s = 1 and s = 3 (pins both per-call numbers), every strategy and topology."""
    sizes = [3000, 517, 64, 9000, 7]
    B = N * 64 * 4
    lay = L.Layout(sizes, N, M, B)
    w0 = master_f32(0, lay.psi)
    zero = [np.zeros(lay.psi, np.uint16) for _ in range(N)]
    ctx = paro.Context(N, M)
    for code in S.paro_strategies():
        for topo, tr, ce in [("ho", "pull", False), ("ho", "push", False), ("two_step", "pull", False),
                             ("flat", "pull", False), ("direct", "push", False), ("ho", "pull", "all")]:
            pl = paro.Plan(ctx, code, sizes, bucket_elems=B, topology=topo, transport=tr, grad_accum=True,
                           copy_engine="all" if ce else False)
            for s in (1, 3):
                res = ST.strategy_accum_step(code, lay, [zero] * s, ST.init_state(w0, lay, code),
                                             nm.AdamScalars(1e-3, 1, accum_steps=s),
                                             topology="two_step" if topo == "direct" else topo)
                for r in range(N):
                    (ai, ae), (si, se) = pl.accum_send_bytes(r)
                    if topo == "direct":    # one-shot: bytes follow the closed form, not the ring trace
                        per_mb, once = A.accum_ops(code)
                        assert (s * ai + si, s * ae + se) == tuple(2 * x for x in A.accum_units_per_rank(
                            code, N, M, lay.psi_pad, s)), (code, r)
                    else:
                        assert (s * ai + si, s * ae + se) == (2 * res.sent[r][0], 2 * res.sent[r][1]), \
                            (code, topo, tr, s, r)
            pl.close()
    ctx.close()


def test_accumulate_needs_grad_accum_plan():
    ctx = paro.Context(4, 2)
    pl = paro.Plan(ctx, "IIG", [4096])
    with pytest.raises(paro.ParoError, match="grad_accum"):
        pl.accum_send_bytes(0)
    with pytest.raises(paro.ParoError, match="NCCL"):
        paro.Plan(ctx, "IIG", [4096], topology="nccl", grad_accum=True)
    pl.close()
    ctx.close()


@pytest.mark.parametrize("N,M", [(8, 4), (8, 2), (4, 2), (9, 3), (8, 1), (8, 8)])
def test_gather_window_bytes_match_oracle(N, M):
    """Forward/backward parameter gathers (NEXT-2): bytes per full pass over
    the buckets == the oracle's simulated AG rounds, every strategy / topology."""
    sizes = [3000, 517, 64, 9000, 7]
    B = N * 64 * 4
    lay = L.Layout(sizes, N, M, B)
    full = nm.bf16_bits_from_f32(ST.pad_flat(master_f32(0, lay.psi), lay.psi_pad, np.float32))
    ctx = paro.Context(N, M)
    for code in S.paro_strategies():
        params = {r: ST.shard_of(full, lay, code[0], r) for r in range(N)}
        for topo, tr in [("ho", "pull"), ("ho", "push"), ("two_step", "pull"), ("flat", "push"), ("h_ring", "pull")]:
            pl = paro.Plan(ctx, code, sizes, bucket_elems=B, topology=topo, transport=tr, gather_windows=2)
            _, sent = ST.param_gather(code, lay, params, topology=topo)
            for r in range(N):
                assert pl.gather_send_bytes(r) == (2 * sent[r][0], 2 * sent[r][1]), (code, topo, tr, r)
            pl.close()
    ctx.close()


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (6, 3), (8, 2), (4, 1), (2, 1)])
def test_fused_inter_allreduce_keeps_table3_bytes(N, M):
    """R31: folding AR_E into Adam (OS = I, g = 2, pull) sends exactly the
    ring's bytes per link class (Table 3 closed form), in fewer rounds; other
    splits (g != 2, M = 1) and push plans are unchanged (OS = G: fuse_allreduce
    = 0 also moves the final hop back into the rounds kernel, never fewer rounds)."""
    ctx = paro.Context(N, M)
    sizes = [1 << 20, 4000037]
    g = N // M
    for code in ("III", "NII", "IIG", "INI", "NNI", "NNG", "NNN"):
        res = {}
        for transport in ("pull", "push"):
            for fuse in (True, False):
                i = paro.Plan(ctx, code, sizes, bucket_elems=1 << 17, transport=transport,
                              fuse_allreduce=fuse).info()
                res[transport, fuse] = (i["step_send_bytes_intra"], i["step_send_bytes_inter"], i["n_rounds"])
        assert len({v[:2] for v in res.values()}) == 1, (code, res)
        psi_pad = paro.Plan(ctx, code, sizes, bucket_elems=1 << 17).info()["psi_pad"]
        intra, inter = res["pull", True][:2]
        full = 2 * psi_pad
        assert inter == 2 * (g - 1) * full // N          # AR_E or RS_E + AG_E: 2(g-1)Psi/N
        assert intra == (M - 1) * full // M * (2 if code[0] == "N" else 1)
        fused = g == 2 and ((M > 1 and code[2] == "I") or (M == 1 and code[2] != "G"))
        if code[2] == "G":   # fuse_allreduce = 0 also keeps OS = G's final hop in the rounds kernel
            for tr in ("pull", "push"):
                assert res[tr, True][2] <= res[tr, False][2]
        else:
            assert (res["pull", True][2] < res["pull", False][2]) == fused
            assert res["push", True][2] == res["push", False][2]


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (8, 1), (6, 3)])
def test_fp32_wire_bytes_and_memory(N, M):
    """wire_dtype = 1 (reading A3): reduction partials travel as fp32, the
    parameter restore stays bf16.  Push transport and the NCCL comparator send
    every reduction element at 4 B: per-rank bytes = 4 x (reduction units) + 2 x
    (restore units), the per-strategy closed form at fp32 width.  Pull plans
    read the raw bf16 gradients at a ring's first hop (the reader pre-scales),
    so they send between the bf16 and the all-fp32 figure.  The G residency is
    4 B per element; copy_engine = 2 is refused."""
    ctx = paro.Context(N, M)
    sizes = [1 << 20, 4000037]
    for code in ("NNN", "NNI", "NIG", "INI", "IIG", "IGG", "GGG", "III"):
        for topo, tr in (("ho", "push"), ("two_step", "push"), ("nccl", "pull"), ("ho", "pull"), ("direct", "pull")):
            kw = dict(bucket_elems=1 << 17, topology=topo, transport=tr)
            b16 = paro.Plan(ctx, code, sizes, **kw).info()
            f32 = paro.Plan(ctx, code, sizes, wire_dtype="fp32", **kw).info()
            grad, rest = A.step_ops(code)
            units = lambda prims: [sum(x) for x in zip(*[A.primitive_units(pr, N, M, b16["psi_pad"])
                                                         for pr in prims])] or [0, 0]
            red, res = units(grad), units(rest)
            full = (4 * red[0] + 2 * res[0], 4 * red[1] + 2 * res[1])
            got = (f32["step_send_bytes_intra"], f32["step_send_bytes_inter"])
            assert (b16["step_send_bytes_intra"], b16["step_send_bytes_inter"]) == (2 * red[0] + 2 * res[0],
                                                                                  2 * red[1] + 2 * res[1])
            if tr == "push" or topo == "nccl":
                assert got == full, (code, topo, tr)
            else:
                assert all(b16[k] <= f32[k] for k in ("step_send_bytes_intra", "step_send_bytes_inter"))
                assert got[0] <= full[0] and got[1] <= full[1], (code, topo, tr)
            assert f32["mem_p_bytes"] == b16["mem_p_bytes"] and f32["mem_os_bytes"] == b16["mem_os_bytes"]
            if code[1] == "G" or (code[1] == "I" and M > 1):   # (M = 1: I is N, the raw bf16 buffer)
                assert f32["mem_g_bytes"] == 2 * b16["mem_g_bytes"]
    with pytest.raises(paro.ParoError, match="fp32"):
        paro.Plan(ctx, "IIG", sizes, wire_dtype="fp32", copy_engine="all")
    paro.Plan(ctx, "IIG", sizes, wire_dtype="fp32", grad_accum=True).close()   # fp32 accumulators
    ctx.close()


LAYERS = lambda d, f, L: [d * 3 + 5] + [d * d, d * d + 7, f * d, d] * L + [d * 3 + 5]


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (8, 1), (6, 3), (1, 1)])
def test_layer_aligned_buckets_layout_and_window_bytes(N, M):
    """bucket_groups (NEXT-2): bucket k holds exactly one layer group
    (dense, padded at its end to N*64), identically in the library and the oracle
    layout; one bucket's forward / backward gather sends Table 3's per-layer
    A-G(P): P = I (IIG, IGG) the MiCS-style intra AG, cluster total N(M-1)/M x
    the layer; P = G on the flat ring (GGG = ZeRO-3) the flat AG
    split (rank-order attribution, A14); P = G on HO-Ring the HO_AG closed form."""
    sizes = LAYERS(64, 176, 3)
    groups = [0, 1, 5, 9, 13]      # embedding, three layers of 4 tensors, head
    lay = L.Layout(sizes, N, M, 0, groups=groups)
    unit = N * 64
    for k, (s0, n) in enumerate(lay.buckets):
        assert n % unit == 0 and s0 % unit == 0
        t1 = groups[k + 1] if k + 1 < len(groups) else len(sizes)
        real = sum(sizes[groups[k]:t1])
        assert lay.real[k] == (s0, s0 + real) and n == -(-real // unit) * unit
        for t in range(groups[k], t1):
            assert s0 <= lay.param_offsets[t] and lay.param_offsets[t] + sizes[t] <= s0 + real
    x = np.arange(1, lay.psi + 1, dtype=np.int64)
    e = lay.expand(x)
    assert e.sum() == x.sum() and all(not e[a:b].any() for (_, b), (a, _) in zip(lay.real, lay.buckets[1:]))
    ctx = paro.Context(N, M)
    for code, topo in (("IIG", "ho"), ("IGG", "ho"), ("GGG", "flat"), ("GGG", "ho"), ("NNG", "ho")):
        pl = paro.Plan(ctx, code, sizes, bucket_groups=groups, topology=topo, gather_windows=2)
        info = pl.info()
        assert info["psi"] == lay.psi and info["psi_pad"] == lay.psi_pad and info["n_buckets"] == len(lay.buckets)
        for b, (s0, n) in enumerate(lay.buckets):
            assert pl.bucket_range(b) == (s0, s0 + n)
            for r in range(N):
                for st in ("P", "G", "OS"):
                    assert pl.shard_range(st, r, b) == lay.residency({"P": code[0], "G": code[1], "OS": code[2]}[st],
                                                                     r, b)
            per = [pl.gather_send_bytes(r, b) for r in range(N)]
            tot = (sum(a for a, _ in per), sum(c for _, c in per))
            if code[0] == "N" or N == 1:
                assert tot == (0, 0)
            elif code[0] == "I" and M > 1 and N // M > 1:
                cell = A.table3("PaRO-IIG", N, M, 1, n)["fwd_ag_p"]
                assert tot == (2 * cell[0], 2 * cell[1]), (code, b)
            elif topo == "flat":
                cell = A.table3("ZeRO-3", N, M, 1, n)["fwd_ag_p"]
                assert tot == (2 * cell[0], 2 * cell[1]), (code, b)
            elif code[0] == "G":
                u = A.primitive_units("HO_AG", N, M, n)
                assert all(x == (2 * u[0], 2 * u[1]) for x in per), (code, b)
        pl.close()
    ctx.close()


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (8, 1), (6, 3), (2, 1), (4, 4)])
def test_oneshot_topology_rounds_and_bytes(N, M):
    """PARO_TOPO_ONESHOT: every collective is one round; a rank reads its
    segment C = B/N from each of the N - 1 peers (RS: (M-1)C intra + (N-M)C
    inter per bucket, the AG the same), NNN's all-reduce reads the whole bucket
    from every peer ((N-1)B, one round); G = I's RS_I / RS_E read the group /
    position peers' chunk / segment ((M-1)B/M, (g-1)C: the ring's bytes).
    Closed forms counted from the definition of the one-shot schedule."""
    ctx = paro.Context(N, M)
    g = N // M
    B = N * 64 * 8
    sizes = [B * 3]
    for code in ("NNN", "GGG", "NNG", "IGG", "IIG", "III"):
        pl = paro.Plan(ctx, code, sizes, bucket_elems=B, topology="oneshot", fuse_allreduce=False)
        info = pl.info()
        C, nb = B // N, info["n_buckets"]
        if code == "NNN":
            want = (2 * (M - 1) * B * nb, 2 * (N - M) * B * nb) if N > 1 else (0, 0)
            rounds = nb
        elif code in ("GGG", "NNG", "IGG"):
            rs = ((M - 1) * C, (N - M) * C)
            if code == "GGG":
                ag = (0, 0)
            elif code == "NNG":
                ag = rs
            else:                                    # IGG: P = I, restore AG_E over the g positions
                ag = (0, (g - 1) * C)
            want = (2 * (rs[0] + ag[0]) * nb, 2 * (rs[1] + ag[1]) * nb)
            rounds = nb * ((1 if N > 1 else 0) + (1 if sum(ag) else 0))
        else:                                        # IIG / III: RS_I + RS_E (+ AG_E of g_hat for III)
            gi = M > 1 and g > 1
            if not gi:
                pl.close()
                continue
            want = (2 * (M - 1) * (B // M) * nb,
                    2 * ((g - 1) * C + (g - 1) * C) * nb)   # RS_E + (IIG: AG_E of params | III: AG_E of g_hat)
            rounds = 3 * nb     # RS_I, RS_E, then AG_E (IIG: of the parameters; III: of g_hat)
        assert (info["step_send_bytes_intra"], info["step_send_bytes_inter"]) == want, code
        assert info["n_rounds"] == rounds, (code, info["n_rounds"], rounds)
        pl.close()
    with pytest.raises(paro.ParoError, match="pull-only"):
        paro.Plan(ctx, "IIG", sizes, topology="oneshot", transport="push")
    ctx.close()


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2), (8, 1), (2, 1)])
def test_oneshot_allreduce_one_or_two_rounds(N, M):
    """One-shot NNN all-reduce: one round ((N-1)B read per rank) while the extra
    bytes over one-shot RS + AG (two rounds, 2(N-1)/N B, the ring's volume) stay
    under ~6 MB (a barrier's worth of NVLink time), always at N = 2; two rounds
    with the ring's bytes for larger buckets."""
    ctx = paro.Context(N, M)
    for B in (N * 64 * 8, N * 64 * (1 << 14)):
        pl = paro.Plan(ctx, "NNN", [2 * B], bucket_elems=B, topology="oneshot", fuse_allreduce=False)
        info = pl.info()
        C = B // N
        one = N == 2 or (N - 1) * (N - 2) * B * 2 // N <= 6 << 20
        if one:
            want = (2 * (M - 1) * B * 2, 2 * (N - M) * B * 2)
        else:
            want = (2 * 2 * (M - 1) * C * 2, 2 * 2 * (N - M) * C * 2)
        assert (info["step_send_bytes_intra"], info["step_send_bytes_inter"]) == want, (B, one)
        assert info["n_rounds"] == 2 * (1 if one else 2)
        pl.close()
    ctx.close()


@pytest.mark.parametrize("N,M", [(8, 4), (4, 2)])
def test_oneshot_large_buckets_run_ho_ring(N, M):
    """The one-shot topology keeps one-shot schedules while a bucket is small
    (<= 256 MiB of payload) and hands larger buckets to the
    HO-Ring schedules (the same canonical bits; all-to-all pulls move less than
    a ring on one NVSwitch box): a large-bucket plan equals the HO-Ring plan in
    rounds and bytes."""
    ctx = paro.Context(N, M)
    big = N * 64 * (1 << 16) * 32         # > 256 MiB of bf16 per bucket
    for code in ("NNN", "IIG", "GGG", "NIG"):
        one = paro.Plan(ctx, code, [2 * big], bucket_elems=big, topology="oneshot", fuse_allreduce=False).info()
        ho = paro.Plan(ctx, code, [2 * big], bucket_elems=big, topology="ho", fuse_allreduce=False).info()
        for k in ("step_send_bytes_intra", "step_send_bytes_inter", "n_rounds", "n_comm_launches"):
            assert one[k] == ho[k], (code, k)
    ctx.close()


def test_param_consumer_needs_a_device_context():
    """paro_set_param_consumer registers a per-bucket consumer for device plans;
    a planning-only context has no steps (PARO_ERR_STATE)."""
    ctx = paro.Context(4, 2)
    pl = paro.Plan(ctx, "IIG", [1 << 16], bucket_elems=1 << 14)
    with pytest.raises(paro.ParoError, match="planning-only"):
        pl.set_param_consumer(lambda *a: None)
    pl.close()
    ctx.close()
