"""Pins for oracle/numerics.py against things other than itself (CPU).

bf16 rounding is pinned to torch's RNE conversion (a library routine) and to
hand-derived bit patterns; the hop and the canonical order to hand-derived
cases where order changes the result; Adam to torch.optim.AdamW and to the
closed form of step 1 (P:225 Adam; readings R2, R5-R7).
"""
import math

import numpy as np
import pytest
import torch

from oracle import numerics as nm


def _torch_bf16_bits(x):
    t = torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


def test_bf16_rne_matches_torch_on_random_and_ties():
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(200_000) * np.exp2(rng.integers(-40, 40, 200_000))).astype(np.float32)
    # exact ties: low 16 bits = 0x8000
    ties = ((rng.integers(0, 2**31, 50_000, dtype=np.uint32) & np.uint32(0x7F7F0000))
            | np.uint32(0x8000)).view(np.float32)
    allx = np.concatenate([x, ties, np.float32([0.0, -0.0, 1.0, np.inf, -np.inf, 3.3895314e38])])
    assert np.array_equal(nm.bf16_bits_from_f32(allx), _torch_bf16_bits(allx))


def test_bf16_hand_values():
    # 1.0 -> 0x3F80; 1 + 2^-8 is a tie -> even (1.0); 1 + 3*2^-8 tie -> 1 + 2^-6 (0x3F82)
    vals = np.float32([1.0, 1.0 + 2.0**-8, 1.0 + 3 * 2.0**-8, -2.0, 3.397e38])
    got = nm.bf16_bits_from_f32(vals)
    assert list(got[:4]) == [0x3F80, 0x3F80, 0x3F82, 0xC000]
    assert got[4] == 0x7F80  # overflow rounds to +inf
    nan = nm.bf16_bits_from_f32(np.float32([np.nan]))
    assert np.isnan(nm.f32_from_bf16_bits(nan))[0]
    # NaN with only low payload bits must stay NaN (not collapse to inf)
    weird = np.uint32([0x7F800001]).view(np.float32)
    assert np.isnan(nm.f32_from_bf16_bits(nm.bf16_bits_from_f32(weird)))[0]


def test_hop_is_fp32_add_then_rne_matches_torch():
    rng = np.random.default_rng(1)
    a = nm.bf16_bits_from_f32(rng.standard_normal(100_000).astype(np.float32))
    b = nm.bf16_bits_from_f32((rng.standard_normal(100_000) * 1e-3).astype(np.float32))
    ta = torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).float()
    tb = torch.from_numpy(b.view(np.int16)).view(torch.bfloat16).float()
    ref = (ta + tb).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(nm.hop(a, b), ref)


def test_canonical_fold_order_hand_case():
    # y0 = 1, y1 = y2 = 2^-8 (half an ulp of 1 in bf16).
    # R_3(0) = (y1 (+) y2) (+) y0 = 2^-7 (+) 1 = 1 + 2^-7 (exact).
    # R_3(1) = (y2 (+) y0) (+) y1: 1 + 2^-8 is a tie -> 1; again -> 1.
    # R_3(2) = (y0 (+) y1) (+) y2 = 1 as well.
    ys = [nm.bf16_bits_from_f32(np.float32([v])) for v in (1.0, 2.0**-8, 2.0**-8)]
    got = [nm.f32_from_bf16_bits(nm.canonical_fold(ys, c))[0] for c in range(3)]
    assert got == [np.float32(1 + 2.0**-7), np.float32(1.0), np.float32(1.0)]


def test_canonical_fold_exact_on_small_integers_any_owner():
    rng = np.random.default_rng(2)
    for k in (1, 2, 3, 5, 8):
        ints = rng.integers(-3, 4, size=(k, 64)).astype(np.float32)
        ys = [nm.bf16_bits_from_f32(row) for row in ints]
        for c in range(k):
            out = nm.f32_from_bf16_bits(nm.canonical_fold(ys, c))
            assert np.array_equal(out, ints.sum(0))


def test_two_member_fold_is_owner_independent():
    """Reading R31's premise: R_2(0; y) == R_2(1; y) bit for bit (one hop, and
    IEEE fp32 addition is commutative), on random bf16 patterns including
    +-0, subnormals, +-inf and NaN (NaN compared by class), while for k = 3 the
    owner changes the bits (the hand case above), so the fused inter all-reduce
    is only exact at g = 2."""
    rng = np.random.default_rng(31)
    bits = rng.integers(0, 1 << 16, size=(2, 1 << 16), dtype=np.uint32).astype(np.uint16)
    bits[0, :6] = [0x0000, 0x8000, 0x0001, 0x7F80, 0xFF80, 0x7FC0]
    bits[1, :6] = [0x8000, 0x0000, 0x8001, 0xFF80, 0x7F80, 0x3F80]
    ys = [bits[0], bits[1]]
    a, b = nm.canonical_fold(ys, 0), nm.canonical_fold(ys, 1)
    fa, fb = nm.f32_from_bf16_bits(a), nm.f32_from_bf16_bits(b)
    assert np.array_equal(np.isnan(fa), np.isnan(fb))
    ok = ~np.isnan(fa)
    assert np.array_equal(a[ok], b[ok])
    # the same as a plain fp32 sum rounded once (torch), either order
    t = (torch.from_numpy(nm.f32_from_bf16_bits(bits[1])) + torch.from_numpy(nm.f32_from_bf16_bits(bits[0])))
    ref = t.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(a[ok], ref[ok])


def test_pack_power_of_two_scale_is_exponent_shift():
    rng = np.random.default_rng(3)
    x = nm.bf16_bits_from_f32((rng.standard_normal(10_000) * 1e-3).astype(np.float32))
    x = x[(x & 0x7F80) > (3 << 7)]   # normal values whose exponent survives -3
    got = nm.pack(x, 1.0 / 8)
    assert np.array_equal(got, x - np.uint16(3 << 7))


def _torch_adamw(w0, grads, lr, wd, b1=0.9, b2=0.95, eps=1e-8):
    p = torch.nn.Parameter(torch.from_numpy(w0.copy()))
    opt = torch.optim.AdamW([p], lr=lr, betas=(b1, b2), eps=eps, weight_decay=wd,
                            foreach=False, fused=False)
    for g in grads:
        p.grad = torch.from_numpy(g.copy())
        opt.step()
    return p.detach().numpy()


@pytest.mark.parametrize("wd", [0.0, 0.1])
def test_adam_matches_torch_adamw_10_steps(wd):
    rng = np.random.default_rng(4)
    n = 1 << 16
    w = (rng.standard_normal(n) * 0.02).astype(np.float32)
    grads = []
    for _ in range(10):
        gb = nm.bf16_bits_from_f32((rng.standard_normal(n) * 1e-3).astype(np.float32))
        grads.append(gb)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    ww = w.copy()
    for t, gb in enumerate(grads, start=1):
        sc = nm.AdamScalars(3e-4, t, weight_decay=wd)
        ww, m, v, _ = nm.adam_update(ww, m, v, gb, sc)
    ref = _torch_adamw(w, [nm.f32_from_bf16_bits(g) for g in grads], 3e-4, wd)
    assert np.max(np.abs(ww - ref)) < 1e-8


def test_adam_step1_closed_form_and_zero_gradient():
    n = 4096
    rng = np.random.default_rng(5)
    w = (rng.standard_normal(n) * 0.02).astype(np.float32)
    g = nm.bf16_bits_from_f32((np.sign(rng.standard_normal(n)) * 1e-2).astype(np.float32))
    sc = nm.AdamScalars(1e-3, 1)
    w1, m1, v1, p1 = nm.adam_update(w, np.zeros(n, np.float32), np.zeros(n, np.float32), g, sc)
    gf = nm.f32_from_bf16_bits(g).astype(np.float64)
    # step 1: m_hat = g, v_hat = g^2 -> update = lr * g / (|g| + eps)
    expect = w.astype(np.float64) - 1e-3 * gf / (np.abs(gf) + 1e-8)
    assert np.max(np.abs(w1 - expect)) < 1e-8
    assert np.allclose(m1, 0.1 * gf, rtol=1e-6)
    assert np.allclose(v1, 0.05 * gf * gf, rtol=1e-5)
    assert np.array_equal(p1, nm.bf16_bits_from_f32(w1))
    # zero gradient with wd = 0 leaves weights unchanged
    z = np.zeros(n, np.uint16)
    w2, _, _, _ = nm.adam_update(w, np.zeros(n, np.float32), np.zeros(n, np.float32), z, sc)
    assert np.array_equal(w2, w)


def test_adam_scalars_reject_step0():
    with pytest.raises(ValueError, match="step must be >= 1"):
        nm.AdamScalars(1e-3, 0)


def test_grad_sq_sum_matches_fsum():
    rng = np.random.default_rng(6)
    g = nm.bf16_bits_from_f32((rng.standard_normal(50_000) * 1e-3).astype(np.float32))
    ref = math.fsum(float(x) ** 2 for x in nm.f32_from_bf16_bits(g))
    assert abs(nm.grad_sq_sum(g) - ref) <= 1e-12 * ref


@pytest.mark.parametrize("N", [3, 5, 6, 7, 9, 12])
def test_pack_non_power_of_two_matches_torch(N):
    """pack = RNE_bf16(fp32(g) * fp32(1/N)) (reading R4) pinned bit for bit to
    torch's own float32 multiply and bfloat16 conversion on 10^6 bf16 patterns
    drawn over every finite exponent, so products land in the normal range, the
    fp32-subnormal range (bf16 subnormals) and underflow to zero; +-inf stay
    inf.  It also equals torch's bf16 rounding of the double quotient g/N:
    for N < 2^15 the exact g/N of an 8-bit-mantissa g is at least 1/(2N)
    bf16-ulp away from a rounding tie, farther than fp32(1/N)'s 2^-16-ulp
    error can move it, so the two fp32 roundings never change the result
    (pack is the correctly rounded per-rank mean contribution).  A truncating
    cast (a plausible mistake) gives other bits on this input set."""
    rng = np.random.default_rng(100 + N)
    bits = rng.integers(0, 1 << 16, size=1_000_000, dtype=np.uint32).astype(np.uint16)
    bits = bits[(bits & 0x7F80) != 0x7F80]                      # finite
    tiny = (rng.integers(0, 0x0300, size=50_000, dtype=np.uint32).astype(np.uint16)
            | (rng.integers(0, 2, size=50_000).astype(np.uint16) << 15))   # |g| < 2^-120
    bits = np.concatenate([bits, tiny, np.uint16([0x7F80, 0xFF80, 0x0000, 0x8000, 0x0001, 0x8001])])
    g = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).float()
    alpha = torch.tensor(np.float32(1.0 / N))
    prod = g * alpha
    ref = prod.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = nm.pack(bits, 1.0 / N)
    assert np.array_equal(got, ref)
    f = nm.f32_from_bf16_bits(got)
    assert (np.abs(f[np.isfinite(f)]) < np.float32(2.0 ** -126)).sum() > 1000    # subnormal results covered
    g64 = nm.f32_from_bf16_bits(bits).astype(np.float64) / N
    dbl = torch.from_numpy(g64).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(dbl, ref)
    trunc = (prod.numpy().view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    assert not np.array_equal(trunc, ref)
