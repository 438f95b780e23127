"""Numerics of the PaRO sync + update step (oracle; test infrastructure only).

The paper fixes the widths: parameters and gradients are 2-byte, optimizer
state is 12 bytes per trainable parameter (fp32 master + m + v) under
"mainstream mixed precision training using Adam" (§3.1.2).  It does
not fix rounding points or reduction order; this module states the readings
used (R2, R5-R7):

* bf16 values are carried as uint16 bit patterns; conversion fp32 -> bf16 is
  IEEE round-to-nearest-even on the bit pattern (R2);
* one reduction hop is  a (+) b = RNE_bf16(fp32(a) + fp32(b))  -- an fp32 add
  followed by one rounding to bf16, not a correctly rounded bf16 add (R2);
* a ring reduce-scatter over k members that delivers block c to member c
  accumulates in the order R_k(c; y) = (((y[c+1] (+) y[c+2]) (+) ...) (+) y[c-1]) (+) y[c]
  (indices mod k), the order a ring with member q sending to q+1 produces (R2);
* Adam is the AdamW form with every fp32 operation rounded once, no fused
  multiply-add, host scalars formed in double and rounded once (R5-R7).
"""
from __future__ import annotations

import math

import numpy as np

F32 = np.float32


# ---------------------------------------------------------------- bf16 <-> fp32
def bf16_bits_from_f32(x) -> np.ndarray:
    """fp32 -> bf16 bit pattern, round-to-nearest-even (R2; P:225 2-byte P/G).

    Overflow rounds to +-inf as IEEE requires; NaN maps to a quiet NaN of the
    same sign (NaN payloads are not compared, R9).
    """
    x = np.asarray(x, dtype=F32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        sign = ((u >> np.uint64(16)) & np.uint64(0x8000)).astype(np.uint16)
        r = np.where(nan, sign | np.uint16(0x7FC0), r)
    return r.astype(np.uint16)


def f32_from_bf16_bits(b) -> np.ndarray:
    """bf16 bit pattern -> fp32 (exact: bf16 is the top half of fp32)."""
    b = np.asarray(b, dtype=np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(F32)


def round_bf16(x) -> np.ndarray:
    """fp32 -> nearest-even bf16, returned as fp32 values."""
    return f32_from_bf16_bits(bf16_bits_from_f32(x))


# ---------------------------------------------------------------- reduction
def hop(a_bits, b_bits) -> np.ndarray:
    """One reduction hop on bf16 bit patterns: RNE_bf16(fp32(a) + fp32(b)) (R2)."""
    return bf16_bits_from_f32(f32_from_bf16_bits(a_bits) + f32_from_bf16_bits(b_bits))


def canonical_fold(ys, c: int, op=hop):
    """R_k(c; y) = (((y[c+1] op y[c+2]) op ...) op y[c-1]) op y[c], indices mod k.

    ``ys`` is a sequence of k equally shaped arrays (one per ring member);
    ``c`` is the member that owns the result.  R_1(0; y) = y[0].
    This is the accumulation order of a ring reduce-scatter in which member q
    sends to q+1 ("each GPU sequentially transfers its shard of data to
    the next GPU"); chosen as the canonical order in R2.
    """
    k = len(ys)
    if k == 1:
        return np.array(ys[0], copy=True)
    acc = ys[(c + 1) % k]
    for t in range(2, k + 1):
        acc = op(acc, ys[(c + t) % k])
    return acc


def hop_f32(a, b) -> np.ndarray:
    """One reduction hop of the fp32 wire (SURVEY reading A3, wire_dtype = 1):
    a plain IEEE fp32 addition of fp32 partials, no bf16 rounding."""
    return (np.asarray(a, dtype=F32) + np.asarray(b, dtype=F32)).astype(F32)


def pack_f32(grad_bits, alpha: float) -> np.ndarray:
    """Pre-scaling on the fp32 wire: x = fp32(g) * fp32(alpha), one fp32
    rounding (exact for power-of-two N), kept in fp32 (reading A3/A4)."""
    with np.errstate(over="ignore", invalid="ignore"):
        return (f32_from_bf16_bits(grad_bits) * F32(alpha)).astype(F32)


def pack(grad_bits, alpha: float) -> np.ndarray:
    """Gradient pre-scaling before the reduction: x = RNE_bf16(fp32(g) * fp32(alpha)).

    alpha = 1/N averages over the N data-parallel ranks (replicas
    average their gradients; placement at pack time is reading R4).
    """
    return bf16_bits_from_f32(f32_from_bf16_bits(grad_bits) * F32(alpha))


# ---------------------------------------------------------------- Adam
class AdamScalars:
    """Per-step host scalars of canonical Adam (R5, R6).

    The hyperparameters are fp32 values (lr, beta1, beta2, eps, weight_decay,
    loss_scale are each rounded to fp32 first, as an fp32 optimizer API
    receives them); every derived scalar is then computed in double precision
    from those fp32 values and rounded once to fp32:
    step_size = lr / (1 - beta1^t);  bc2s = sqrt(1 - beta2^t);
    decay = 1 - lr * weight_decay;  s_g = 1 / loss_scale (unscale, R4).
    With gradient accumulation over s micro-batches the accumulated sum is
    turned into the mini-batch mean here: s_g = 1 / (loss_scale * s) (R27);
    without pre-division (predivide = 0) the rank average too:
    s_g = 1 / (loss_scale * s * N).
    """

    def __init__(self, lr, step, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0,
                 loss_scale=1.0, clip_coef=1.0, accum_steps=1, post_div=1):
        if step < 1:
            raise ValueError("step must be >= 1")
        if accum_steps < 1:
            raise ValueError("accum_steps must be >= 1")
        f = lambda x: float(F32(x))
        lr, b1, b2 = f(lr), f(beta1), f(beta2)
        weight_decay, loss_scale, eps = f(weight_decay), f(loss_scale), f(eps)
        self.b1 = F32(b1)
        self.omb1 = F32(1.0 - b1)
        self.b2 = F32(b2)
        self.omb2 = F32(1.0 - b2)
        self.step_size = F32(lr / (1.0 - b1 ** step))
        self.bc2s = F32(math.sqrt(1.0 - b2 ** step))
        self.eps = F32(eps)
        self.wd = float(weight_decay)
        self.decay = F32(1.0 - lr * float(weight_decay))
        # post_div = N when the 1/N average is not applied at pack time
        # (predivide = 0): the sum is averaged here, in the same rounding
        self.s_g = F32((1.0 / (float(loss_scale) * accum_steps * post_div)) * float(clip_coef))


def adam_update(master, m, v, ghat_bits, sc: AdamScalars):
    """Canonical fp32 Adam on one owned shard (P:225 mixed-precision Adam; R5-R7).

    Inputs: fp32 arrays master, m, v (not modified) and the reduced gradient
    as bf16 bits (uint16; bf16 wire) or as fp32 values (float32; fp32 wire).  Returns (master', m', v', param_bf16_bits).  Every line is
    one IEEE fp32 operation rounded to nearest; NumPy float32 array
    arithmetic never contracts to FMA.

        w  = w * decay                  (only when weight_decay != 0)
        gr = fp32(g_hat) * s_g
        m  = b1 * m + omb1 * gr
        v  = b2 * v + omb2 * (gr * gr)
        d  = sqrt(v) / bc2s + eps
        w  = w - step_size * (m / d)
        p  = RNE_bf16(w)
    """
    w = np.asarray(master, dtype=F32)
    m = np.asarray(m, dtype=F32)
    v = np.asarray(v, dtype=F32)
    with np.errstate(invalid="ignore", over="ignore"):   # non-finite inputs propagate (R9)
        if sc.wd != 0.0:
            w = w * sc.decay
        gr = _ghat_f32(ghat_bits) * sc.s_g
        m2 = sc.b1 * m + sc.omb1 * gr
        v2 = sc.b2 * v + sc.omb2 * (gr * gr)
        d = np.sqrt(v2) / sc.bc2s + sc.eps
        w2 = w - sc.step_size * (m2 / d)
    return w2.astype(F32), m2.astype(F32), v2.astype(F32), bf16_bits_from_f32(w2)


def _ghat_f32(ghat):
    """g_hat as fp32 values: bf16 bit patterns are widened exactly, fp32 kept."""
    ghat = np.asarray(ghat)
    return ghat.astype(F32) if ghat.dtype == F32 else f32_from_bf16_bits(ghat)


def grad_sq_sum(ghat_bits, s_g=F32(1.0)) -> float:
    """sum_i (fp32(g_hat_i) * s_g)^2 in fp64 (norm reporting, R8)."""
    gr = (_ghat_f32(ghat_bits) * F32(s_g)).astype(np.float64)
    return float(np.sum(gr * gr))
