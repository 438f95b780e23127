"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This module holds NO arithmetic of the PaRO method: it only assembles bit
patterns from a counter-based hash.  The CUDA side implements the identical
generator (synth_grad_kernel / init_range_kernel in
paper_2310_06003_b200/csrc/kernels.cu); a GPU test checks the two produce the
same bits.

Generator (DESIGN.md §5 "Input recipe"):

    splitmix64(x): x += 0x9E3779B97F4A7C15
                   z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9
                   z = (z ^ (z >> 27)) * 0x94D049BB133111EB
                   return z ^ (z >> 31)
    key(seed, tag, rank, step) = splitmix64(splitmix64(seed ^ tag) ^ ((rank << 32) | step))
    h_i = splitmix64(key ^ i)                     (i = flat element index)

    gradient (bf16 bits): sign = h >> 63, exponent = 114 + (h >> 8) % 5,
        mantissa = (h >> 16) & 0x7F        -> |g| in [2^-13, 2^-8), sigma ~ 1e-3
    master (fp32 bits):   sign = h >> 63, exponent = 119 + (h >> 8) % 5,
        mantissa = h & 0x7FFFFF            -> |w| in [2^-8, 2^-3), typical ~0.03

Both are exactly representable by construction (no rounding anywhere).
"""
from __future__ import annotations

import numpy as np

U64 = np.uint64
GOLDEN = U64(0x9E3779B97F4A7C15)
MIX1 = U64(0xBF58476D1CE4E5B9)
MIX2 = U64(0x94D049BB133111EB)

TAG_GRAD = 0x4752414400000000  # "GRAD"
TAG_MASTER = 0x4D41535400000000  # "MAST"
SEED = 1234


def splitmix64(x):
    x = np.asarray(x, dtype=U64)
    with np.errstate(over="ignore"):
        x = x + GOLDEN
        z = (x ^ (x >> U64(30))) * MIX1
        z = (z ^ (z >> U64(27))) * MIX2
    return z ^ (z >> U64(31))


def key(seed, tag, rank, step):
    k0 = splitmix64(np.array([np.uint64(seed) ^ np.uint64(tag)], dtype=U64))
    ctr = (np.uint64(rank) << U64(32)) | np.uint64(step)
    return int(splitmix64(k0 ^ ctr)[0])


def _hash(k, start, n):
    idx = np.arange(start, start + n, dtype=U64)
    return splitmix64(idx ^ U64(k))


def grad_bits(rank, step, start, n, seed=SEED):
    """bf16 bit patterns of rank `rank`'s gradient at `step` for flat indices [start, start+n)."""
    h = _hash(key(seed, TAG_GRAD, rank, step), start, n)
    sign = (h >> U64(63)).astype(np.uint16)
    expo = (U64(114) + (h >> U64(8)) % U64(5)).astype(np.uint16)
    mant = ((h >> U64(16)) & U64(0x7F)).astype(np.uint16)
    return ((sign << np.uint16(15)) | (expo << np.uint16(7)) | mant).astype(np.uint16)


def master_f32(start, n, seed=SEED, rank=0):
    """fp32 initial master weights for flat indices [start, start+n)."""
    h = _hash(key(seed, TAG_MASTER, rank, 0), start, n)
    sign = (h >> U64(63)).astype(np.uint32)
    expo = (U64(119) + (h >> U64(8)) % U64(5)).astype(np.uint32)
    mant = (h & U64(0x7FFFFF)).astype(np.uint32)
    return ((sign << np.uint32(31)) | (expo << np.uint32(23)) | mant).view(np.float32)


# ----------------------------------------------------------------- edge inputs
def edge_grad_bits(kind, n, rank=0, step=1, seed=SEED):
    """Edge-case gradients (bf16 bits): zeros, small integers, specials, near-max."""
    if kind == "zeros":
        return np.zeros(n, np.uint16)
    h = _hash(key(seed, TAG_GRAD ^ 0xE, rank, step), 0, n)
    if kind == "smallint":       # integers in [-3, 3]: exact in any summation order
        vals = ((h >> U64(20)) % U64(7)).astype(np.int64) - 3
        f = vals.astype(np.float32)
        return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    if kind == "nearmax":        # exponent 253/254: sums overflow to inf
        sign = (h >> U64(63)).astype(np.uint16)
        expo = (U64(253) + (h >> U64(8)) % U64(2)).astype(np.uint16)
        mant = ((h >> U64(16)) & U64(0x7F)).astype(np.uint16)
        return ((sign << np.uint16(15)) | (expo << np.uint16(7)) | mant).astype(np.uint16)
    if kind == "specials":       # regular gradients with +inf / -inf / NaN injected
        g = grad_bits(rank, step, 0, n, seed)
        sel = (h >> U64(40)) % U64(997)
        g = np.where(sel == 1, np.uint16(0x7F80), g)
        g = np.where(sel == 2, np.uint16(0xFF80), g)
        g = np.where(sel == 3, np.uint16(0x7FC0), g)
        return g.astype(np.uint16)
    raise ValueError(kind)


# ----------------------------------------------------------------- model shapes
def llama_ffn(d):
    """FFN hidden size 256 * ceil((8d/3) / 256) (LLaMA convention)."""
    h = int(2 * 4 * d / 3)
    return 256 * ((h + 255) // 256)


LLAMA = {"7B": (4096, 32), "13B": (5120, 40), "30B": (6656, 60), "65B": (8192, 80)}


def llama_param_sizes(name, vocab=32000):
    """Per-tensor element counts of a LLaMA-style model, in declaration order."""
    d, L = LLAMA[name]
    f = llama_ffn(d)
    sizes = [vocab * d]
    for _ in range(L):
        sizes += [d * d, d * d, d * d, d * d, f * d, d * f, f * d, d, d]
    sizes += [d, vocab * d]
    return sizes


def ragged_param_sizes():
    """Small ragged list exercising padding and unaligned parameter starts."""
    return [3, 64, 100, 7, 512, 1, 4096 + 5]


# ----------------------------------------------------------------- padded flat layouts
def grad_flat(rank, step, psi_pad, real, seed=SEED):
    """Gradient bits over a flat layout of psi_pad elements whose real (non-padding)
    ranges are `real` [(begin, end), ...]: element i carries grad_bits at index i,
    padding is zero.  For the dense layout real = [(0, psi)]; with layer-aligned
    buckets every bucket has its own padded tail.  (The library's generator writes
    the same bits: paro_synth_grads.)"""
    out = np.zeros(psi_pad, np.uint16)
    for a, e in real:
        if e > a:
            out[a:e] = grad_bits(rank, step, a, e - a, seed)
    return out


def master_flat(psi_pad, real, seed=SEED):
    """Initial fp32 masters over a padded flat layout (zero on the padding)."""
    out = np.zeros(psi_pad, np.float32)
    for a, e in real:
        if e > a:
            out[a:e] = master_f32(a, e - a, seed)
    return out
