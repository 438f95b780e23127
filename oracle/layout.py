"""Flat layout, buckets and the PaRO shard map (oracle; test infrastructure only).

Notation: N GPUs, groups of M, g = N/M groups, Psi parameters.
Rank r belongs to group j = r div M at position p = r mod M (R20).

Reading R1 (position-major nested shard map; the paper is silent, Fig 4 is
illegible at P:389): inside a bucket of B_b elements

* intra-group chunk of position p:  [p*B_b/M, (p+1)*B_b/M)
* global segment of rank (j, p):    k = p*g + j,  [k*B_b/N, (k+1)*B_b/N)

so the global segment of (j, p) lies inside the intra chunk of p.  That is the
only contiguous layout in which the OS=G shard is a sub-range of the P=I shard
(needed by PaRO-IGG/IIG: "model parameter shards are obtained from other
groups through an inter-group all-gather").

Reading R21 (padding): each bucket is a multiple of N*64 elements; Psi is
zero-padded to Psi_pad = ceil(Psi / (N*64)) * N*64.

Layer-aligned buckets (NEXT-2, "obtains a complete replica of model
parameters through the intra-group all-gather" layer by layer in the forward /
backward pass): with `groups` (tensor indices at which a bucket starts; the
first is 0) bucket k holds exactly tensors [groups[k], groups[k+1]), laid out
densely and zero-padded at its end to a multiple of N*64, so one bucket's
gather is one layer group's parameters.  Psi_pad is then the sum of the padded
group sizes and the padding lies at the end of every bucket.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .strategy import divisor, validate_cluster

QUANTUM = 64  # elements per shard granule (R21)


def _ceil_div(a, b):
    return -(-a // b)


@dataclass
class Layout:
    param_sizes: list
    N: int
    M: int
    bucket_elems: int
    groups: list = None                      # tensor indices starting a bucket (layer-aligned buckets)
    g: int = field(init=False)
    psi: int = field(init=False)
    psi_pad: int = field(init=False)
    B: int = field(init=False)
    buckets: list = field(init=False)        # [(start, size)]
    param_offsets: list = field(init=False)  # flat start of each param

    def __post_init__(self):
        self.N, self.M, self.g = validate_cluster(self.N, self.M)
        if any(int(s) < 0 for s in self.param_sizes):
            raise ValueError("param sizes must be >= 0")
        unit = self.N * QUANTUM
        self.psi = int(sum(int(s) for s in self.param_sizes))
        if self.groups is not None:
            self._grouped(unit)
            return
        self.psi_pad = _ceil_div(self.psi, unit) * unit
        self.B = max(unit, (int(self.bucket_elems) // unit) * unit)
        offs, o = [], 0
        for s in self.param_sizes:
            offs.append(o)
            o += int(s)
        self.param_offsets = offs
        self.buckets = []
        self.real = []
        start = 0
        while start < self.psi_pad:
            size = min(self.B, self.psi_pad - start)
            self.buckets.append((start, size))
            self.real.append((start, min(start + size, self.psi)))
            start += size

    def _grouped(self, unit):
        n = len(self.param_sizes)
        gs = [int(x) for x in self.groups]
        if not gs or gs[0] != 0 or any(b <= a for a, b in zip(gs, gs[1:])) or gs[-1] >= max(n, 1):
            raise ValueError("bucket groups must start at tensor 0 and increase strictly below n_params")
        bounds = gs + [n]
        offs, o = [], 0
        self.buckets, self.real = [], []
        for k in range(len(gs)):
            start = o
            for t in range(bounds[k], bounds[k + 1]):
                offs.append(o)
                o += int(self.param_sizes[t])
            size = _ceil_div(o - start, unit) * unit
            if size:
                self.buckets.append((start, size))
                self.real.append((start, o))
            o = start + size
        self.param_offsets = offs
        self.psi_pad = o
        self.B = max([unit] + [n for _, n in self.buckets])

    def expand(self, x, fill=0):
        """Place a per-tensor concatenation (length Psi, declaration order) into
        the flat layout (length Psi_pad), `fill` on the padding."""
        x = np.asarray(x)
        out = np.full(self.psi_pad, fill, dtype=x.dtype)
        o = 0
        for off, sz in zip(self.param_offsets, self.param_sizes):
            out[off:off + int(sz)] = x[o:o + int(sz)]
            o += int(sz)
        return out

    # -- rank geometry -------------------------------------------------------
    def rank_jp(self, r):
        return r // self.M, r % self.M

    def rank_of(self, j, p):
        return j * self.M + p

    # -- residency ranges (flat element indices) ------------------------------
    def chunk(self, b, p):
        """Intra-group chunk of position p in bucket b (R1)."""
        s, n = self.buckets[b]
        c = n // self.M
        return s + p * c, s + (p + 1) * c

    def segment(self, b, k):
        """Global segment k of bucket b (R1)."""
        s, n = self.buckets[b]
        c = n // self.N
        return s + k * c, s + (k + 1) * c

    def seg_index(self, r):
        j, p = self.rank_jp(r)
        return p * self.g + j

    def residency(self, level, r, b):
        """Flat range a rank holds of a state at `level` in bucket b."""
        j, p = self.rank_jp(r)
        s, n = self.buckets[b]
        if level == "N":
            return s, s + n
        if level == "I":
            return self.chunk(b, p)
        if level == "G":
            return self.segment(b, self.seg_index(r))
        raise ValueError(level)

    def shard_numel(self, level):
        return self.psi_pad // divisor(level, self.N, self.M)

    def shard_ranges(self, level, r):
        """Bucket-major list of flat ranges making up rank r's shard buffer."""
        return [self.residency(level, r, b) for b in range(len(self.buckets))]

    def owner_segment(self, i):
        """(j, p) owning flat element i under the global-segment map (R1)."""
        for b, (s, n) in enumerate(self.buckets):
            if s <= i < s + n:
                k = (i - s) // (n // self.N)
                p, j = divmod(k, self.g)
                return j, p
        raise IndexError(i)
