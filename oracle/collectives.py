"""Round-synchronous collective simulators (oracle; test infrastructure only).

All N ranks live in one process (the approach of S:339 "Deterministic
in-process simulation of a grouped GPU cluster").  A bucket is split
into N equal segments; segment k = p*g + j belongs to rank (j, p) and the g
segments p*g .. p*g+g-1 form the intra-group chunk of position p (layout R1).

Every simulator works on real payloads with a caller-supplied combine
operator ``op`` (the bf16 hop of numerics.hop for the numerics contract,
integer addition for exact pins), and returns a Trace: the list of rounds,
each a list of messages (src_rank, dst_rank, units).  Link class of a message
is "inter" iff src and dst are in different groups.

Ring convention (R20): members are ordered ascending, member q sends to q+1.
A ring reduce-scatter delivers block c to member c with accumulation order
R_k(c; y) (numerics.canonical_fold, R2): the chain for block c starts at
member c+1 and ends at c.  A ring all-gather moves block (q - t) from q to q+1
in round t ("ring order is rank id ascending, wrapping").

Topologies
----------
flat ring     P:399 "each GPU sequentially transfers its shard of data to the next GPU"
two-step      P:148-149: intra RS then inter RS (AG: inter then intra)
HO-Ring       P:406-410 (Fig 4): intra and inter rings run concurrently, then an
              intra completion ring (AG); RS is the exact dual (R16, R17)
H-Ring        P:146-147: one leader per group for inter traffic
"""
from __future__ import annotations

import numpy as np


class Trace:
    def __init__(self, M):
        self.M = M
        self.rounds = []

    def extend(self, other_rounds):
        self.rounds.extend(other_rounds)

    def n_rounds(self):
        return len(self.rounds)

    def link(self, a, b):
        return "inter" if a // self.M != b // self.M else "intra"

    def sent(self, r):
        """[intra, inter] units sent by rank r over the whole trace."""
        out = [0, 0]
        for rnd in self.rounds:
            for (s, d, u) in rnd:
                if s == r:
                    out[0 if self.link(s, d) == "intra" else 1] += u
        return out

    def totals(self):
        tot = [0, 0]
        for rnd in self.rounds:
            for (s, d, u) in rnd:
                tot[0 if self.link(s, d) == "intra" else 1] += u
        return tot


def merge_concurrent(*round_lists):
    """Rings that run at the same time share round indices (HO-Ring overlap)."""
    n = max((len(r) for r in round_lists), default=0)
    out = [[] for _ in range(n)]
    for rl in round_lists:
        for t, msgs in enumerate(rl):
            out[t].extend(msgs)
    return out


def _cat(parts):
    return np.concatenate(parts) if len(parts) else np.zeros(0)


# ----------------------------------------------------------------- ring kernels
def ring_reduce_scatter(ranks, contrib, op, defer_last=False):
    """Ring RS over members ranks[0..k-1].

    contrib(q, c) -> member q's contribution to block c (array).
    Returns (result, rounds): result[q] is block q reduced in order R_k(q; .);
    with defer_last the final local combine at the owner is left to the caller
    and result[q] = (received_partial_or_None, ) so the owner can add a value
    that becomes ready later (HO-Ring phase 2, R16).
    """
    k = len(ranks)
    rounds = []
    if k == 1:
        return ({0: (None,)} if defer_last else {0: contrib(0, 0)}), rounds
    # round 0: member q sends its own contribution to block q-1 (chain start c+1 = q)
    send = {q: contrib(q, (q - 1) % k) for q in range(k)}
    result = {}
    for t in range(k - 1):
        msgs = [(ranks[q], ranks[(q + 1) % k], int(send[q].size)) for q in range(k)]
        rounds.append(msgs)
        recv = {(q + 1) % k: send[q] for q in range(k)}
        nxt = {}
        for q in range(k):
            c = (q - t - 2) % k          # block whose chain reaches member q at round t
            if t == k - 2:
                assert c == q
                result[q] = (recv[q],) if defer_last else op(recv[q], contrib(q, q))
            else:
                nxt[q] = op(recv[q], contrib(q, c))
        send = nxt
    return result, rounds


def ring_all_gather(ranks, blocks):
    """Ring AG: member q starts with blocks[q]; returns (have[q] = list of k blocks, rounds)."""
    k = len(ranks)
    have = {q: {q: blocks[q]} for q in range(k)}
    rounds = []
    for t in range(k - 1):
        msgs = []
        for q in range(k):
            c = (q - t) % k
            have[(q + 1) % k][c] = have[q][c]
            msgs.append((ranks[q], ranks[(q + 1) % k], int(np.asarray(have[q][c]).size)))
        rounds.append(msgs)
    return {q: [have[q][c] for c in range(k)] for q in range(k)}, rounds


# ----------------------------------------------------------------- geometry
class Geometry:
    """(N, M, g) with rank r = j*M + p and segment k = p*g + j (R1, R20)."""

    def __init__(self, N, M):
        assert N % M == 0
        self.N, self.M, self.g = N, M, N // M

    def r(self, j, p):
        return j * self.M + p

    def jp(self, r):
        return divmod(r, self.M)

    def seg(self, j, p):
        return p * self.g + j

    def chunk_segs(self, p):
        return [p * self.g + jj for jj in range(self.g)]


# ----------------------------------------------------------------- reduce-scatter
def rs_flat_ring(geo, X, op):
    """Flat ring RS over all N ranks in rank order; rank r keeps segment seg(r).

    X[r] = list of N segment arrays.  Returns (out[r] = segment, Trace).
    """
    N = geo.N
    own = [geo.seg(*geo.jp(r)) for r in range(N)]
    res, rounds = ring_reduce_scatter(list(range(N)), lambda q, c: X[q][own[c]], op)
    tr = Trace(geo.M)
    tr.extend(rounds)
    return {r: res[r] for r in range(N)}, tr


def rs_intra(geo, X, op):
    """RS_I: per group j, ring over positions; (j,p) keeps the chunk p partial.

    X[r] = list of N segments.  Returns (Y[r] = concatenated chunk partial, rounds).
    """
    g, M = geo.g, geo.M
    Y, all_rounds = {}, []
    for j in range(g):
        ranks = [geo.r(j, p) for p in range(M)]
        res, rounds = ring_reduce_scatter(
            ranks, lambda q, c, j=j: _cat([X[geo.r(j, q)][s] for s in geo.chunk_segs(c)]), op)
        for p in range(M):
            Y[geo.r(j, p)] = res[p]
        all_rounds.append(rounds)
    return Y, merge_concurrent(*all_rounds)


def rs_inter(geo, Y, op):
    """RS_E: per position p, ring over groups on chunk p; (j,p) keeps segment p*g+j.

    Y[r] = chunk-sized array (g segments).  Returns (out[r] = segment, rounds).
    """
    g, M = geo.g, geo.M
    out, all_rounds = {}, []
    for p in range(M):
        ranks = [geo.r(j, p) for j in range(g)]
        def contrib(q, c, p=p):
            y = Y[geo.r(q, p)]
            C = y.size // g
            return y[c * C:(c + 1) * C]
        res, rounds = ring_reduce_scatter(ranks, contrib, op)
        for j in range(g):
            out[geo.r(j, p)] = res[j]
        all_rounds.append(rounds)
    return out, merge_concurrent(*all_rounds)


def rs_two_step(geo, X, op):
    """Grouped two-step RS: RS_I then RS_E (Eq. 1)."""
    Y, r1 = rs_intra(geo, X, op)
    out, r2 = rs_inter(geo, Y, op)
    tr = Trace(geo.M)
    tr.extend(r1)
    tr.extend(r2)
    return out, tr, Y


def rs_ho_ring(geo, X, op):
    """HO-Ring reduce-scatter (dual of the all-gather, R16).

    Phase 1: per group j, intra ring RS of the foreign-group segments: block p'
      = segments p'*g + jj for jj != j  ((M-1) rounds of (g-1)C).
    Phase 2 (concurrent): (i) per position p, inter ring RS over groups; member
      jj contributes its group partial of segment p*g+x (from phase 1 for x != jj)
      and the owner adds its own-group partial last; (ii) per group, intra ring RS
      of the own-group segments ((M-1) rounds of C) producing that partial.
    Returns (out[r] = segment, Trace, own_partial) where own_partial[r] is
    the group-j partial of segment seg(r) (the intra-RS value kept for G = I).
    """
    g, M = geo.g, geo.M
    tr = Trace(M)
    # phase 1
    P1, ph1 = {}, []
    if g > 1:
        for j in range(g):
            ranks = [geo.r(j, p) for p in range(M)]
            foreign = [jj for jj in range(g) if jj != j]
            def contrib(q, c, j=j, foreign=foreign):
                return _cat([X[geo.r(j, q)][geo.seg(jj, c)] for jj in foreign])
            res, rounds = ring_reduce_scatter(ranks, contrib, op)
            for p in range(M):
                P1[geo.r(j, p)] = res[p]
            ph1.append(rounds)
        tr.extend(merge_concurrent(*ph1))
    # phase 2 (ii): intra RS of own-group segments
    S, ph2b = {}, []
    for j in range(g):
        ranks = [geo.r(j, p) for p in range(M)]
        res, rounds = ring_reduce_scatter(ranks, lambda q, c, j=j: X[geo.r(j, q)][geo.seg(j, c)], op)
        for p in range(M):
            S[geo.r(j, p)] = res[p]
        ph2b.append(rounds)
    # phase 2 (i): inter ring RS with deferred final add of the own-group partial
    out, ph2a = {}, []
    for p in range(M):
        ranks = [geo.r(j, p) for j in range(g)]
        def contrib(q, c, p=p):
            # member q (= group jj) contributes its group partial of segment p*g+c, c != q
            foreign = [jj for jj in range(g) if jj != q]
            blk = P1[geo.r(q, p)]
            C = blk.size // (g - 1)
            i = foreign.index(c)
            return blk[i * C:(i + 1) * C]
        res, rounds = ring_reduce_scatter(ranks, contrib, op, defer_last=True)
        for j in range(g):
            (recv,) = res[j]
            own = S[geo.r(j, p)]
            out[geo.r(j, p)] = own.copy() if recv is None else op(recv, own)
        ph2a.append(rounds)
    tr.extend(merge_concurrent(*(ph2a + ph2b)))
    return out, tr, S


def rs_canonical(geo, X, op):
    """Closed form of the hierarchical order (no rounds): for segment k = p*g + j,
    S_j' = R_M(p; X[(j',0..M-1)][k]) and g_hat = R_g(j; S_0..S_{g-1}) (R2)."""
    from .numerics import canonical_fold
    out = {}
    for r in range(geo.N):
        j, p = geo.jp(r)
        k = geo.seg(j, p)
        S = [canonical_fold([X[geo.r(jj, pp)][k] for pp in range(geo.M)], p, op)
             for jj in range(geo.g)]
        out[r] = canonical_fold(S, j, op)
    return out


# ----------------------------------------------------------------- all-gather
def ag_inter(geo, Z):
    """AG_E: per position p, ring over groups; (j,p) ends with chunk p (list of g segs)."""
    g, M = geo.g, geo.M
    out, all_rounds = {}, []
    for p in range(M):
        ranks = [geo.r(j, p) for j in range(g)]
        have, rounds = ring_all_gather(ranks, [Z[geo.r(j, p)] for j in range(g)])
        for j in range(g):
            out[geo.r(j, p)] = have[j]
        all_rounds.append(rounds)
    return out, merge_concurrent(*all_rounds)


def ag_intra(geo, Y):
    """AG_I: per group, ring over positions of chunk-sized blocks; (j,p) ends with all M chunks."""
    g, M = geo.g, geo.M
    out, all_rounds = {}, []
    for j in range(g):
        ranks = [geo.r(j, p) for p in range(M)]
        have, rounds = ring_all_gather(ranks, [Y[geo.r(j, p)] for p in range(M)])
        for p in range(M):
            out[geo.r(j, p)] = have[p]
        all_rounds.append(rounds)
    return out, merge_concurrent(*all_rounds)


def ag_flat_ring(geo, Z):
    """Flat ring AG over ranks in order; returns (segs[r] = dict seg -> array, Trace)."""
    N = geo.N
    have, rounds = ring_all_gather(list(range(N)), [Z[r] for r in range(N)])
    tr = Trace(geo.M)
    tr.extend(rounds)
    out = {r: {geo.seg(*geo.jp(c)): have[r][c] for c in range(N)} for r in range(N)}
    return out, tr


def ag_two_step(geo, Z):
    """AG_E then AG_I (H-Ring without a leader; the 2D two-step of P:148)."""
    A, r1 = ag_inter(geo, Z)
    Yc = {r: _cat(A[r]) for r in A}
    B, r2 = ag_intra(geo, Yc)
    tr = Trace(geo.M)
    tr.extend(r1)
    tr.extend(r2)
    out = {}
    for r in range(geo.N):
        d = {}
        for p, chunk in enumerate(B[r]):
            C = chunk.size // geo.g
            for jj in range(geo.g):
                d[geo.seg(jj, p)] = chunk[jj * C:(jj + 1) * C]
        out[r] = d
    return out, tr


def ag_ho_ring(geo, Z):
    """HO-Ring all-gather (Fig 4; R17).

    Phase A (concurrent, max(M-1, g-1) rounds): intra ring AG of own segment
    within the group and inter ring AG of own segment across groups at the
    same position ("transmits its own shards simultaneously through the intra-
    and inter-group communication rings").
    Phase B (M-1 rounds, only if g > 1): intra ring AG of each rank's g-1
    foreign-group segments ("an intra-group communication ring is executed to
    gather the remaining shards within the group").
    Returns (segs[r] = dict seg -> array, Trace).
    """
    g, M = geo.g, geo.M
    have = {r: {geo.seg(*geo.jp(r)): Z[r]} for r in range(geo.N)}
    intra_rounds, inter_rounds = [], []
    for j in range(g):
        ranks = [geo.r(j, p) for p in range(M)]
        h, rounds = ring_all_gather(ranks, [Z[geo.r(j, p)] for p in range(M)])
        for p in range(M):
            for pp in range(M):
                have[geo.r(j, p)][geo.seg(j, pp)] = h[p][pp]
        intra_rounds.append(rounds)
    for p in range(M):
        ranks = [geo.r(j, p) for j in range(g)]
        h, rounds = ring_all_gather(ranks, [Z[geo.r(j, p)] for j in range(g)])
        for j in range(g):
            for jj in range(g):
                have[geo.r(j, p)][geo.seg(jj, p)] = h[j][jj]
        inter_rounds.append(rounds)
    tr = Trace(M)
    tr.extend(merge_concurrent(*(intra_rounds + inter_rounds)))
    if g > 1:
        phB = []
        for j in range(g):
            ranks = [geo.r(j, p) for p in range(M)]
            foreign = [jj for jj in range(g) if jj != j]
            blocks = [_cat([have[geo.r(j, p)][geo.seg(jj, p)] for jj in foreign]) for p in range(M)]
            h, rounds = ring_all_gather(ranks, blocks)
            for p in range(M):
                for pp in range(M):
                    blk = h[p][pp]
                    C = blk.size // (g - 1)
                    for i, jj in enumerate(foreign):
                        have[geo.r(j, p)][geo.seg(jj, pp)] = blk[i * C:(i + 1) * C]
            phB.append(rounds)
        tr.extend(merge_concurrent(*phB))
    return have, tr


def ag_h_ring(geo, Z):
    """H-Ring all-gather with one leader (position 0) per group.

    Phase 1: intra ring AG of own segment (M-1 rounds of C).
    Phase 2: leaders run an inter ring AG of group blocks (g-1 rounds of M*C).
    Phase 3: ring broadcast of the (g-1) foreign group blocks from the leader
    through positions 1..M-1 (M-1 rounds of (g-1)*M*C).
    """
    g, M = geo.g, geo.M
    have = {r: {} for r in range(geo.N)}
    tr = Trace(M)
    ph1 = []
    for j in range(g):
        ranks = [geo.r(j, p) for p in range(M)]
        h, rounds = ring_all_gather(ranks, [Z[geo.r(j, p)] for p in range(M)])
        for p in range(M):
            for pp in range(M):
                have[geo.r(j, p)][geo.seg(j, pp)] = h[p][pp]
        ph1.append(rounds)
    tr.extend(merge_concurrent(*ph1))
    if g > 1:
        leaders = [geo.r(j, 0) for j in range(g)]
        blocks = [_cat([have[geo.r(j, 0)][geo.seg(j, pp)] for pp in range(M)]) for j in range(g)]
        h, rounds = ring_all_gather(leaders, blocks)
        for j in range(g):
            for jj in range(g):
                blk = h[j][jj]
                C = blk.size // M
                for pp in range(M):
                    have[geo.r(j, 0)][geo.seg(jj, pp)] = blk[pp * C:(pp + 1) * C]
        tr.extend(rounds)
        for t in range(M - 1):
            msgs = []
            for j in range(g):
                src, dst = geo.r(j, t), geo.r(j, t + 1)
                units = 0
                for jj in range(g):
                    if jj == j:
                        continue
                    for pp in range(M):
                        s = geo.seg(jj, pp)
                        have[dst][s] = have[src][s]
                        units += int(np.asarray(have[src][s]).size)
                msgs.append((src, dst, units))
            tr.rounds.append(msgs)
    return have, tr


def ho_rounds(N, M):
    """Closed-form HO-Ring round count: max(M-1, g-1) + (M-1)*[g>1] (R17)."""
    g = N // M
    return max(M - 1, g - 1) + (M - 1) * (1 if g > 1 else 0)
