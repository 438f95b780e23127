"""PaRO strategy space (oracle; test infrastructure only).

Three sharding states per model state, ordered by granularity
N (no sharding) < I (intra-group) < G (global)  (§3.1.1).
A strategy is a 3-letter code over {N, I, G} in P/G/OS order (Table 1,
P:267 "P/G/OS represents the combination of sharding strategies").
27 codes exist; Principle 1 keeps those with S_P >= S_OS and
S_G >= S_OS, leaving the 14 rows of Table 1.
"""
from __future__ import annotations

import itertools

LEVELS = "NIG"
RANK = {"N": 0, "I": 1, "G": 2}

# Table 1 row labels, in the paper's order.
TABLE1_ROWS = ["NNN", "NNI", "NNG", "NII", "NIG", "NGG", "INI", "ING",
               "III", "IIG", "IGG", "GNG", "GIG", "GGG"]

# Table 1 recommendation matrix, columns Psi'=Psi, Psi'>=Psi/6, Psi'<Psi/6, PEFT
# (check mark = True).  Advisory only: it does not change what a step computes.
TABLE1_MATRIX = {
    "NNN": (1, 1, 1, 1), "NNI": (1, 1, 1, 1), "NNG": (1, 1, 1, 0),
    "NII": (1, 1, 1, 0), "NIG": (1, 1, 1, 0), "NGG": (1, 1, 1, 0),
    "INI": (0, 0, 0, 1), "ING": (0, 1, 1, 0), "III": (0, 0, 1, 0),
    "IIG": (1, 1, 0, 0), "IGG": (1, 1, 1, 0), "GNG": (0, 1, 1, 1),
    "GIG": (0, 1, 1, 0), "GGG": (1, 1, 1, 0),
}

NAMED = {"NNN": "DDP", "NNG": "ZeRO-1", "NGG": "ZeRO-2", "III": "MiCS", "GGG": "ZeRO-3"}


class StrategyError(ValueError):
    pass


def parse(code: str):
    """'IIG' -> ('I', 'I', 'G').  Error strings follow S:63."""
    if not isinstance(code, str) or len(code) != 3:
        raise StrategyError("strategy code must have 3 characters")
    for i, ch in enumerate(code):
        if ch not in LEVELS:
            raise StrategyError(f"invalid shard level '{ch}' at position {i + 1}")
    return code[0], code[1], code[2]


def satisfies_principle1(code: str) -> bool:
    """S_P >= S_OS and S_G >= S_OS in the paper's granularity order.

    Granularity runs coarse to fine N > I > G, so the condition says
    OS is sharded at least as finely as P and G: RANK[OS] >= RANK[P], RANK[G]
    with RANK N=0, I=1, G=2.
    """
    p, g, o = parse(code)
    return RANK[o] >= RANK[p] and RANK[o] >= RANK[g]


def validate(code: str):
    """Parse and reject codes that violate Principle 1 (reading R22)."""
    p, g, o = parse(code)
    if not satisfies_principle1(code):
        raise StrategyError(
            f"strategy '{code}' violates Principle 1 (S_P>=S_OS and S_G>=S_OS)")
    return p, g, o


def enumerate_all():
    """All 27 codes, lexicographic in N<I<G per position."""
    return ["".join(t) for t in itertools.product(LEVELS, repeat=3)]


def paro_strategies():
    """The 14 Principle-1 codes, in enumeration order."""
    return [c for c in enumerate_all() if satisfies_principle1(c)]


def divisor(level: str, N: int, M: int) -> int:
    """Residency divisor of a level: N -> 1, I -> M, G -> N."""
    return {"N": 1, "I": M, "G": N}[level]


def validate_cluster(n_gpus: int, group_size: int):
    """(N, M) -> (N, M, g); error string follows S:73."""
    if n_gpus < 1 or group_size < 1:
        raise StrategyError("n_gpus and group_size must be >= 1")
    if n_gpus % group_size != 0:
        raise StrategyError("group_size must divide n_gpus")
    return n_gpus, group_size, n_gpus // group_size
