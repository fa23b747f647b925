"""Conditional-swap strategy names (reference `swaps.py:18`, codes 0..8).

On the CPU the nine styles are different instruction sequences with one
observable contract: after the swap the pair is ordered by key, items move as
whole units, and equal keys never exchange (reference `netsort_core.h:28-31`,
pinned by acceptance gate A04).  On sm_100a every style compiles to the same
predicate + SEL / IMNMX sequence, so the strategy is validated and recorded but
selects no different device code.
"""

STRATEGIES = ("ISwp", "TCOp", "Tie", "JXhg", "4Cm", "4CmS", "6Cm", "2CPm", "2CPp")
SWAP_CODES = {name: code for code, name in enumerate(STRATEGIES)}
_BRANCH_FREE = frozenset({"TCOp", "4Cm", "4CmS", "6Cm", "2CPm", "2CPp"})


def strategy_is_branch_free(strategy: str) -> bool:
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown swap strategy {strategy!r}")
    return strategy in _BRANCH_FREE
