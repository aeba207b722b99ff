"""ORACLE — test infrastructure only, never the product path.

CPU restatement of the block-buffer slot mapping.
The reference has no BlockStore; SPEC.md:550-553 and 568-576 define it:
a slice-accessed tensor gets a BlockStore whose block extent along a dim is
"determined by the largest slice access to the tensor", point-accessed
tensors a PointStore.  The B200 executor's storage for a tensor is one of

  * the full box (canonical C layout over the domain): slot of t = t;
  * folded along a loop dim (produced and consumed within one iteration,
    executor.find_folds): slot = 0;
  * a ring of two time blocks of bs steps (swap.py: a swap-managed
    activation of a time-blocked acting recurrence): step t of block
    kb = t // bs lives in ring row (kb mod 2) * bs + t mod bs.

Parity for this is unpinned by the reference (no test exists there), so
this module is the pin: tests/test_slots.py checks the executor's view
arithmetic (swap.adjust_views) against `ring_row` on every point, and the
device ring contents after a swapped run against the host copy.
"""

from __future__ import annotations


def ring_row(t: int, bs: int, nslots: int = 2) -> int:
    """Storage row of time step t in a ring of `nslots` blocks of bs steps."""
    kb = t // bs
    return (kb % nslots) * bs + (t - kb * bs)


def storage_row(t: int, kind: str, bs: int = 0) -> int:
    """Row of step t along a tensor's time dim for each storage kind."""
    if kind == "full":
        return t
    if kind == "folded":
        return 0
    if kind == "ring":
        return ring_row(t, bs)
    raise ValueError(kind)


def block_extent(slices, extent: int) -> int:
    """SPEC select_storage: the block extent along a dim is the largest slice
    access; `slices` = [(lo, hi)] evaluated windows (half-open, clipped to
    [0, extent)).  No slice access: a point store (extent 1)."""
    best = 1 if not slices else 0
    for lo, hi in slices:
        lo, hi = max(0, lo), min(extent, hi)
        best = max(best, hi - lo)
    return best
