"""Multi-rank decomposition of a batched-mode batch (host logic, numpy only).

The batched semi-parallel extension (no reference counterpart,
SPEC.md:321) splits every batch -- a contiguous slice of the visit order
(engine.py:177-181) -- across the ranks of a process group.  Every rank holds
the whole (replicated) object and probes; the object update of a batch needs
the numerators/denominators summed over ALL of the batch's positions.

Instead of all-reducing the canvas band the batch touches, the batch is split
spatially and the canvas rows are owned:

  1. shares: the batch's positions sorted by anchor row (stable), cut into
     ``world`` contiguous runs (``batch_slice`` sizes) -- each rank's positions
     cover a compact row band [lo_r, hi_r) (hi_r = its last anchor row + W);
  2. ownership: rank r owns rows [lo_r, lo_{r+1}) (the last rank up to its
     hi), so the owned ranges tile the batch's band without overlap;
  3. halo transfers: rank r's accumulator rows that fall in another rank's
     owned range (at most about W rows past lo_{r+1}) are sent to that owner,
     which adds them in rank order -- the only reduction traffic;
  4. each owner applies the object update to its rows and the updated rows are
     all-gathered, so every rank ends with the same canvas.

The row numbers are canvas rows (anchor row minus the canvas origin).
"""

from __future__ import annotations

import numpy as np


def batch_slice(n_batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous share [lo, hi) of a batch of n_batch positions for one rank."""
    base, extra = divmod(n_batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def rank_shares(anchor_rows: np.ndarray, world: int) -> list[np.ndarray]:
    """Indices into the batch of every rank's share (sorted by anchor row,
    stable, so equal rows keep batch order)."""
    rows = np.asarray(anchor_rows)
    order = np.argsort(rows, kind="stable")
    return [order[slice(*batch_slice(len(rows), r, world))] for r in range(world)]


def row_bands(anchor_rows: np.ndarray, shares, window: int, height: int) -> list[tuple[int, int]]:
    """[lo, hi) canvas rows each rank's positions touch; (0, 0) for an empty share."""
    rows = np.asarray(anchor_rows)
    out = []
    for sh in shares:
        if len(sh) == 0:
            out.append((0, 0))
            continue
        lo = max(0, int(rows[sh].min()))
        hi = min(height, int(rows[sh].max()) + window)
        out.append((lo, max(lo, hi)))
    return out


def ownership(bands) -> list[tuple[int, int]]:
    """Owned row ranges: rank r owns [lo_r, next non-empty lo), the last
    non-empty rank up to the band end; empty shares own nothing."""
    live = [r for r, (lo, hi) in enumerate(bands) if hi > lo]
    owns = [(0, 0)] * len(bands)
    end = max((bands[r][1] for r in live), default=0)
    for k, r in enumerate(live):
        lo = bands[r][0]
        hi = bands[live[k + 1]][0] if k + 1 < len(live) else end
        owns[r] = (lo, max(lo, hi))
    return owns


def halo_transfers(bands, owns) -> list[tuple[int, int, int, int]]:
    """(src, dst, row_lo, row_hi): accumulator rows src computed that dst owns,
    in (dst, src) order -- the order the owner adds them."""
    out = []
    for dst, (olo, ohi) in enumerate(owns):
        if ohi <= olo:
            continue
        for src, (lo, hi) in enumerate(bands):
            if src == dst or hi <= lo:
                continue
            a, b = max(lo, olo), min(hi, ohi)
            if b > a:
                out.append((src, dst, a, b))
    return out
