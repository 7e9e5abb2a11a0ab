"""Multi-GPU partitioning: one process per GPU, torch.distributed for plumbing.

Two decompositions; the reference itself has no
distributed backend (its only parallelism is a thread pool over tiles,
liftfuse/engine.py:421-438):

* **Batch shards** (:func:`shard_range`) -- independent images split across
  ranks; no data-path collective at all.
* **Row strips** (:class:`RowStrips`) -- one very large image split into
  horizontal bands of rows.  Per level, each rank exchanges the fused kernel's
  dependency cone (``up``/``down`` quad rows, i.e. 2*up / 2*down pixel rows of
  that level's input) with its neighbours through NCCL send/recv, computes its
  interior rows while the halos are in flight, then the two boundary bands.
  The strip kernel (``b2dwt_forward_rows``) reflects only at the GLOBAL image
  edges, so the result is bit-identical to the single-GPU transform -- the
  tiled executor's halo argument (engine.py:404-417) applied across GPUs.

The exchange logic takes a ``band_forward`` callable so it can be exercised on
CPU with gloo in tests; on GPUs it is :meth:`Transform.forward_rows`.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["shard_range", "RowStrips", "StripLayout"]


def _in_place(t):
    """A message buffer that is the tensor itself (no staging copy)."""
    if not t.is_contiguous():
        raise ValueError("halo slices must be contiguous rows of the strip buffer")
    return t


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) share of ``n_items`` for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class StripLayout:
    """Pixel-row geometry of one rank's strip at one level."""

    height: int      # global image height (pixels) at this level
    width: int
    row0: int        # first global pixel row owned
    rows: int        # pixel rows owned (even)
    halo_top: int    # pixel rows received from rank-1 (0 on rank 0)
    halo_bot: int    # pixel rows received from rank+1 (0 on the last rank)

    @property
    def buffer_rows(self) -> int:
        return self.halo_top + self.rows + self.halo_bot

    @property
    def quad_rows(self) -> tuple[int, int]:
        return self.row0 // 2, (self.row0 + self.rows) // 2


class RowStrips:
    """Row-strip decomposition of one image across ``world`` ranks.

    ``cone = (up, down)`` is the fused kernel's vertical dependency cone in
    quad rows (``Transform.cone[:2]``).  Buffers are laid out
    ``[halo_top | owned rows | halo_bot]`` so halos are received in place and
    every band handed to the kernel is one contiguous slice.
    """

    def __init__(self, height: int, width: int, rank: int, world: int, cone, levels: int = 1):
        if height % (world << levels):
            raise ValueError(f"height {height} must be divisible by world*2^levels = {world << levels}")
        if width % (1 << levels):
            raise ValueError(f"width {width} must be divisible by 2^levels")
        self.height, self.width = height, width
        self.rank, self.world = rank, world
        self.up, self.down = int(cone[0]), int(cone[1])
        self.levels = levels
        per = height // world
        if per < 2 * max(self.up, self.down, 1) << (levels - 1):
            raise ValueError("strips are thinner than the exchanged halo")

    def layout(self, level: int = 0) -> StripLayout:
        h, w = self.height >> level, self.width >> level
        per = h // self.world
        return StripLayout(
            height=h,
            width=w,
            row0=self.rank * per,
            rows=per,
            halo_top=2 * self.up if self.rank > 0 else 0,
            halo_bot=2 * self.down if self.rank < self.world - 1 else 0,
        )

    # -- exchange ---------------------------------------------------------------
    def exchange(self, buf, level: int = 0, group=None):
        """Post the halo send/recv for ``buf`` (shape [buffer_rows, W]); returns
        the requests.  Sends: owned top 2*down rows to rank-1, owned bottom
        2*up rows to rank+1; receives into the halo rows."""
        import torch.distributed as dist

        L = self.layout(level)
        own = buf[L.halo_top:L.halo_top + L.rows]
        ops = []
        # whole-row slices of a row-contiguous buffer: sent and received in place
        if self.rank > 0:
            ops.append(dist.P2POp(dist.irecv, _in_place(buf[:L.halo_top]), self.rank - 1, group))
            ops.append(dist.P2POp(dist.isend, _in_place(own[:2 * self.down]), self.rank - 1, group))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, _in_place(own[L.rows - 2 * self.up:]), self.rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, _in_place(buf[L.halo_top + L.rows:]), self.rank + 1, group))
        return dist.batch_isend_irecv(ops) if ops else []

    # -- compute ------------------------------------------------------------------
    def _bands(self, level: int):
        """(interior, [boundary bands]) as (out_q0, out_q1) global quad rows."""
        L = self.layout(level)
        q0, q1 = L.quad_rows
        top = self.up if self.rank > 0 else 0
        bot = self.down if self.rank < self.world - 1 else 0
        interior = (q0 + top, q1 - bot)
        edges = []
        if top:
            edges.append((q0, q0 + top))
        if bot:
            edges.append((q1 - bot, q1))
        return interior, edges

    def _run_band(self, band_forward, buf, level, out_rows, out):
        L = self.layout(level)
        r0, r1 = out_rows
        if r1 <= r0:
            return
        q0 = L.quad_rows[0]
        buf_q0 = q0 - L.halo_top // 2  # global quad row of buffer row 0
        b0 = max(0, r0 - self.up)
        b1 = min(L.height // 2, r1 + self.down)
        band = buf[2 * (b0 - buf_q0):2 * (b1 - buf_q0)]
        band_forward(band, 2 * b0, L.height, r0, r1, tuple(o[r0 - q0:r1 - q0] for o in out))

    def forward(self, band_forward, buf, out, level: int = 0, group=None, overlap: bool = True):
        """One level: exchange halos of ``buf`` and transform the owned rows
        into ``out`` = (ll, hl, lh, hh) planes of the owned quad rows."""
        interior, edges = self._bands(level)
        if overlap:
            reqs = self.exchange(buf, level, group)
            self._run_band(band_forward, buf, level, interior, out)
            for r in reqs:
                r.wait()
        else:
            for r in self.exchange(buf, level, group):
                r.wait()
            self._run_band(band_forward, buf, level, interior, out)
        for e in edges:
            self._run_band(band_forward, buf, level, e, out)

    # -- inverse -----------------------------------------------------------------
    # The inverse strips the four subband planes instead: rank r owns quad rows
    # [row0/2, (row0+rows)/2) of every plane plus `up` / `down` halo quad rows of
    # the INVERSE program's cone (construct the RowStrips with
    # Transform.inv_plan.cone[:2]); bands go through ``band_inverse`` =
    # Transform.inverse_rows, which reflects only at global edges, so the image
    # rows are bit-identical to the single-GPU inverse.  The buffer is laid out
    # [quad row, plane, column] so one quad row of all four planes is contiguous:
    # each neighbour's halo travels as ONE packed message (not one per plane),
    # and the kernel reads each plane with a row pitch of 4 x W/2.

    def _sub_halos(self):
        return (self.up if self.rank > 0 else 0), (self.down if self.rank < self.world - 1 else 0)

    def allocate_subbands(self, new_empty, level: int = 0):
        """[halo_top + owned + halo_bot quad rows, 4, W/2] buffer of the planes."""
        L = self.layout(level)
        ht, hb = self._sub_halos()
        return new_empty((ht + L.rows // 2 + hb, 4, L.width // 2))

    def owned_subbands(self, sb, level: int = 0):
        """The owned quad rows as a [4, rows, W/2] view (plane-major, pitched)."""
        ht, _ = self._sub_halos()
        return sb[ht:ht + self.layout(level).rows // 2].permute(1, 0, 2)

    def exchange_subbands(self, sb, level: int = 0, group=None):
        """Post the per-plane halo send/recv of a subband buffer; returns the requests."""
        import torch.distributed as dist

        q = self.layout(level).rows // 2
        ht, hb = self._sub_halos()
        own = sb[ht:ht + q]
        ops = []  # one packed message per neighbour and direction (all four planes' rows)
        if self.rank > 0:
            ops.append(dist.P2POp(dist.irecv, _in_place(sb[:ht]), self.rank - 1, group))
            ops.append(dist.P2POp(dist.isend, _in_place(own[:self.down]), self.rank - 1, group))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, _in_place(own[q - self.up:]), self.rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, _in_place(sb[ht + q:]), self.rank + 1, group))
        return dist.batch_isend_irecv(ops) if ops else []

    def _run_inverse_band(self, band_inverse, sb, level, out_rows, out):
        L = self.layout(level)
        r0, r1 = out_rows
        if r1 <= r0:
            return
        q0 = L.quad_rows[0]
        buf_q0 = q0 - self._sub_halos()[0]  # global quad row of buffer row 0
        b0 = max(0, r0 - self.up)
        b1 = min(L.height // 2, r1 + self.down)
        band = tuple(sb[b0 - buf_q0:b1 - buf_q0, c] for c in range(4))  # pitched planes
        band_inverse(band, b0, L.height, r0, r1, out[2 * (r0 - q0):2 * (r1 - q0)])

    def inverse(self, band_inverse, sb, out, level: int = 0, group=None, overlap: bool = True):
        """One level of the inverse: exchange the planes' halos and rebuild the
        owned image rows into ``out`` ([rows, W])."""
        interior, edges = self._bands(level)
        reqs = self.exchange_subbands(sb, level, group)
        if not overlap:
            for r in reqs:
                r.wait()
            reqs = []
        self._run_inverse_band(band_inverse, sb, level, interior, out)
        for r in reqs:
            r.wait()
        for e in edges:
            self._run_inverse_band(band_inverse, sb, level, e, out)

    def allocate(self, new_empty, level: int = 0):
        """Buffer for level ``level``: ``new_empty(shape)`` -> tensor."""
        L = self.layout(level)
        return new_empty((L.buffer_rows, L.width))

    def owned(self, buf, level: int = 0):
        L = self.layout(level)
        return buf[L.halo_top:L.halo_top + L.rows]

    def dwt(self, band_forward, buf0, new_empty, group=None, overlap: bool = True):
        """Multi-level strips: level l's LL is written straight into the owned
        rows of level l+1's buffer.  Returns (ll_owned, [(hl, lh, hh) owned])."""
        details = []
        buf = buf0
        for lvl in range(self.levels):
            L = self.layout(lvl)
            nq = L.rows // 2
            if lvl + 1 < self.levels:
                nxt = self.allocate(new_empty, lvl + 1)
                ll = self.owned(nxt, lvl + 1)
            else:
                nxt = None
                ll = new_empty((nq, L.width // 2))
            hl, lh, hh = (new_empty((nq, L.width // 2)) for _ in range(3))
            self.forward(band_forward, buf, (ll, hl, lh, hh), lvl, group, overlap)
            details.append((hl, lh, hh))
            buf = nxt if nxt is not None else ll
        return buf, details
