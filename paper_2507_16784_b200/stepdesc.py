"""Host-side builder of the per-step descriptor (tim_step_header + records).

The host plans a step purely in counts; the descriptor is the single int32
buffer every kernel of the step reads (include/timrun.h).
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib as L

_HDR = [
    "n_rows", "n_rows_pad", "n_new", "n_segs", "n_dec", "n_ext", "n_jobs", "n_ops", "n_phases",
    "n_last", "dec_total", "off_new", "off_segs", "off_dec", "off_dec_prefix", "off_ext", "off_jobs",
    "off_spans", "off_ops", "off_phases", "off_last", "ext_total", "off_ext_prefix",
    "split_dec_ctas", "split_ext_ctas", "serial",
]


class StepDesc:
    """Accumulates one step's records and packs them into an int32 array."""

    __slots__ = ("new", "segs", "dec", "ext", "jobs", "spans", "ops", "phase_starts", "last",
                 "n_rows", "_last_kind", "offsets", "rows_pad", "last_pad", "ctas", "serial", "last_mask")

    def __init__(self):
        self.new: list = []      # (slot, logical_idx, token, row, live_idx)
        self.segs: list = []     # (slot, m, n, row_off)
        self.dec: list = []      # decode tiles (row, slot, kv_len, nq, m, group)
        self.ext: list = []      # multi-token tiles (row, slot, kv_len, nq, m, group)
        self.jobs: list = []     # (slot, old_len, s, reencode_from, span_off, n_spans, out_row, keep)
        self.spans: list = []    # start, end (flattened pairs)
        self.ops: list = []      # (kind, slot, table_off, count, sp_before, owner)
        self.phase_starts: list = []
        self.last: list = []     # rows whose logits are produced
        self.last_mask: list = []  # per `last` row: device mask id of its masked pick (-1: none)
        self.n_rows = 0
        self._last_kind = -1
        self.offsets: dict = {}
        self.rows_pad: int | None = None   # row buffers padded to this many rows (graph bucket)
        self.last_pad = 0                  # `last` padded to this many entries (graph bucket)
        self.ctas = 0                      # SMs of the one-launch attention (mode 2 split)
        self.serial = 0                    # step serial for the attention plan (0: no plan)

    # ------------------------------------------------------------- page ops
    def op(self, kind: int, slot: int, table_off: int, count: int, sp_before: int,
           owner: int) -> None:
        if count <= 0:
            return
        if kind != self._last_kind:
            self.phase_starts.append(len(self.ops))
            self._last_kind = kind
        self.ops.append((kind, slot, table_off, count, sp_before, owner))

    def job(self, slot, old_len, s, reencode_from, spans, out_row, keep) -> None:
        off = len(self.spans) // 2
        for a, b in spans:
            self.spans.extend((a, b))
        self.jobs.append((slot, old_len, s, reencode_from, off, len(spans), out_row, keep))

    # Cost model of the one-launch attention (mode 2), in SM-microseconds,
    # calibrated on B200 on bench.py's own mixed steps (tools/split_sweep.py:
    # every sampled mixed step of the C2 trajectory re-packed under each
    # candidate and its layer-0 launch timed): a decode-tile CTA streams ~36
    # KB/us of page rows next to the items; a multi-token item costs ~8 us
    # (Q load, pipeline fill and drain, epilogue -- items on one CTA run back to
    # back) plus ~0.8 us per 64-key block for each of its (up to two) 32-query
    # blocks; items are dealt longest-first, round-robin.  Round-2 sweeps (K2
    # with P in TMEM and a 5-stage ring): (3.0, 1.2, 40 KB/us) 66.5-69.2 us ->
    # (8.0, 0.8, 36 KB/us) 63.4-64.6 us per mixed launch (run-to-run noise ~2
    # us).  TIMRUN_EXT_COST="item,block" overrides.
    DEC_US_PER_TOKEN = 4096 / 36e3
    EXT_US_PER_ITEM, EXT_US_PER_QBLOCK_BLOCK = (
        float(x) for x in os.environ.get("TIMRUN_EXT_COST", "8.0,0.8").split(","))

    def _split_cost(self, ext: list) -> tuple[float, int]:
        """(estimated us, CTAs for the items) of the best split for `ext`."""
        G = self.ctas
        times = sorted((self.EXT_US_PER_ITEM + self.EXT_US_PER_QBLOCK_BLOCK * ((e[3] + 31) // 32)
                        * ((e[2] + 63) // 64) for e in ext), reverse=True)
        n = len(times)
        if not self.dec:
            return (sum(times[0::min(G, n)]), G)
        w0 = sum(d[2] for d in self.dec) * self.DEC_US_PER_TOKEN
        best, best_g1 = None, 1
        for g1 in range(1, min(G - 1, n) + 1):
            t1 = sum(times[0::g1])          # CTA 0's items (longest first, round-robin)
            t = max(w0 / (G - g1), t1)
            if best is None or t < best:
                best, best_g1 = t, g1
        return (best, best_g1)

    def attention_split(self) -> tuple[int, int]:
        """CTAs given to the decode tiles and to the multi-token items when
        both run in one launch: minimise the slower side's estimated time."""
        G = self.ctas
        if G <= 0 or not self.ext:
            return (G, 0)
        if not self.dec:
            return (0, G)
        g1 = self._split_cost(self.ext)[1]
        return (G - g1, g1)

    @staticmethod
    def halve_items(ext: list) -> list:
        """Each item of > 32 queries as two items of <= 32 (the kernel skips a
        32-query item's second MMA tile): the K/V slice is streamed twice, but
        the work comes in half-size pieces."""
        out = []
        for row, slot, kv_len, nq, fresh, grp in ext:
            if nq <= 32:
                out.append((row, slot, kv_len, nq, fresh, grp))
            else:
                out.append((row, slot, kv_len - (nq - 32), 32, fresh, grp))
                out.append((row + 32, slot, kv_len, nq - 32, fresh, grp))
        return out

    def choose_item_size(self) -> None:
        """Whole items (two MMA tiles sharing each K/V block) are the cheaper
        work per query; halves only pay when SMs would otherwise idle: a step
        with no decode rows (prefill / extend only) and fewer items than half
        the CTAs.  (Halving against the mode-2 split as well, whenever the
        cost model predicted a gain, measured 62.9 -> 62.2 us and 78.9 -> 75.0
        us in tools/attn_mixed_bench.py but 61.2 -> 62.0 us on the bench's
        mixed steps, so mixed steps keep whole items.)  TIMRUN_HALVE_ITEMS=0
        disables, =2 also halves in mixed steps when the model predicts a gain."""
        mode = os.environ.get("TIMRUN_HALVE_ITEMS", "1")
        if mode == "0" or self.ctas <= 0 or not self.ext or all(e[3] <= 32 for e in self.ext):
            return
        halves = self.halve_items(self.ext)
        if not self.dec:
            if 2 * len(self.ext) <= self.ctas:
                self.ext = halves
        elif mode == "2" and self._split_cost(halves)[0] < 0.97 * self._split_cost(self.ext)[0]:
            self.ext = halves

    # ---------------------------------------------------------------- pack
    def pack(self) -> np.ndarray:
        """Header, then `last` (first, so its offset is fixed at HEADER_INTS and a
        captured graph can index it), then the other record arrays."""
        parts = []
        off = L.HEADER_INTS
        hdr = dict.fromkeys(_HDR, 0)

        def add(name, rows, width):
            nonlocal off
            arr = np.asarray(rows, dtype=np.int32).reshape(-1)
            if width:
                assert arr.size == len(rows) * width
            hdr["off_" + name] = off
            parts.append(arr)
            off += arr.size

        last = list(self.last) + [0] * max(0, self.last_pad - len(self.last))
        add("last", last, 0)
        # mask ids right after `last` (a fixed offset for a captured graph too)
        add("last_mask", list(self.last_mask) + [-1] * (len(last) - len(self.last_mask)), 0)
        add("new", self.new, L.NEW_FIELDS)
        add("segs", self.segs, L.SEG_FIELDS)
        add("dec", self.dec, L.DEC_FIELDS)
        prefix = np.zeros(len(self.dec) + 1, dtype=np.int64)
        if self.dec:
            prefix[1:] = np.cumsum([d[2] for d in self.dec])
        assert prefix[-1] < 2**31
        hdr["off_dec_prefix"] = off
        parts.append(prefix.astype(np.int32))
        off += prefix.size
        self.choose_item_size()
        # longest items first: the kernel deals them round-robin to its CTAs
        self.ext.sort(key=lambda e: -e[2])
        add("ext", self.ext, L.EXT_FIELDS)
        eprefix = np.zeros(len(self.ext) + 1, dtype=np.int64)
        if self.ext:
            eprefix[1:] = np.cumsum([e[2] for e in self.ext])
        assert eprefix[-1] < 2**31
        hdr["off_ext_prefix"] = off
        parts.append(eprefix.astype(np.int32))
        off += eprefix.size
        add("jobs", self.jobs, L.JOB_FIELDS)
        add("spans", self.spans, 0)
        add("ops", self.ops, L.OP_FIELDS)
        phases = list(self.phase_starts) + [len(self.ops)]
        hdr["off_phases"] = off
        parts.append(np.asarray(phases, dtype=np.int32))
        off += len(phases)
        hdr.update(
            n_rows=self.n_rows,
            n_rows_pad=self.n_rows if self.rows_pad is None else max(self.rows_pad, self.n_rows),
            n_new=len(self.new), n_segs=len(self.segs), n_dec=len(self.dec), n_ext=len(self.ext),
            n_jobs=len(self.jobs), n_ops=len(self.ops), n_phases=len(self.phase_starts),
            n_last=len(last), dec_total=int(prefix[-1]), ext_total=int(eprefix[-1]),
        )
        hdr["split_dec_ctas"], hdr["split_ext_ctas"] = self.attention_split()
        hdr["serial"] = self.serial
        self.offsets = hdr
        head = np.zeros(L.HEADER_INTS, dtype=np.int32)
        for i, k in enumerate(_HDR):
            head[i] = hdr[k]
        return np.concatenate([head] + parts)
