"""Host-side logic of the product package vs the oracle (CPU-only): prune
buffer, coalesce, the KV-pruned metric, and the step-descriptor packing the
kernels read (include/timrun.h layout)."""

import random

import numpy as np
import pytest

from oracle import pruning as opr
from paper_2507_16784_b200 import _lib as L
from paper_2507_16784_b200.pruning import (PruneBuffer, PrunePlan, RequestMetrics, ZeroLength,
                                           coalesce, kv_pruned_pct, suffix_start)
from paper_2507_16784_b200.spans import TokenSpan
from paper_2507_16784_b200.stepdesc import _HDR, StepDesc


def _span_list(spans):
    return [(s.start, s.end) for s in spans]


def test_prune_buffer_matches_oracle_random():
    """pruning.py:61-84 semantics over random nested span streams, T in 0..5."""
    rng = random.Random(5)
    for _ in range(300):
        t = rng.randrange(0, 6)
        subsume = rng.random() < 0.7
        mine, ref = PruneBuffer(t, subsume), opr.Buffer(t, subsume)
        pos = 0
        for _ in range(rng.randrange(1, 12)):
            # a closing list starts after the previous ones or encloses some of them
            if rng.random() < 0.3 and mine.entries:
                a = min(e.start for e in mine.entries) - rng.randrange(0, 3)
                a = max(a, 0)
            else:
                a = pos + rng.randrange(0, 5)
            b = max(a + 1, pos) + rng.randrange(1, 9)
            pos = b
            try:
                p1 = mine.on_list_closed(TokenSpan(a, b))
            except AssertionError:
                with pytest.raises(AssertionError):
                    ref_entries = [e for e in ref.entries if not (a <= e.start and e.end <= b)] \
                        if subsume else list(ref.entries)
                    ref_entries.append(opr.Span(a, b))
                    assert all(ref_entries[i].start < ref_entries[i + 1].start
                               for i in range(len(ref_entries) - 1))
                break
            p2 = ref.on_list_closed(opr.Span(a, b))
            assert (p1 is None) == (p2 is None)
            if p1 is not None:
                assert _span_list(p1.evict_spans) == [(s.start, s.end) for s in p2.spans]
                assert p1.reencode_from == p2.reencode_from
                assert p1.freed_token_count == p2.freed
            assert _span_list(mine.entries) == [(s.start, s.end) for s in ref.entries]
    with pytest.raises(ValueError):
        PruneBuffer(-1)


def test_coalesce_matches_oracle_random():
    """pruning.py:87-99 (tests/test_pruning.py:74-93 shape)."""
    rng = random.Random(1)
    for _ in range(300):
        plans, oplans = [], []
        for _ in range(rng.randint(1, 5)):
            a = rng.randrange(0, 50)
            b = a + rng.randrange(1, 10)
            plans.append(PrunePlan([TokenSpan(a, b)], a, b - a))
            oplans.append(opr.Plan([opr.Span(a, b)], a, b - a))
        p, o = coalesce(plans), opr.coalesce(oplans)
        assert _span_list(p.evict_spans) == [(s.start, s.end) for s in o.spans]
        assert p.reencode_from == o.reencode_from and p.freed_token_count == o.freed
    with pytest.raises(ValueError):
        coalesce([])


def test_suffix_start_is_reference_scan():
    rng = random.Random(2)
    for _ in range(200):
        live = sorted(rng.sample(range(200), rng.randrange(0, 60)))
        r = rng.randrange(0, 210)
        s0 = 0
        while s0 < len(live) and live[s0] < r:   # pruning.py:126-128
            s0 += 1
        assert suffix_start(live, r) == s0


def test_metric_and_metrics_shape():
    assert kv_pruned_pct(1569.2, 3362.2) == pytest.approx(0.533, abs=1e-3)
    assert kv_pruned_pct(3218.6, 8974.7) == pytest.approx(0.641, abs=1e-3)
    assert kv_pruned_pct(500, 500) == 0.0 and kv_pruned_pct(900, 300) == 0.0
    assert 0.0 <= kv_pruned_pct(1, 10**9) < 1.0
    with pytest.raises(ZeroLength):
        kv_pruned_pct(10, 0)
    d = RequestMetrics(output_len=100, max_cache=60, position_high_water=60, tool_calls=2,
                       pruned_tokens=55).to_dict()
    assert set(d) == {"output_len", "max_cache", "kv_pruned", "position_high_water", "tool_calls",
                      "pruned_tokens"}
    assert d["kv_pruned"] == pytest.approx(0.4)


def test_step_descriptor_layout():
    """The packed descriptor matches tim_step_header: header fields, record
    widths, `last` first (fixed offset for captured graphs), phase starts."""
    sd = StepDesc()
    sd.new += [(0, 5, 7, 0, 3), (1, 9, 8, 1, 0)]
    sd.segs += [(0, 3, 1, 0), (1, 0, 1, 1)]
    sd.dec += [(0, 0, 4, 1, 3, 0), (1, 1, 1, 1, 0, 0)]
    sd.op(L.OP_FREE, 0, 2, 3, 10, 0)
    sd.op(L.OP_FREE, 1, 0, 2, 13, 1)
    sd.op(L.OP_ALLOC, 0, 2, 1, 15, 0)
    sd.job(0, 5, 2, 4, [(4, 6)], 0, 1)
    sd.last += [0, 1]
    sd.n_rows = 2
    sd.rows_pad, sd.last_pad = 64, 4
    arr = sd.pack()
    hdr = {k: int(arr[i]) for i, k in enumerate(_HDR)}
    assert len(_HDR) <= L.HEADER_INTS
    assert hdr["off_last"] == L.HEADER_INTS and hdr["n_last"] == 4
    assert list(arr[L.HEADER_INTS:L.HEADER_INTS + 4]) == [0, 1, 0, 0]
    assert hdr["n_rows"] == 2 and hdr["n_rows_pad"] == 64
    assert hdr["n_phases"] == 2   # FREE run, then ALLOC
    assert list(arr[hdr["off_phases"]:hdr["off_phases"] + 3]) == [0, 2, 3]
    assert hdr["dec_total"] == 5
    assert list(arr[hdr["off_dec_prefix"]:hdr["off_dec_prefix"] + 3]) == [0, 4, 5]
    ops = arr[hdr["off_ops"]:hdr["off_ops"] + 3 * L.OP_FIELDS].reshape(3, L.OP_FIELDS)
    assert ops[2].tolist() == [L.OP_ALLOC, 0, 2, 1, 15, 0]
    job = arr[hdr["off_jobs"]:hdr["off_jobs"] + L.JOB_FIELDS].tolist()
    assert job == [0, 5, 2, 4, 0, 1, 0, 1]
    assert arr[hdr["off_spans"]:hdr["off_spans"] + 2].tolist() == [4, 6]
    assert arr.dtype == np.int32


def test_header_fields_match_c_struct():
    """stepdesc._HDR is tim_step_header's field order (include/timrun.h)."""
    import re
    from pathlib import Path
    text = (Path(__file__).resolve().parents[1] / "include" / "timrun.h").read_text()
    body = re.search(r"typedef struct \{(.*?)\} tim_step_header;", text, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        for part in decl.replace("int32_t", "").split(","):
            part = part.strip()
            if part:
                names.append(part)
    fields = [n for n in names if not n.startswith("reserved")]
    assert fields == list(_HDR)
    reserved = int(re.search(r"reserved\[(\d+)\]", body).group(1))
    assert len(fields) + reserved == L.HEADER_INTS


def _ext_items(n_rows, m, heads=8, qpi=64):
    items = []
    for q0 in range(0, n_rows, qpi):
        nq = min(qpi, n_rows - q0)
        for h in range(heads):
            items.append((q0, 0, m + q0 + nq, nq, m, h))
    return items


def test_attention_split_cost_model():
    """mode-2 CTA split: degenerate lists take every CTA; otherwise both sides
    get >= 1 CTA, the ext side never more CTAs than items, and more
    multi-token work never gets fewer CTAs."""
    def split(n_dec_keys, ext):
        sd = StepDesc()
        sd.ctas = 148
        if n_dec_keys:
            per = n_dec_keys // 64
            sd.dec += [(i, i, per, 1, per - 1, 0) for i in range(64)]
        sd.ext += ext
        return sd.attention_split()

    assert split(44000, []) == (148, 0)
    assert split(0, _ext_items(150, 600)) == (0, 148)
    prev = 0
    for n_rows in (8, 40, 150, 440, 900, 1600):
        ext = _ext_items(n_rows, 700)
        g0, g1 = split(44000, ext)
        assert g0 + g1 == 148 and g0 >= 1 and 1 <= g1 <= len(ext)
        assert g1 >= prev
        prev = g1


def test_pack_sorts_items_and_stamps_serial():
    sd = StepDesc()
    sd.ext += [(0, 0, 100, 8, 92, 0), (0, 0, 700, 40, 660, 1), (0, 0, 300, 8, 292, 2)]
    sd.serial, sd.ctas = 17, 148
    arr = sd.pack()
    hdr = {k: int(arr[i]) for i, k in enumerate(_HDR)}
    # extend-only step with few items: the 40-query item is halved (32 + 8)
    assert hdr["serial"] == 17 and hdr["n_ext"] == 4
    ext = arr[hdr["off_ext"]:hdr["off_ext"] + 4 * L.EXT_FIELDS].reshape(4, L.EXT_FIELDS)
    assert ext[:, 2].tolist() == [700, 692, 300, 100]   # longest first (round-robin dealing)
    assert hdr["split_dec_ctas"] == 0 and hdr["split_ext_ctas"] == 148


def test_item_halving():
    """A > 32-query item splits into rows [row, row+32) and [row+32, row+nq)
    with the causal key counts of each half; whole items are kept in mixed
    steps and in extend-only steps with enough items for the CTAs."""
    halves = StepDesc.halve_items([(10, 3, 700, 64, 636, 5), (80, 3, 900, 20, 880, 2)])
    assert halves == [(10, 3, 668, 32, 636, 5), (42, 3, 700, 32, 636, 5), (80, 3, 900, 20, 880, 2)]
    for q in range(64):   # every query keeps its visible-key limit kv_len - nq + qi
        row, kv, nq = (halves[0][0], 668, 32) if q < 32 else (halves[1][0], 700, 32)
        assert kv - nq + (10 + q - row) == 700 - 64 + q

    def run(n_items, with_dec):
        sd = StepDesc()
        sd.ctas = 148
        sd.ext += [(0, 0, 700, 64, 636, h % 8) for h in range(n_items)]
        if with_dec:
            sd.dec += [(i, i, 700, 1, 699, 0) for i in range(64)]
        sd.choose_item_size()
        return len(sd.ext)

    assert run(16, False) == 32         # idle SMs: halves
    assert run(100, False) == 100       # enough items: whole
    assert run(16, True) == 16          # mixed step: whole (default)
