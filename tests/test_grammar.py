"""The native grammar tracker (csrc/grammar.cpp via paper_2507_16784_b200.grammar)
against the REFERENCE tracker's own outputs (CPU, host code only):

* lifecycle events of the 157 golden documents (tracker.py Tracker.feed,
  tests/golden/events.json.gz), offsets / depths / payloads bit-exact;
* allowed_mask at EVERY position of 112 documents (40 golden streams, 72
  reference random_mask_walk documents under tools / no tools (incl. prefix-sharing
  tool names s / search / search_web) and depth limits
  16 / 2 / 1), tests/golden/masks.json.gz;
* the Rejected message (byte index and context) for inadmissible tokens.
"""

import gzip
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2507_16784_b200.grammar import Grammar, TokenMask
from paper_2507_16784_b200.structure import Rejected
from paper_2507_16784_b200.tokenizer import build_tokenizer

GOLDEN = Path(__file__).resolve().parent / "golden"
TOK = build_tokenizer()


def _load(name):
    with gzip.open(GOLDEN / name, "rt", encoding="utf-8") as f:
        return json.load(f)


def test_events_match_reference_tracker():
    recs = _load("events.json.gz")
    assert len(recs) == 157
    for r in recs:
        g = Grammar(r["tool_names"], 16, TOK)
        tr = g.tracker()
        got = []
        for tid in r["stream"]:
            for e in tr.feed(tid):
                got.append([e.kind, e.offset, e.depth, e.payload])
        assert got == r["events"], r["gen"]
        assert tr.done and tr.consumed == len(r["stream"])


def test_masks_match_reference_allowed_mask_everywhere():
    gold = _load("masks.json.gz")
    V = gold["vocab"]
    masks = [np.unpackbits(np.frombuffer(bytes.fromhex(h), dtype=np.uint8), bitorder="little")[:V]
             for h in gold["masks"]]
    positions = 0
    for d in gold["docs"]:
        g = Grammar(d["tools"], d["depth"], TOK)
        tr = g.tracker()
        for pos, tid in enumerate(d["stream"] + [None]):
            m = tr.allowed_mask()
            want = np.nonzero(masks[d["mask_idx"][pos]])[0].tolist()
            assert list(m.ids) == want, (d["tools"], d["depth"], pos)
            positions += 1
            if tid is not None:
                tr.feed(tid)
        assert tr.done
    assert positions > 10000


def test_rejected_messages_match_reference():
    gold = _load("masks.json.gz")
    checked = 0
    for d in gold["docs"]:
        by_pos: dict = {}
        for pos, t, msg in d["rejects"]:
            by_pos.setdefault(pos, []).append((t, msg))
        g = Grammar(d["tools"], d["depth"], TOK)
        tr = g.tracker()
        for pos, tid in enumerate(d["stream"] + [None]):
            for t, msg in by_pos.get(pos, ()):
                probe = tr.clone()
                with pytest.raises(Rejected) as ei:
                    probe.feed(t)
                assert str(ei.value) == msg
                checked += 1
            if tid is not None:
                tr.feed(tid)
    assert checked > 500


def test_mask_memo_ids_and_finish_tokens():
    """Masks are numbered in creation order and shared through the memo; the
    finish set holds exactly the admitted tokens whose bytes emit Done."""
    g = Grammar([], 16, TOK)
    tr = g.tracker()
    doc = '[{"thought":"a","conclusion":"b"}]'
    ids = TOK.tokenize(doc)
    seen = []
    for tid in ids:
        m = tr.allowed_mask()
        assert isinstance(m, TokenMask) and m.admits(tid)
        seen.append(m.mask_id)
        ev = tr.feed(tid)
        if any(e.kind == "Done" for e in ev):
            assert tid in m.finish_ids and m.can_finish
        elif m.can_finish:
            assert tid not in m.finish_ids
    assert tr.done
    assert max(seen) < g.mask_count
    # a second tracker over the same document reuses the memoised masks
    tr2 = g.tracker()
    again = []
    for tid in ids:
        again.append(tr2.allowed_mask().mask_id)
        tr2.feed(tid)
    assert again == seen
    closing = [m for m in map(g.mask, range(g.mask_count)) if m.can_finish]
    assert closing and all(TOK.pieces[t] in (b"]", b"}]") for m in closing for t in m.finish_ids)


def test_snapshot_restore_and_depth():
    g = Grammar(["search"], 2, TOK)
    tr = g.tracker()
    for tid in TOK.tokenize('[{"thought":"x","subtasks":[{'):
        tr.feed(tid)
    assert tr.current_depth() == 1
    snap = tr.snapshot()
    with pytest.raises(Rejected):
        tr.feed(TOK.token_for(b'"subtasks":') if hasattr(TOK, "token_for") else 999)
    tr.restore(snap)
    tr.feed(TOK.tokenize('"thought":')[0])
    assert tr.consumed == len(TOK.tokenize('[{"thought":"x","subtasks":[{')) + 1
