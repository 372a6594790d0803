"""Tokenizer and the native grammar tracker's events vs the reference (golden vectors made by
oracle/gen_golden.py from threadrun's tokenizer.py and tracker.py)."""

import gzip
import json

import pytest

from paper_2507_16784_b200.grammar import Grammar
from paper_2507_16784_b200.structure import Rejected
from paper_2507_16784_b200.tokenizer import build_tokenizer


def _load(golden, name):
    with gzip.open(golden / name, "rt", encoding="utf-8") as f:
        return json.load(f)


def test_tokenizer_matches_reference(golden):
    tok = build_tokenizer()
    for text, ids in _load(golden, "tokenizer.json.gz"):
        assert tok.tokenize(text) == ids
        assert tok.detokenize(ids) == text.encode("utf-8")
    assert tok.vocab_size == 265


def test_events_match_reference_tracker(golden):
    tok = build_tokenizer()
    recs = _load(golden, "events.json.gz")
    assert len(recs) > 150
    for rec in recs:
        sc = Grammar(rec["tool_names"], 16, tok).tracker()
        got = []
        for t in rec["stream"]:
            got.extend([e.kind, e.offset, e.depth, e.payload] for e in sc.feed(t))
        assert got == rec["events"], rec["gen"]
        assert sc.done


def test_stream_equals_document_tokens(golden):
    tok = build_tokenizer()
    for rec in _load(golden, "events.json.gz"):
        assert tok.detokenize(rec["stream"]).decode() == rec["text"]


def test_rejects_non_document():
    tok = build_tokenizer()
    with pytest.raises(Rejected):
        Grammar([], 16, tok).tracker().feed(ord("x"))
    sc = Grammar([], 16, tok).tracker()
    for t in tok.tokenize('[{"thought":"a","conclusion":"b"}]'):
        sc.feed(t)
    assert sc.done
    with pytest.raises(Rejected):
        sc.feed(ord("]"))


def test_make_trace_from_text_matches_reference(golden):
    from paper_2507_16784_b200.traces import make_trace_from_text
    for rec in _load(golden, "events.json.gz"):
        tr = make_trace_from_text(rec["text"])
        assert tr.script == rec["script"], rec["gen"]
        assert {str(k): v for k, v in tr.tool_responses.items()} == rec["tool_responses"]
        assert tr.tool_names == rec["tool_names"]


def test_deep_doc_structure_matches_reference_shape(golden):
    """deep_recursion_doc has the reference generator's token geometry
    (schema.py:449-471): same length and identical structure events."""
    from paper_2507_16784_b200.traces import deep_recursion_doc, make_trace_from_text
    tok = build_tokenizer()
    for rec in _load(golden, "events.json.gz"):
        if rec["gen"][0] != "deep_recursion_tree":
            continue
        _, levels, branching, seed = rec["gen"]
        tr = make_trace_from_text(deep_recursion_doc(levels, branching, seed=seed + 100))
        assert len(tr.script) == len(rec["script"])
        sc = Grammar(tr.tool_names, 16, tok).tracker()
        got = [[e.kind, e.offset, e.depth, e.payload] for t in tr.script for e in sc.feed(t)]
        assert got == rec["events"]
