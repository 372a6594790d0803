"""Oracle restatement of the reference prune rule (threadrun/pruning.py).  Test-only."""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Span:
    """Half-open logical-token range (schema.py:36-57 TokenSpan)."""
    start: int
    end: int

    def __len__(self) -> int:
        return self.end - self.start

    def contains(self, o: "Span") -> bool:
        return self.start <= o.start and o.end <= self.end


@dataclass
class Plan:
    """pruning.py:29-33 PrunePlan"""
    spans: list
    reencode_from: int
    freed: int


class SpanOutOfRange(RuntimeError):
    pass


class Buffer:
    """pruning.py:61-84: FIFO of capacity T with nested-list subsumption."""

    def __init__(self, threshold: int, subsume: bool = True):
        if threshold < 0:
            raise ValueError("threshold must be >= 0")
        self.threshold, self.subsume, self.entries = threshold, subsume, []

    def on_list_closed(self, span: Span):
        if self.subsume:
            self.entries = [e for e in self.entries if not span.contains(e)]
        self.entries.append(span)
        if len(self.entries) > self.threshold:
            victim = self.entries.pop(0)
            return Plan([victim], victim.start, len(victim))
        return None


def coalesce(plans):
    """pruning.py:87-99: sorted, merged, disjoint spans; reencode_from = min start."""
    if not plans:
        raise ValueError("no plans to coalesce")
    spans = sorted((s for p in plans for s in p.spans), key=lambda s: s.start)
    merged = []
    for s in spans:
        if merged and s.start <= merged[-1].end:
            if s.end > merged[-1].end:
                merged[-1] = Span(merged[-1].start, s.end)
        else:
            merged.append(s)
    return Plan(merged, merged[0].start, sum(len(s) for s in merged))


def apply(plan, table, live, tokens):
    """pruning.py:102-133 -> (freed page ids, suffix tokens, suffix_start, new_live)."""
    if len(live) != len(table):
        raise SpanOutOfRange("live list and page table desynchronized")
    for s in plan.spans:
        if s.end > len(tokens):
            raise SpanOutOfRange(f"span [{s.start},{s.end}) beyond {len(tokens)}")
    evict = set()
    for s in plan.spans:
        evict.update(range(s.start, s.end))
    s0 = 0
    while s0 < len(live) and live[s0] < plan.reencode_from:
        s0 += 1
    freed = table.truncate_from(s0)
    new_live = live[:s0] + [i for i in live[s0:] if i not in evict]
    return freed, [tokens[i] for i in new_live[s0:]], s0, new_live


def kv_pruned_pct(max_cache: float, output_len: float) -> float:
    """pruning.py:136-143"""
    if output_len <= 0:
        raise ValueError("output_len must be positive")
    v = 1.0 - max_cache / output_len
    return 0.0 if v < 0.0 else min(v, 1.0 - 1e-12)


def evictions(list_spans, threshold: int, subsume: bool = True):
    """pruning.py:146-168 rule oracle over the ordered SubtaskListClosed spans."""
    queued, order = [], []
    for span in list_spans:
        if subsume:
            queued = [q for q in queued if not span.contains(q)]
        queued.append(span)
        if len(queued) > threshold:
            order.append(queued.pop(0))
    return order


def surgery(seq, spans):
    """oracles.py:97-102"""
    drop = set()
    for s in spans:
        drop.update(range(s.start, s.end))
    return [x for i, x in enumerate(seq) if i not in drop]
