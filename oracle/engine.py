"""Oracle restatement of the reference step loop (threadrun/scheduler.py).  Test-only.

A sequential, per-request CPU engine in exactly the reference's order:
admissions (scheduler.py:279-290) -> tool deliveries (292-301) -> advances in
submission order (303-316) -> starvation (318, 337-341).  Each advance applies
due plans (385-411), extends at start=len(live) (360-383) and selects the next
scripted token (413-442); events come from a per-trace event table keyed by
generation offset (the reference tracker's output, recorded as golden data),
so the oracle does not depend on the product's structure scanner.

The backend is either accounting-only (ScriptedModel semantics, model.py:
195-233) or the numeric oracle Model (oracle/model.py).  Tool responses come
from trace overrides (scheduler.py:469-472).
"""

from __future__ import annotations

import json

from .model import PositionOverflow
from .paging import OutOfPages, PagePool, PageTable
from .pruning import Buffer, Span, SpanOutOfRange, apply, coalesce


class ScriptError(RuntimeError):
    pass


class TokenLimit(RuntimeError):
    pass


class Rejected(RuntimeError):
    pass


FAULTS = (PositionOverflow, ScriptError, TokenLimit, Rejected)
TERMINAL = ("finished", "failed")


class Accounting:
    """model.py:195-233 ScriptedModel: one page per token, no arithmetic."""

    def __init__(self, position_limit: int):
        self.position_limit = position_limit

    def make_pool(self, capacity):
        return PagePool(capacity)

    def _fwd(self, n, positions, table, pool):
        for p in positions:
            if p >= self.position_limit:
                raise PositionOverflow(int(p), self.position_limit)
        table.append(pool.alloc(table.request_id, n))
        return None

    def prefill(self, tokens, positions, table, pool):
        return self._fwd(len(tokens), positions, table, pool)

    def extend(self, tokens, start, table, pool):
        return self._fwd(len(tokens), range(start, start + len(tokens)), table, pool)


class Req:
    def __init__(self, rid, prompt, script, responses, events, threshold, subsume, max_out):
        self.rid = rid
        self.prompt = list(prompt)
        self.logical = list(prompt)
        self.pending: list[int] = []
        self.live: list[int] = []
        self.table = PageTable(rid)
        self.buffer = Buffer(threshold, subsume)
        self.plans: list = []
        self.status = "queued"
        self.failure = None
        self.script = list(script)
        self.pos = 0
        self.responses = responses
        self.events = events            # {generation offset: [(kind, payload), ...]}
        self.fed = 0                    # tokens fed to the (virtual) tracker
        self.tool_calls = 0
        self.pending_tool = None
        self.max_out = max_out
        self.starved = 0
        self.eviction_log: list = []
        self.applied_spans: list = []
        self.first_encoded: set = set()
        self.output_len = 0
        self.max_cache = 0
        self.high_water = 0
        self.pruned_tokens = 0
        self.last_logits = None
        self.transitions = ["queued"]

    def set_status(self, s):
        if s != self.status:
            self.status = s
            self.transitions.append(s)

    @property
    def prompt_len(self):
        return len(self.prompt)

    @property
    def encoded_count(self):
        return len(self.logical) - len(self.pending)

    def metrics(self):
        from .pruning import kv_pruned_pct
        return {"output_len": self.output_len, "max_cache": self.max_cache,
                "kv_pruned": kv_pruned_pct(self.max_cache, self.output_len) if self.output_len else 0.0,
                "position_high_water": self.high_water, "tool_calls": self.tool_calls,
                "pruned_tokens": self.pruned_tokens}


class Engine:
    def __init__(self, backend, *, max_batch=8, threshold=1, position_limit=256, pool_pages=0,
                 max_queue=64, starvation_steps=50, subsume=True, max_output_tokens=200_000,
                 tokenize=None):
        self.backend = backend
        self.max_batch = max_batch
        self.threshold = threshold
        self.position_limit = position_limit
        self.starvation_steps = starvation_steps
        self.subsume = subsume
        self.max_output_tokens = max_output_tokens
        self.max_queue = max_queue
        self.pool = backend.make_pool(pool_pages or max_batch * position_limit)
        self.tokenize = tokenize
        self.requests: dict = {}
        self.queue: list = []
        self.results: dict = {}
        self.step_index = 0
        self._n = 0

    def submit(self, prompt_tokens, script, responses, events, threshold=None, subsume=None):
        if len(prompt_tokens) >= self.position_limit:
            raise ValueError("prompt too long")
        rid = f"r{self._n}"
        self._n += 1
        self.requests[rid] = Req(rid, prompt_tokens, script, responses or {}, events,
                                 self.threshold if threshold is None else threshold,
                                 self.subsume if subsume is None else subsume,
                                 self.max_output_tokens)
        self.queue.append(rid)
        return rid

    def active(self):
        return sum(1 for r in self.requests.values()
                   if r.status in ("decoding", "awaiting_tool", "extending"))

    def all_terminal(self):
        return all(r.status in TERMINAL for r in self.requests.values()) and not self.queue

    def step(self):
        flops = 0
        decoded = {}
        parked = []
        while self.queue and self.active() < self.max_batch:
            req = self.requests[self.queue[0]]
            try:
                flops += self._activate(req)
            except OutOfPages:
                req.starved += 1
                parked.append(req)
                break
            except FAULTS as e:
                self._fail(req, f"{type(e).__name__}: {e}")
            self.queue.pop(0)
        for req in list(self.requests.values()):
            if req.pending_tool is not None:
                value = req.pending_tool
                req.pending_tool = None
                try:
                    self._integrate(req, value[0])
                except FAULTS as e:
                    self._fail(req, f"{type(e).__name__}: {e}")
        for req in list(self.requests.values()):
            if req.status != "decoding":
                continue
            try:
                before = len(req.first_encoded)
                flops += self._advance(req)
                decoded[req.rid] = len(req.first_encoded) - before
                req.starved = 0
            except OutOfPages:
                req.starved += 1
                parked.append(req)
            except FAULTS as e:
                self._fail(req, f"{type(e).__name__}: {e}")
        over = [r for r in parked if r.starved > self.starvation_steps]
        if over:
            self._fail(max(over, key=lambda r: len(r.live)), "OutOfPages: starved past deadlock limit")
        self.step_index += 1
        st = [r.status for r in self.requests.values()]
        return {
            "report": [self.step_index, st.count("decoding"), st.count("awaiting_tool"),
                       st.count("finished"), st.count("failed"), self.pool.free_count, flops],
            "request_live": {r.rid: len(r.live) for r in self.requests.values()
                             if r.status not in TERMINAL},
            "decoded": decoded,
        }

    def _activate(self, req):
        flops = 0
        logits = None
        if req.prompt:
            positions = list(range(len(req.prompt)))
            logits = self.backend.prefill(req.prompt, positions, req.table, self.pool)
            req.live = list(range(len(req.prompt)))
            for i, p in enumerate(positions):
                flops += p + 1
                req.first_encoded.add(i)
            self._touch(req)
        req.set_status("decoding")
        self._select(req, logits)
        return flops

    def _advance(self, req):
        self._apply_due(req)
        assert req.pending
        idxs = req.pending
        toks = [req.logical[i] for i in idxs]
        start = len(req.live)
        if start + len(toks) > self.position_limit:
            raise PositionOverflow(start + len(toks) - 1, self.position_limit)
        logits = self.backend.extend(toks, start, req.table, self.pool)
        req.last_logits = logits
        flops = 0
        for i, idx in enumerate(idxs):
            if idx not in req.first_encoded:
                flops += start + i + 1
                req.first_encoded.add(idx)
        req.live = req.live + idxs
        req.pending = []
        self._touch(req)
        self._select(req, logits)
        return flops

    def _apply_due(self, req):
        due = [p for p in req.plans if max(s.end for s in p.spans) <= req.encoded_count]
        if not due:
            return
        req.plans = [p for p in req.plans if p not in due]
        plan = coalesce(due)
        freed, _tok, s0, new_live = apply(plan, req.table, req.live, req.logical)
        self.pool.free(freed)
        req.pruned_tokens += len(req.live) - len(new_live)
        req.applied_spans.extend(plan.spans)
        req.pending = new_live[s0:] + req.pending
        req.live = new_live[:s0]

    def _feed(self, req, tid):
        evs = req.events.get(req.fed, ())
        req.fed += 1
        if evs == "reject":
            raise Rejected(f"token {tid} rejected")
        for kind, payload in evs:
            self._event(req, kind, payload)

    def _select(self, req, logits):
        if req.pos >= len(req.script):
            raise ScriptError("script exhausted before document completed")
        tid = req.script[req.pos]
        req.pos += 1
        if req.events.get(req.fed) == "reject":
            raise ScriptError(f"scripted token {tid} not admitted")
        req.logical.append(tid)
        req.pending.append(len(req.logical) - 1)
        req.output_len += 1
        if req.output_len > req.max_out:
            raise TokenLimit(f"output exceeded {req.max_out} tokens")
        self._feed(req, tid)

    def _event(self, req, kind, payload):
        if kind == "SubtaskListClosed":
            span = Span(payload["span_start"] + req.prompt_len, payload["span_end"] + req.prompt_len)
            plan = req.buffer.on_list_closed(span)
            if plan is not None:
                req.plans.append(plan)
                req.eviction_log.extend(Span(s.start - req.prompt_len, s.end - req.prompt_len)
                                        for s in plan.spans)
        elif kind == "ToolResultSlotOpened":
            idx = req.tool_calls
            req.tool_calls += 1
            req.pending_tool = (req.responses.get(idx),)
            req.set_status("awaiting_tool")
        elif kind == "Done":
            self._finish(req)

    def _integrate(self, req, value):
        if req.status in TERMINAL:
            return
        req.set_status("extending")
        ids = self.tokenize(json.dumps(value, separators=(",", ":"), ensure_ascii=False))
        for tid in ids:
            req.logical.append(tid)
            req.pending.append(len(req.logical) - 1)
            self._feed(req, tid)
        req.output_len += len(ids)
        if req.status == "extending":
            req.set_status("decoding")

    def _touch(self, req):
        n = len(req.live)
        req.max_cache = max(req.max_cache, n)
        req.high_water = max(req.high_water, n)
        assert len(req.live) == len(req.table)

    def _finish(self, req):
        self.pool.free(req.table.truncate_from(0))
        req.live = []
        req.set_status("finished")
        self.results[req.rid] = {"status": "finished", "metrics": req.metrics()}

    def _fail(self, req, reason):
        if req.status in TERMINAL:
            return
        self.pool.free(req.table.truncate_from(0))
        req.live = []
        req.failure = reason
        req.set_status("failed")
        self.results[req.rid] = {"status": "failed", "failure": reason, "metrics": req.metrics()}


def event_table(events) -> dict:
    """Golden event list [[kind, offset, depth, payload], ...] -> {offset: [(kind, payload)]}."""
    table: dict = {}
    for kind, offset, _depth, payload in events:
        table.setdefault(offset, []).append((kind, payload))
    return table
