"""Replay traces and synthetic TIM-structured trajectories.

A trace is the scripted side of a request (threadrun/traces.py:23-62): the
token stream the model emits with every tool_result value cut out (the engine
inserts the tool response itself) plus the responses by call index.

`make_trace_from_text` derives a trace from a canonical document: the value
of the k-th `"tool_result":` key token is exactly tokenize(json.dumps(v)) of
the k-th tool result in document order, so cutting it out reproduces the
reference's make_trace.  `deep_recursion_doc` writes the long-horizon
document family (full `levels`-deep, `branching`-wide task trees with
`text_chars`-letter texts — the shape of schema.py:449-471) with its own RNG.
"""

from __future__ import annotations

import gzip
import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .tokenizer import build_tokenizer

TOOL_RESULT_KEY = b'"tool_result":'


@dataclass
class Trace:
    script: list
    tool_responses: dict = field(default_factory=dict)
    tool_names: list = field(default_factory=list)
    text: str = ""

    def to_json(self) -> str:
        return json.dumps({"script": self.script,
                           "tool_responses": {str(k): v for k, v in self.tool_responses.items()},
                           "tool_names": self.tool_names}, separators=(",", ":"), ensure_ascii=False)

    @classmethod
    def from_json(cls, text: str) -> "Trace":
        d = json.loads(text)
        return cls(script=list(d["script"]),
                   tool_responses={int(k): v for k, v in d.get("tool_responses", {}).items()},
                   tool_names=list(d.get("tool_names", [])))


def _walk(tasks):
    for t in tasks:
        yield t
        if isinstance(t.get("subtasks"), list):
            yield from _walk(t["subtasks"])


def make_trace_from_text(text: str, tokenizer=None) -> Trace:
    tok = tokenizer or build_tokenizer()
    ids = tok.tokenize(text)
    doc = json.loads(text)
    uses = [t for t in _walk(doc) if "tool_name" in t]
    responses = {i: t["tool_result"] for i, t in enumerate(uses)}
    names: list = []
    for t in uses:
        if t["tool_name"] not in names:
            names.append(t["tool_name"])
    key = tok.token_for(TOOL_RESULT_KEY)
    script: list = []
    call = 0
    i = 0
    while i < len(ids):
        script.append(ids[i])
        if ids[i] == key:
            val = tok.tokenize(json.dumps(responses[call], separators=(",", ":"), ensure_ascii=False))
            if ids[i + 1: i + 1 + len(val)] != val:
                raise ValueError(f"tool_result {call} does not re-tokenize in place")
            i += len(val)
            call += 1
        i += 1
    return Trace(script=script, tool_responses=responses, tool_names=names, text=text)


def deep_recursion_doc(levels: int, branching: int, seed: int = 0, text_chars: int = 1) -> str:
    rng = np.random.default_rng(seed)
    letters = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz", dtype=np.uint8)

    def text() -> str:
        return json.dumps(bytes(rng.choice(letters, text_chars)).decode())

    def task(depth: int) -> str:
        s = '{"thought":' + text()
        if depth + 1 < levels:
            s += ',"subtasks":[' + ",".join(task(depth + 1) for _ in range(branching)) + "]"
        return s + ',"conclusion":' + text() + "}"

    return "[" + task(0) + "]"


def load_corpus(path) -> list:
    """A gzip JSON list of canonical documents (tests/golden/corpus_*.json.gz)."""
    with gzip.open(Path(path), "rt", encoding="utf-8") as f:
        return json.load(f)
