"""Incremental structure scanner: lifecycle events of a reasoning-tree document.

Host-side producer of the prune input.  It consumes the
generated token stream one token at a time (bytes of each piece through a
small pushdown machine) and emits the reference's lifecycle events at the
same token offsets, depths and payloads as threadrun's Tracker.feed
(tracker.py:301-310, events 33-40):

  TaskOpened(d)            '{' opening a task            (schema.py:198-199)
  ThoughtClosed(d)         closing quote of the thought  (schema.py:201-205)
  ToolParamsReady(d, p)    '}' closing the parameters    (schema.py:214-222)
  ToolResultSlotOpened(d,p) the "tool_result": key       (schema.py:223-231)
  SubtaskListOpened(d+1)   '[' of the subtasks value     (schema.py:236-238)
  SubtaskListClosed(d+1, {span_start, span_end})          (schema.py:244-252)
                           span_start = token of the ',' before "subtasks":
                           (tracker.py:677-679,737-743,756-762), span_end =
                           closing token + 1 (tracker.py:785-796)
  TaskClosed(d)            '}' closing a task
  Done(0)                  ']' closing the document

It does NOT compute admissible-token masks (grammar-constrained sampling is
out of scope for the B200 path, SURVEY §2.1 tracker row); it rejects only
structurally impossible bytes (unbalanced brackets, content outside the
root list), raising `Rejected` like the reference.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

TASK_OPENED = "TaskOpened"
THOUGHT_CLOSED = "ThoughtClosed"
TOOL_PARAMS_READY = "ToolParamsReady"
TOOL_RESULT_SLOT_OPENED = "ToolResultSlotOpened"
SUBTASK_LIST_OPENED = "SubtaskListOpened"
SUBTASK_LIST_CLOSED = "SubtaskListClosed"
TASK_CLOSED = "TaskClosed"
DONE = "Done"


@dataclass
class StructureEvent:
    kind: str
    offset: int
    depth: int
    payload: dict | None = None

    def to_json(self) -> str:
        d = {"kind": self.kind, "offset": self.offset, "depth": self.depth}
        if self.payload is not None:
            d["payload"] = self.payload
        return json.dumps(d, separators=(",", ":"), ensure_ascii=False)


class Rejected(ValueError):
    """Token not admissible (tracker.py:56-65)."""

    def __init__(self, token_id: int, piece: bytes, byte_index: int, context: str):
        self.token_id, self.piece, self.byte_index = token_id, piece, byte_index
        super().__init__(f"token {token_id} ({piece!r}) rejected at piece byte {byte_index}: {context}")


# frame kinds
_ROOT, _LIST, _TASK, _OBJ, _ARR = range(5)
# task phases
_KEY, _COLON, _VALUE, _AFTER = range(4)
_WS = frozenset(b" \t\r\n")
_QUOTE, _BSLASH = 0x22, 0x5C
_SCALAR_END = frozenset(b",}] \t\r\n")


class _Frame:
    __slots__ = ("kind", "depth", "phase", "key", "last_comma", "sub_comma", "tool_name",
                 "params_text", "span_start", "is_root")

    def __init__(self, kind, depth=0):
        self.kind = kind
        self.depth = depth
        self.phase = _KEY
        self.key = b""
        self.last_comma = -1
        self.sub_comma = -1
        self.tool_name = ""
        self.params_text = ""
        self.span_start = -1
        self.is_root = False

    def copy(self) -> "_Frame":
        f = _Frame(self.kind, self.depth)
        for s in self.__slots__:
            setattr(f, s, getattr(self, s))
        return f


class StructureScanner:
    """Feed token ids; get the events each token completes."""

    def __init__(self, tokenizer):
        self.pieces = tokenizer.pieces
        self.frames: list[_Frame] = [_Frame(_ROOT)]
        self.consumed = 0
        self.done = False
        self._in_str = False
        self._esc = False
        self._sink = None         # bytearray collecting string bytes (keys, tool_name)
        self._str_role = 0        # 0 none, 1 task key, 2 task value, 3 generic
        self._scalar = False
        self._capture = None      # bytearray capturing the parameters object
        self._cap_depth = 0
        self._tok = 0
        self._events: list = []

    # ------------------------------------------------------------------ api
    @property
    def depth(self) -> int:
        for f in reversed(self.frames):
            if f.kind == _TASK:
                return f.depth
        return 0

    def snapshot(self):
        return ([f.copy() for f in self.frames], self.consumed, self.done, self._in_str, self._esc,
                None if self._sink is None else bytearray(self._sink), self._str_role,
                self._scalar, None if self._capture is None else bytearray(self._capture),
                self._cap_depth)

    def restore(self, snap) -> None:
        (frames, self.consumed, self.done, self._in_str, self._esc, sink, self._str_role,
         self._scalar, cap, self._cap_depth) = snap
        self.frames = frames
        self._sink, self._capture = sink, cap

    def feed(self, token_id: int) -> list[StructureEvent]:
        piece = self.pieces[token_id]
        self._tok = self.consumed
        self._events = []
        # fast path: plain string content (the bulk of every document)
        if self._in_str and not self._esc and len(piece) == 1:
            b = piece[0]
            if b != _QUOTE and b != _BSLASH:
                if self._sink is not None:
                    self._sink.append(b)
                if self._capture is not None:
                    self._capture.append(b)
                self.consumed += 1
                return self._events
        for i, b in enumerate(piece):
            if not self._byte(b):
                raise Rejected(token_id, piece, i, self._context())
        self.consumed += 1
        return self._events

    def feed_all(self, ids) -> list[StructureEvent]:
        out = []
        for t in ids:
            out.extend(self.feed(t))
        return out

    # ------------------------------------------------------------- internals
    def _context(self) -> str:
        if self.done:
            return "document already complete"
        names = {_ROOT: "root", _LIST: "list", _TASK: "task", _OBJ: "object", _ARR: "array"}
        return f"in {names[self.frames[-1].kind]}" + (" inside string" if self._in_str else "")

    def _emit(self, kind, depth, payload=None):
        self._events.append(StructureEvent(kind, self._tok, depth, payload))

    def _byte(self, b: int) -> bool:
        if self.done:
            return False
        if self._capture is not None:
            self._capture.append(b)
        if self._in_str:
            if self._esc:
                self._esc = False
            elif b == _BSLASH:
                self._esc = True
            elif b == _QUOTE:
                self._in_str = False
                self._end_string()
                return True
            if self._sink is not None:
                self._sink.append(b)
            return True
        if self._scalar:
            if b not in _SCALAR_END:
                return True
            self._scalar = False
            self._value_done()
            # fall through: the delimiter is structural
        if b in _WS:
            return True
        f = self.frames[-1]
        k = f.kind
        if k == _TASK:
            return self._task_byte(f, b)
        if k == _LIST:
            return self._list_byte(f, b)
        if k == _OBJ or k == _ARR:
            return self._generic_byte(f, b)
        # root: the document must open with '['
        if b == 0x5B:
            lst = _Frame(_LIST, 0)
            lst.is_root = True
            lst.phase = _VALUE
            self.frames[-1] = lst
            return True
        return False

    def _start_string(self, role, sink):
        self._in_str = True
        self._esc = False
        self._str_role = role
        self._sink = sink

    def _end_string(self):
        role = self._str_role
        f = self.frames[-1]
        if role == 1:                      # task key finished, expect ':'
            f.key = bytes(self._sink)
            f.phase = _COLON
        elif role == 2:                    # task string value finished
            if f.key == b"thought":
                self._emit(THOUGHT_CLOSED, f.depth)
            elif f.key == b"tool_name":
                f.tool_name = self._sink.decode("utf-8", "replace")
            f.phase = _AFTER
        else:
            self._value_done_generic(f)
        self._sink = None
        self._str_role = 0

    def _value_done(self):
        f = self.frames[-1]
        if f.kind == _TASK:
            f.phase = _AFTER
        else:
            self._value_done_generic(f)

    @staticmethod
    def _value_done_generic(f):
        if f.kind == _OBJ:
            # generic object alternates key/value; phase toggled by ':' and ','
            if f.phase == _VALUE:
                f.phase = _AFTER
        elif f.kind == _ARR:
            f.phase = _AFTER

    def _task_byte(self, f: _Frame, b: int) -> bool:
        ph = f.phase
        if ph == _KEY:
            if b == _QUOTE:
                self._start_string(1, bytearray())
                return True
            return False
        if ph == _COLON:
            if b != 0x3A:
                return False
            f.phase = _VALUE
            if f.key == b"tool_result":
                self._emit(TOOL_RESULT_SLOT_OPENED, f.depth,
                           {"tool_name": f.tool_name, "parameters_text": f.params_text})
            elif f.key == b"subtasks":
                f.sub_comma = f.last_comma
            return True
        if ph == _VALUE:
            if b == _QUOTE:
                self._start_string(2, bytearray() if f.key == b"tool_name" else None)
                return True
            if b == 0x7B:  # {
                self.frames.append(_Frame(_OBJ, f.depth))
                self.frames[-1].phase = _KEY
                if f.key == b"parameters":
                    self._capture = bytearray(b"{")
                    self._cap_depth = len(self.frames)
                return True
            if b == 0x5B:  # [
                if f.key == b"subtasks":
                    lst = _Frame(_LIST, f.depth + 1)
                    lst.span_start = f.sub_comma
                    lst.phase = _VALUE
                    self.frames.append(lst)
                    self._emit(SUBTASK_LIST_OPENED, f.depth + 1)
                else:
                    a = _Frame(_ARR, f.depth)
                    a.phase = _VALUE
                    self.frames.append(a)
                return True
            if b in b"}],:":
                return False
            self._scalar = True
            return True
        # _AFTER: ',' or '}'
        if b == 0x2C:
            f.last_comma = self._tok
            f.phase = _KEY
            return True
        if b == 0x7D:
            self._emit(TASK_CLOSED, f.depth)
            self.frames.pop()
            parent = self.frames[-1]
            parent.phase = _AFTER
            return True
        return False

    def _list_byte(self, f: _Frame, b: int) -> bool:
        if f.phase == _VALUE:                       # expecting a task
            if b == 0x7B:
                self.frames.append(_Frame(_TASK, f.depth))
                self._emit(TASK_OPENED, f.depth)
                return True
            return False
        if b == 0x2C:
            f.phase = _VALUE
            return True
        if b == 0x5D:
            self.frames.pop()
            if f.is_root:
                self._emit(DONE, 0)
                self.done = True
            else:
                self._emit(SUBTASK_LIST_CLOSED, f.depth,
                           {"span_start": f.span_start, "span_end": self._tok + 1})
                self.frames[-1].phase = _AFTER
            return True
        return False

    def _generic_byte(self, f: _Frame, b: int) -> bool:
        close = 0x7D if f.kind == _OBJ else 0x5D
        if b == close:
            self.frames.pop()
            if self._capture is not None and len(self.frames) + 1 == self._cap_depth:
                parent = self.frames[-1]
                parent.params_text = self._capture.decode("utf-8", "replace")
                self._capture = None
                self._emit(TOOL_PARAMS_READY, parent.depth,
                           {"tool_name": parent.tool_name, "parameters_text": parent.params_text})
            self._value_done()
            return True
        if b == 0x7D or b == 0x5D:
            return False
        if b == _QUOTE:
            self._start_string(3, None)
            return True
        if b == 0x3A:
            if f.kind == _OBJ:
                f.phase = _VALUE
            return True
        if b == 0x2C:
            f.phase = _KEY if f.kind == _OBJ else _VALUE
            return True
        if b == 0x7B:
            o = _Frame(_OBJ, f.depth)
            o.phase = _KEY
            self.frames.append(o)
            return True
        if b == 0x5B:
            a = _Frame(_ARR, f.depth)
            a.phase = _VALUE
            self.frames.append(a)
            return True
        self._scalar = True
        return True
