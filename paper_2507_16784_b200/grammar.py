"""Grammar tracker and admissible-token masks, native.

`Grammar` / `Tracker` mirror threadrun's ThreadGrammar / Tracker
(tracker.py:177-353): same constructor arguments, `feed(token_id) -> events`,
`allowed_mask() -> TokenMask`, `Rejected` on an inadmissible token.  The byte
machine, the event emission and the memoised masks run in C++
(csrc/grammar.cpp, C ABI in include/timrun.h); Python only marshals.  Masks
carry a stable id (creation order within the grammar) so the engine can keep
them in a device table and pick tokens with tim_masked_argmax.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .structure import (DONE, SUBTASK_LIST_CLOSED, SUBTASK_LIST_OPENED, TASK_CLOSED, TASK_OPENED,
                        THOUGHT_CLOSED, TOOL_PARAMS_READY, TOOL_RESULT_SLOT_OPENED, Rejected,
                        StructureEvent)
from .tokenizer import build_tokenizer

DEFAULT_DEPTH_LIMIT = 16      # schema.py DEFAULT_DEPTH_LIMIT

_KINDS = (TASK_OPENED, THOUGHT_CLOSED, TOOL_PARAMS_READY, TOOL_RESULT_SLOT_OPENED, SUBTASK_LIST_OPENED,
          SUBTASK_LIST_CLOSED, TASK_CLOSED, DONE)


def _packed(items: list[bytes]):
    offs = np.zeros(len(items) + 1, dtype=np.int32)
    for i, b in enumerate(items):
        offs[i + 1] = offs[i] + len(b)
    data = np.frombuffer(b"".join(items) or b"\0", dtype=np.uint8).copy()
    return data, offs


class TokenMask:
    """Admissible next-token ids (tracker.py:128-157) plus the memo id."""

    __slots__ = ("ids", "_set", "_arrays", "mask_id", "can_finish", "finish_ids")

    def __init__(self, ids, mask_id: int = -1, can_finish: bool = False, finish_ids=()):
        self.ids = tuple(sorted(ids))
        self._set = frozenset(self.ids)
        self._arrays: dict[int, np.ndarray] = {}
        self.mask_id = mask_id
        self.can_finish = can_finish
        self.finish_ids = frozenset(finish_ids)

    def admits(self, token_id: int) -> bool:
        return token_id in self._set

    def __contains__(self, token_id: int) -> bool:
        return token_id in self._set

    def __len__(self) -> int:
        return len(self.ids)

    def as_array(self, vocab_size: int) -> np.ndarray:
        arr = self._arrays.get(vocab_size)
        if arr is None:
            arr = np.zeros(vocab_size, dtype=bool)
            arr[[i for i in self.ids if i < vocab_size]] = True
            self._arrays[vocab_size] = arr
        return arr


class Grammar:
    """ThreadGrammar(tools, depth_limit, tokenizer) (tracker.py:177-200)."""

    def __init__(self, tools=(), depth_limit: int = DEFAULT_DEPTH_LIMIT, tokenizer=None):
        if depth_limit < 1:
            raise ValueError("depth_limit must be >= 1")
        names = [t if isinstance(t, str) else t.name for t in tools]
        if len(set(names)) != len(names):
            raise ValueError("tool names must be unique")
        self.tokenizer = tokenizer or build_tokenizer()
        self.depth_limit = depth_limit
        self.tool_names = tuple(names)
        self.json_depth_limit = max(2, 2 * depth_limit)
        lib = L.load()
        pdata, poffs = _packed(list(self.tokenizer.pieces))
        tdata, toffs = _packed([n.encode("utf-8") for n in names])
        self._h = lib.tim_grammar_create(pdata.ctypes.data, poffs.ctypes.data, len(self.tokenizer.pieces),
                                         tdata.ctypes.data, toffs.ctypes.data, len(names), depth_limit)
        if not self._h:
            raise ValueError("tim_grammar_create rejected the grammar")
        self.words = lib.tim_grammar_mask_words(self._h)
        self._masks: list[TokenMask] = []

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                L.load().tim_grammar_destroy(h)
            except Exception:      # interpreter shutdown
                pass
            self._h = None

    def tracker(self) -> "Tracker":
        return Tracker(self)

    @property
    def mask_count(self) -> int:
        return L.load().tim_grammar_mask_count(self._h)

    def mask_words(self, mask_id: int) -> np.ndarray:
        w = np.zeros(self.words, dtype=np.uint32)
        L.load().tim_grammar_mask(self._h, mask_id, w.ctypes.data, None, None)
        return w

    def mask(self, mask_id: int) -> TokenMask:
        while len(self._masks) <= mask_id:
            i = len(self._masks)
            w = np.zeros(self.words, dtype=np.uint32)
            f = np.zeros(self.words, dtype=np.uint32)
            L.load().tim_grammar_mask(self._h, i, w.ctypes.data, f.ctypes.data, None)
            ids = np.nonzero(np.unpackbits(w.view(np.uint8), bitorder="little"))[0]
            fin = np.nonzero(np.unpackbits(f.view(np.uint8), bitorder="little"))[0]
            self._masks.append(TokenMask(ids.tolist(), i, bool(len(fin)), fin.tolist()))
        return self._masks[mask_id]


class Tracker:
    """Mutable parse state over one request's emission stream (tracker.py:206-366)."""

    __slots__ = ("grammar", "_h", "_ne", "_f", "_np", "_nl", "_pp", "_pl")

    def __init__(self, grammar: Grammar, handle=None):
        self.grammar = grammar
        self._h = handle or L.load().tim_tracker_create(grammar._h)
        self._ne = C.c_int32(0)
        self._f = (C.c_int32 * 5)()
        self._np, self._nl = C.c_char_p(), C.c_int32(0)
        self._pp, self._pl = C.c_char_p(), C.c_int32(0)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                L.load().tim_tracker_destroy(h)
            except Exception:      # interpreter shutdown
                pass
            self._h = None

    # -------------------------------------------------------------- state
    def clone(self) -> "Tracker":
        return Tracker(self.grammar, L.load().tim_tracker_clone(self._h))

    deep_copy = clone

    def snapshot(self) -> "Tracker":
        return self.clone()

    def restore(self, snap: "Tracker") -> None:
        """Adopt `snap`'s state (snap must not be used afterwards)."""
        self._h, snap._h = snap._h, self._h

    def _state(self):
        c, d, dep, rb = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        L.load().tim_tracker_state(self._h, C.byref(c), C.byref(d), C.byref(dep), C.byref(rb))
        return c.value, bool(d.value), dep.value, rb.value

    @property
    def consumed(self) -> int:
        return self._state()[0]

    @property
    def done(self) -> bool:
        return self._state()[1]

    def current_depth(self) -> int:
        return self._state()[2]

    # ---------------------------------------------------------------- api
    def feed(self, token_id: int) -> list[StructureEvent]:
        """Consume one token; return the lifecycle events it completed."""
        lib = L.load()
        rc = lib.tim_tracker_feed(self._h, int(token_id), C.byref(self._ne))
        if rc != L.TIM_OK:
            _, _, _, rb = self._state()
            pieces = self.grammar.tokenizer.pieces
            piece = pieces[token_id] if 0 <= token_id < len(pieces) else b""
            ctx = lib.tim_tracker_context(self._h).decode()
            raise Rejected(int(token_id), piece, max(rb, 0), ctx)
        n = self._ne.value
        if n == 0:
            return []
        out = []
        for i in range(n):
            lib.tim_tracker_event(self._h, i, self._f, C.byref(self._np), C.byref(self._nl),
                                  C.byref(self._pp), C.byref(self._pl))
            kind, off, depth, a, b = self._f[0], self._f[1], self._f[2], self._f[3], self._f[4]
            payload = None
            if kind == 5:
                payload = {"span_start": a, "span_end": b}
            elif kind in (2, 3):
                name = C.string_at(self._np, self._nl.value).decode("utf-8")
                params = C.string_at(self._pp, self._pl.value).decode("utf-8")
                payload = {"tool_name": name, "parameters_text": params}
            out.append(StructureEvent(_KINDS[kind], off, depth, payload))
        return out

    def mask_state(self) -> tuple[int, int, bool]:
        """(mask id, admitted count, an admitted token completes the document)."""
        mid, cnt, fin = C.c_int32(), C.c_int32(), C.c_int32()
        L.load().tim_tracker_mask(self._h, C.byref(mid), C.byref(cnt), C.byref(fin))
        return mid.value, cnt.value, bool(fin.value)

    def allowed_mask(self) -> TokenMask:
        """Admissible next tokens; memoised on the machine-state signature."""
        return self.grammar.mask(self.mask_state()[0])
