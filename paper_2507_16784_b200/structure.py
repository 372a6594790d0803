"""Lifecycle events of a reasoning-tree document and the Rejected error
(tracker.py:33-65): the types the native grammar tracker (grammar.py,
csrc/grammar.cpp) reports.

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
