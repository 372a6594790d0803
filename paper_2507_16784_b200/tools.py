"""Minimal tool plumbing for the engine (drop-in shapes of threadrun/toolhub.py).

Tool I/O is off the attention path (SURVEY §2.1 toolhub row, OUT OF SCOPE);
benchmarks use trace overrides (scheduler.py:469-472).  This module keeps the
call/response/handle contract and a small local registry so requests can
still park on non-blocking tools: ToolCall/ToolResponse/Handle
(toolhub.py:31-88) and a thread-pool hub for local callables
(toolhub.py:102-147, without HTTP endpoints or JSON-schema validation).
"""

from __future__ import annotations

import threading
import time
from concurrent.futures import Future, ThreadPoolExecutor
from dataclasses import dataclass


@dataclass
class ToolSpec:
    name: str
    description: str = ""
    timeout_ms: int = 5000


@dataclass
class ToolCall:
    request_id: str
    call_index: int
    tool_name: str
    parameters: dict
    dispatched_at: float = 0.0
    deadline: float = 0.0


@dataclass
class ToolResponse:
    request_id: str
    call_index: int
    ok: bool
    value: object = None
    error_kind: str | None = None
    error_message: str | None = None
    latency_ms: float = 0.0

    def result_value(self) -> object:
        if self.ok:
            return self.value
        return {"error": f"{self.error_kind}: {self.error_message}"}


class Handle:
    """One in-flight call; poll() is non-blocking and reports a response once."""

    def __init__(self, call: ToolCall, future: Future | None, immediate: ToolResponse | None = None):
        self.call, self.future, self.immediate = call, future, immediate
        self.consumed = False

    def poll(self) -> ToolResponse | None:
        if self.consumed:
            raise RuntimeError("handle already consumed")
        now = time.monotonic()
        if self.immediate is not None:
            self.consumed = True
            return self.immediate
        if self.future.done():
            self.consumed = True
            resp = self.future.result()
            resp.latency_ms = (now - self.call.dispatched_at) * 1000.0
            return resp
        if now > self.call.deadline:
            self.consumed = True
            self.future.cancel()
            ms = int((self.call.deadline - self.call.dispatched_at) * 1000)
            return ToolResponse(self.call.request_id, self.call.call_index, ok=False,
                                error_kind="Timeout", error_message=f"no response within {ms} ms",
                                latency_ms=(now - self.call.dispatched_at) * 1000.0)
        return None


class ToolHub:
    """Registry of local tool callables impl(params, call_index) run on threads."""

    def __init__(self, max_workers: int = 8):
        self._tools: dict = {}
        self._lock = threading.Lock()
        self._pool: ThreadPoolExecutor | None = None
        self._max_workers = max_workers

    def register(self, spec: ToolSpec, impl) -> None:
        with self._lock:
            if spec.name in self._tools:
                raise ValueError(f"duplicate tool {spec.name}")
            self._tools[spec.name] = (spec, impl)

    def dispatch(self, call: ToolCall) -> Handle:
        call.dispatched_at = time.monotonic()
        entry = self._tools.get(call.tool_name)
        if entry is None:
            return Handle(call, None, ToolResponse(call.request_id, call.call_index, ok=False,
                                                   error_kind="UnknownTool",
                                                   error_message=call.tool_name))
        spec, impl = entry
        call.deadline = call.dispatched_at + spec.timeout_ms / 1000.0
        if self._pool is None:
            self._pool = ThreadPoolExecutor(max_workers=self._max_workers)

        def run():
            try:
                return ToolResponse(call.request_id, call.call_index, ok=True,
                                    value=impl(call.parameters, call.call_index))
            except Exception as e:  # tool failure becomes an error result
                return ToolResponse(call.request_id, call.call_index, ok=False,
                                    error_kind=type(e).__name__, error_message=str(e))

        return Handle(call, self._pool.submit(run))
