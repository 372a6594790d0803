"""Device-resident page-size-1 KV pool (drop-in for threadrun/paging.py).

Layout in HBM (one pool per model):
  K, V        : [layers][capacity][kv_heads][head_dim]  (bf16 or fp32).  One
                token of one layer is a contiguous Hkv*D row (2 KiB of K and
                2 KiB of V at the Qwen3-8B shape), which the decode kernel
                streams with one TMA bulk copy per row.
  free_stack  : int32[capacity], LIFO, initialised [cap-1 .. 0] (paging.py:40)
  owner       : int32[capacity], owner code per page or -1 (paging.py:41)

The device is authoritative for page ids.  The host keeps only the stack
pointer (`free_count`), which is a deterministic function of the planned
alloc/free counts; ids, `allocated` and `free_list` are read back lazily.
`alloc`/`free` here are the reference's per-call API (paging.py:52-67), run
through the same K5 kernel as the batched engine path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .stepdesc import StepDesc

ANY_OWNER = -2


class OutOfPages(RuntimeError):
    def __init__(self, needed: int, available: int):
        self.needed = needed
        self.available = available
        super().__init__(f"need {needed} pages, {available} free")


class DoubleFree(RuntimeError):
    def __init__(self, page_id: int):
        self.page_id = page_id
        super().__init__(f"page {page_id} freed while not allocated")


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


class DevicePagePool:
    """Fixed pool of single-token KV pages on the GPU with a LIFO allocator."""

    def __init__(self, capacity: int, kv_shape: tuple[int, int, int] | None = None,
                 dtype=torch.float32, device: str | torch.device = "cuda"):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        L.load()
        self.capacity = int(capacity)
        self.device = torch.device(device)
        self.dtype = dtype
        self.kv_shape = kv_shape
        self.free_stack = torch.empty(capacity, dtype=torch.int32, device=self.device)
        self.owner = torch.empty(capacity, dtype=torch.int32, device=self.device)
        self.err = torch.zeros(2, dtype=torch.int32, device=self.device)
        # device free-stack pointer + executed-descriptor count (tim_step_account)
        self.acct = torch.tensor([capacity, 0], dtype=torch.int32, device=self.device)
        L.call("tim_pool_init", self.free_stack.data_ptr(), self.owner.data_ptr(), capacity,
               stream_handle())
        self._sp = self.capacity
        self._codes: dict[object, int] = {}
        self._owners: list[object] = []
        self._scratch = None
        # host mirror of `owner` for the per-call API (DoubleFree checks without
        # a device readback); invalidated by the engine's planned ops
        self._owner_host = np.full(capacity, -1, dtype=np.int32)
        self._mirror_valid = True
        self.K_layers = self.V_layers = None
        if kv_shape is not None:
            layers, heads, head_dim = kv_shape
            shape = (layers, capacity, heads, head_dim)
            self.K_layers = torch.zeros(shape, dtype=dtype, device=self.device)
            self.V_layers = torch.zeros(shape, dtype=dtype, device=self.device)

    # ------------------------------------------------------------ views
    @property
    def K(self):
        """Reference-shaped view (capacity, layers, heads, head_dim); writes go through."""
        return None if self.K_layers is None else self.K_layers.permute(1, 0, 2, 3)

    @property
    def V(self):
        return None if self.V_layers is None else self.V_layers.permute(1, 0, 2, 3)

    @property
    def free_count(self) -> int:
        return self._sp

    @property
    def free_list(self) -> list[int]:
        return self.free_stack[: self._sp].cpu().tolist()

    # ---------------------------------------------------------- owners
    def owner_code(self, owner) -> int:
        code = self._codes.get(owner)
        if code is None:
            code = len(self._owners)
            self._codes[owner] = code
            self._owners.append(owner)
        return code

    @property
    def allocated(self) -> dict:
        own = self.owner.cpu().numpy()
        idx = np.nonzero(own >= 0)[0]
        return {int(p): self._owners[int(own[p])] for p in idx}

    def live_tokens(self, request_id) -> int:
        code = self._codes.get(request_id)
        if code is None:
            return 0
        return int((self.owner == code).sum().item())

    def snapshot(self) -> dict:
        per: dict = {}
        alloc = self.allocated
        for o in alloc.values():
            per.setdefault(str(o), {"live_tokens": 0})["live_tokens"] += 1
        return {"capacity": self.capacity, "free": self._sp, "allocated": len(alloc),
                "per_request": per}

    # -------------------------------------------- planned (engine) path
    def plan_alloc(self, sd: StepDesc, slot: int, table_off: int, n: int, owner_code: int) -> None:
        """Reserve n pages for table[slot][table_off:] in the step's op list."""
        if n > self._sp:
            raise OutOfPages(n, self._sp)
        sd.op(L.OP_ALLOC, slot, table_off, n, self._sp, owner_code)
        self._sp -= n

    def plan_free(self, sd: StepDesc, slot: int, table_off: int, n: int, owner_code: int) -> None:
        if self._sp + n > self.capacity:
            raise DoubleFree(-1)
        sd.op(L.OP_FREE, slot, table_off, n, self._sp, owner_code)
        self._sp += n

    def run_ops(self, step_dev: torch.Tensor, tables: torch.Tensor, _percall: bool = False) -> None:
        if not _percall:
            self._mirror_valid = False
        L.call("tim_page_ops", step_dev.data_ptr(), self.free_stack.data_ptr(),
               self.owner.data_ptr(), self.capacity, tables.data_ptr(), tables.shape[1],
               self.err.data_ptr(), stream_handle())
        if _percall:
            self.account(step_dev)

    def account(self, step_dev: torch.Tensor, slot_acct: torch.Tensor | None = None,
                reports: torch.Tensor | None = None) -> None:
        """Device counters of one executed descriptor (tim_step_account)."""
        n_slots = 0 if slot_acct is None else slot_acct.numel() // 2
        L.call("tim_step_account", step_dev.data_ptr(), self.acct.data_ptr(),
               None if slot_acct is None else slot_acct.data_ptr(), n_slots,
               None if reports is None else reports.data_ptr(), 0 if reports is None else reports.shape[0],
               self.err.data_ptr(), stream_handle())

    def check(self) -> None:
        """Synchronise and raise the reference exception for a device error."""
        code = np.zeros(1, dtype=np.int32)
        detail = np.zeros(1, dtype=np.int32)
        L.call("tim_read_error", self.err.data_ptr(), code.ctypes.data, detail.ctypes.data,
               stream_handle())
        raise_device_error(int(code[0]), int(detail[0]))

    # ---------------------------------------------- per-call API (paging.py:52-67)
    def _scratch_row(self, n: int) -> torch.Tensor:
        """(1, >= n + 2) int32: n page ids, then a copy of the error word, so one
        D2H read returns both."""
        if self._scratch is None or self._scratch.shape[1] < n + 2:
            self._scratch = torch.empty((1, max(n + 2, 64)), dtype=torch.int32, device=self.device)
        return self._scratch

    def _owners_host(self) -> np.ndarray:
        if not self._mirror_valid:
            self._owner_host = self.owner.cpu().numpy().copy()
            self._mirror_valid = True
        return self._owner_host

    def _run_percall(self, sd: StepDesc, scratch: torch.Tensor, n: int) -> np.ndarray:
        step = torch.from_numpy(sd.pack()).pin_memory().to(self.device, non_blocking=True)
        self.run_ops(step, scratch, _percall=True)
        scratch[0, n:n + 2].copy_(self.err)
        host = scratch[0, : n + 2].cpu().numpy()  # the one synchronisation of the call
        if host[n] != L.TIM_OK:
            self.err.zero_()
            raise_device_error(int(host[n]), int(host[n + 1]))
        return host[:n]

    def alloc(self, request_id, n: int) -> list[int]:
        if n < 0:
            raise ValueError("n must be >= 0")
        if n > self._sp:
            raise OutOfPages(n, self._sp)
        if n == 0:
            return []
        code = self.owner_code(request_id)
        sd = StepDesc()
        self.plan_alloc(sd, 0, 0, n, code)
        ids = self._run_percall(sd, self._scratch_row(n), n)
        if self._mirror_valid:
            self._owner_host[ids] = code
        return ids.tolist()

    def free(self, page_ids) -> None:
        ids = [int(p) for p in page_ids]
        if not ids:
            return
        own = self._owners_host()
        bad = None
        good = []
        seen = set()
        for pid in ids:  # reference frees in order and stops at the first bad id
            if not (0 <= pid < self.capacity) or own[pid] < 0 or pid in seen:
                bad = pid
                break
            seen.add(pid)
            good.append(pid)
        if good:
            scratch = self._scratch_row(len(good))
            scratch[0, : len(good)].copy_(torch.tensor(good, dtype=torch.int32).pin_memory(),
                                          non_blocking=True)
            sd = StepDesc()
            self.plan_free(sd, 0, 0, len(good), ANY_OWNER)
            self._run_percall(sd, scratch, len(good))
            own[good] = -1
        if bad is not None:
            raise DoubleFree(bad)


# Reference-compatible alias.
PagePool = DevicePagePool


class PageTable:
    """Ordered working-memory index -> page id (paging.py:86-107), host side."""

    def __init__(self, request_id):
        self.request_id = request_id
        self.pages: list[int] = []

    def __len__(self) -> int:
        return len(self.pages)

    def append(self, page_ids) -> None:
        self.pages.extend(page_ids)

    def truncate_from(self, working_index: int) -> list[int]:
        removed = self.pages[working_index:]
        del self.pages[working_index:]
        return removed

    def check(self) -> None:
        if len(set(self.pages)) != len(self.pages):
            raise AssertionError("page table not injective")


class KvPage:
    """View of one page's per-layer key/value states (paging.py:110-116)."""

    def __init__(self, pool: DevicePagePool, page_id: int):
        self.page_id = page_id
        self.k = pool.K[page_id]
        self.v = pool.V[page_id]


def gather(pool: DevicePagePool, table) -> tuple[np.ndarray, np.ndarray]:
    """Working-memory K and V in logical order, (layers, n, heads, dim), as numpy."""
    if pool.K_layers is None:
        raise RuntimeError("accounting-only pool has no KV arrays")
    pages = list(table.pages)
    if not pages:
        raise ValueError("empty page table")
    idx = torch.tensor(pages, dtype=torch.long, device=pool.device)
    k = pool.K_layers.index_select(1, idx).float().cpu().numpy()
    v = pool.V_layers.index_select(1, idx).float().cpu().numpy()
    return k, v


def raise_device_error(code: int, detail: int) -> None:
    if code == L.TIM_OK:
        return
    if code == L.TIM_OUT_OF_PAGES:
        raise OutOfPages(detail, -1)
    if code == L.TIM_DOUBLE_FREE:
        raise DoubleFree(detail)
    if code == L.TIM_SPAN_OUT_OF_RANGE:
        from .pruning import SpanOutOfRange
        raise SpanOutOfRange(f"device prune desync on slot {detail}")
    raise L.TimrunError(code, f"device error detail={detail}")
