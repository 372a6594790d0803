"""Model backends on the B200 (drop-in for threadrun/model.py) and the step runtime.

`B200Transformer` implements the reference backend protocol (position_limit,
make_pool, prefill, extend, decode_step; model.py:115-183) with the same
arithmetic as TinyTransformer (weightless RMSNorm, rotate-half RoPE, causal
attention over page-size-1 pages, non-gated SiLU MLP, tied logits), extended
with GQA (`kv_heads`) and an MLP width field (`mlp_dim`) for the Qwen3-8B
shaped configuration.  With weight_init="reference" the weights are drawn from
the reference's numpy RNG stream (model.py:87-103), so fp32 runs reproduce the
reference to rounding.

`StepRuntime` owns the device state of a batched engine: block tables, live
lists and logical token streams per request slot, row buffers, activations
and the decode workspace.  One engine step = one descriptor upload + K4
(prune compaction) + K5 (page ops) + row staging + one batched forward over
every request's new tokens (mixed decode / re-encode / prefill rows).
GEMMs go to cuBLAS through torch; attention, RoPE+KV store, paging and the
per-row kernels are libtimrun.
"""

from __future__ import annotations

import ctypes
import json
import math
import os
from dataclasses import asdict, dataclass
from pathlib import Path

import numpy as np
import torch

from . import _lib as L
from .paging import DevicePagePool, PageTable, raise_device_error, stream_handle
from .stepdesc import StepDesc


class PositionOverflow(RuntimeError):
    def __init__(self, position: int, limit: int):
        super().__init__(f"position {position} >= limit {limit}")
        self.position = position
        self.limit = limit


class EmptyExtend(ValueError):
    pass


class EmptyMask(RuntimeError):
    """Grammar dead end: no token admissible."""


@dataclass
class ModelConfig:
    layers: int = 2
    heads: int = 4
    head_dim: int = 16
    vocab: int = 512
    position_limit: int = 256
    rope_base: float = 10000.0
    seed: int = 0
    precision: str = "float32"       # "float32" | "bfloat16"
    kv_heads: int = 0                # 0: same as heads (reference)
    mlp_dim: int = 0                 # 0: 4 * model_dim (reference)
    weight_init: str = "reference"   # "reference" (numpy stream) | "device" (torch RNG on GPU)

    @property
    def model_dim(self) -> int:
        return self.heads * self.head_dim

    @property
    def n_kv(self) -> int:
        return self.kv_heads or self.heads

    @property
    def n_mlp(self) -> int:
        return self.mlp_dim or 4 * self.model_dim

    @property
    def dtype(self):
        return np.float64 if self.precision == "float64" else np.float32

    @property
    def torch_dtype(self):
        return {"float32": torch.float32, "bfloat16": torch.bfloat16}[self.precision]

    @property
    def tim_dtype(self) -> int:
        return L.DTYPE_BF16 if self.precision == "bfloat16" else L.DTYPE_F32

    def kv_shape(self) -> tuple[int, int, int]:
        return (self.layers, self.n_kv, self.head_dim)

    def kv_bytes_per_token(self) -> int:
        """K + V bytes of one working-memory token over all layers."""
        return 2 * self.layers * self.n_kv * self.head_dim * (2 if self.precision == "bfloat16" else 4)

    def to_json_file(self, path) -> None:
        Path(path).write_text(json.dumps(asdict(self), indent=2))

    @classmethod
    def from_json_file(cls, path) -> "ModelConfig":
        return cls(**json.loads(Path(path).read_text()))


def qwen3_8b_shape(**over) -> ModelConfig:
    """Qwen3-8B-shaped TIM decoder (BASELINE config 2): 36 layers, hidden 4096,
    32 q / 8 kv heads of 128, MLP 12288, rope base 1e6, bf16, vocab 512."""
    kw = dict(layers=36, heads=32, kv_heads=8, head_dim=128, mlp_dim=12288, vocab=512,
              position_limit=40960, rope_base=1e6, precision="bfloat16", weight_init="device")
    kw.update(over)
    return ModelConfig(**kw)


def _reference_weights(cfg: ModelConfig):
    """numpy draw in the order of model.py:91-103 (emb, then wq wk wv wo w1 w2 per layer)."""
    dm = cfg.model_dim
    rng = np.random.default_rng(cfg.seed)
    scale = 1.0 / np.sqrt(dm)

    def mat(*shape):
        return (rng.standard_normal(shape) * scale).astype(np.float32)

    emb = mat(cfg.vocab, dm)
    kvd = cfg.n_kv * cfg.head_dim
    layers = []
    for _ in range(cfg.layers):
        layers.append([mat(dm, dm), mat(dm, kvd), mat(dm, kvd), mat(dm, dm),
                       mat(dm, cfg.n_mlp), mat(cfg.n_mlp, dm)])
    return emb, layers


def _rope_tables(cfg: ModelConfig):
    """cos/sin of the fp32 angle pos*inv_freq, inv_freq built as model.py:104-105."""
    half = cfg.head_dim // 2
    inv = (cfg.rope_base ** (-np.arange(half) / half)).astype(np.float32)
    pos = np.arange(cfg.position_limit, dtype=np.float32)
    ang = pos[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


class StepRuntime:
    """Device state + executor of batched engine steps for one pool."""

    def __init__(self, model, pool: DevicePagePool, max_slots: int, logical_cap: int):
        self.model = model
        self.pool = pool
        self.dev = pool.device
        P = model.position_limit
        self.max_slots = max_slots
        self.scratch_slot = max_slots
        S = max_slots + 1
        self.tables = torch.full((S, P), -1, dtype=torch.int32, device=self.dev)
        self.live = torch.zeros((S, P), dtype=torch.int32, device=self.dev)
        self.logical = torch.zeros((S, max(logical_cap, 1)), dtype=torch.int32, device=self.dev)
        self.counters = torch.zeros(S + 1, dtype=torch.int32, device=self.dev)
        self._rows = 0
        self._step_cap = 0
        self.step_dev = None
        self.step_host = None
        self.sms = L.load().tim_sm_count()
        self.serial = 0              # step serial stamped into descriptors (attention plan)
        self.last_tokens = None
        self.last_logits = None
        self.launches = 0
        self._last_upload_bytes = 0
        self.use_graphs = (model is not None and getattr(model, "has_weights", False) and max_slots > 0
                           and os.environ.get("TIMRUN_GRAPHS", "1") != "0")
        self.graphs: dict = {}
        self.graph_pool = None
        self.gstep = None
        self.recording = None        # list -> record descriptors instead of executing
        self.prologue_events = None  # list -> CUDA events around K4 + K5 + staging
        self.phase_events = None     # list -> CUDA events around pre / attn0 / post (diagnostics)
        self.attn_events = None      # list -> CUDA events around layer-0 decode attention
        # admissible-token masks of unscripted picks (grammar.py), by device id;
        # a fixed buffer, so captured graphs keep their address
        self.mask_words = (getattr(model, "vocab_size", 512) + 31) // 32 if model is not None else 16
        self.masks = torch.zeros((self.MASK_CAP, self.mask_words), dtype=torch.int32, device=self.dev)
        self.n_masks = 0
        # StepReport / metrics from device counters (tim_step_account): per slot
        # table length + high-water mark, and a ring of per-descriptor records
        self.slot_acct = torch.zeros(2 * max(max_slots, 1), dtype=torch.int32, device=self.dev)
        self.reports = torch.zeros((self.REPORT_RING, 4 + 3 * max(max_slots, 1)), dtype=torch.int32,
                                   device=self.dev)

    REPORT_RING = 1024

    MASK_CAP = 1 << 14

    def add_mask(self, words: np.ndarray) -> int:
        """Store one admissible-token bitmask on the device; returns its id."""
        if self.n_masks >= self.MASK_CAP:
            raise RuntimeError("device mask table full (raise StepRuntime.MASK_CAP)")
        row = np.zeros(self.mask_words, dtype=np.uint32)
        n = min(len(words), self.mask_words)
        row[:n] = words[:n]
        self.masks[self.n_masks].copy_(torch.from_numpy(row.view(np.int32)))
        self.n_masks += 1
        return self.n_masks - 1

    # ----------------------------------------------------------- buffers
    def grow_logical(self, n: int) -> None:
        """Reallocate the per-slot token streams to hold n indices (doubling).
        Only eager kernels (K4, row staging) read this buffer, so no captured
        graph holds its address."""
        cap = self.logical.shape[1]
        if n <= cap:
            return
        new_cap = max(n, 2 * cap)
        buf = torch.zeros((self.logical.shape[0], new_cap), dtype=torch.int32, device=self.dev)
        buf[:, :cap] = self.logical
        self.logical = buf

    def _ensure_rows(self, n: int) -> None:
        if n <= self._rows:
            return
        R = 1 << max(6, (n - 1).bit_length())
        if self.use_graphs:
            R = max(R, self.GRAPH_BUCKETS[-1])
            self.graphs = {}          # captured graphs point at the old buffers
        d = self.dev
        self.row_tokens = torch.zeros(R, dtype=torch.int32, device=d)
        self.row_pages = torch.full((R,), -1, dtype=torch.int32, device=d)
        self.row_pos = torch.zeros(R, dtype=torch.int32, device=d)
        if self.model is not None and self.model.has_weights:
            self.model.alloc_activations(self, R)
        self._rows = R

    def upload(self, arr: np.ndarray) -> torch.Tensor:
        """Copy a packed descriptor to the device through a ring of pinned
        buffers; a buffer is rewritten only after its previous copy completed."""
        n = arr.size
        if n > self._step_cap:
            cap = 1 << max(10, (n - 1).bit_length())
            self._ring = [torch.empty(cap, dtype=torch.int32, pin_memory=True) for _ in range(4)]
            self._ring_ev = [None] * 4
            self._ring_i = 0
            self.step_dev = torch.empty(cap, dtype=torch.int32, device=self.dev)
            self._step_cap = cap
        i = self._ring_i
        self._ring_i = (i + 1) % len(self._ring)
        ev = self._ring_ev[i]
        if ev is not None:
            ev.synchronize()
        host = self._ring[i]
        host[:n].numpy()[:] = arr
        self._last_upload_bytes = n * 4
        self.step_dev[:n].copy_(host[:n], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._ring_ev[i] = ev
        return self.step_dev[:n]

    # -------------------------------------------------------------- step
    # Row buckets of the captured forward graphs.  Fine-grained because steps
    # with re-encode / tool rows are GEMM-compute heavy (~10 GFLOP per row over
    # 36 layers at the C2 shape): padding 300 rows to 512 would cost ~40 %.
    # Larger steps run eagerly at their exact row count.
    GRAPH_BUCKETS = (64, 96, 128, 160, 192, 224, 256, 320, 384, 448, 512, 640, 768, 896, 1024,
                     1280, 1536, 1792, 2048, 2560, 3072, 3584, 4096)

    def graph_bucket(self, n_rows: int):
        if not self.use_graphs:
            return None
        for b in self.GRAPH_BUCKETS:
            if n_rows <= b:
                return b
        return None

    def precapture(self) -> None:
        """Capture every (row bucket, has-extend) forward graph up front, on a
        sanitised empty step (no rows: page -1 everywhere, no decode/extend
        work), so no capture ever lands inside a timed region."""
        if not self.use_graphs:
            return
        self._ensure_rows(self.GRAPH_BUCKETS[-1])
        for b in self.GRAPH_BUCKETS:
            sd = StepDesc()
            sd.rows_pad = b
            sd.last_pad = self.max_slots
            arr = sd.pack()
            if self.gstep is None or self.gstep.numel() < arr.size:
                self.gstep = torch.zeros(1 << 16, dtype=torch.int32, device=self.dev)
            self.gstep[: arr.size].copy_(torch.from_numpy(arr))
            L.call("tim_stage_rows", self.gstep.data_ptr(), self.tables.data_ptr(),
                   self.tables.shape[1], self.live.data_ptr(), self.live.shape[1],
                   self.logical.data_ptr(), self.logical.shape[1], self.row_tokens.data_ptr(),
                   self.row_pages.data_ptr(), self.row_pos.data_ptr(), stream_handle())
            for has_ext in (False, True):
                if (b, has_ext) not in self.graphs:
                    self.graphs[(b, has_ext)] = self.model._capture(self, b, self.max_slots, has_ext)
        torch.cuda.synchronize()

    def run_step(self, sd: StepDesc, forward: bool = True):
        """Execute one planned step; returns the greedy tokens of sd.last rows
        (device tensor) or None when there is nothing to encode.  In record
        mode the packed descriptor is only stored (see replay)."""
        b = self.graph_bucket(sd.n_rows) if forward and sd.n_rows else None
        if b is not None:
            sd.rows_pad = b
            sd.last_pad = self.max_slots
        sd.ctas = self.sms
        self.serial = (self.serial % 0x7FFFFFFF) + 1
        sd.serial = self.serial
        arr = sd.pack()
        self._ensure_rows(max(sd.rows_pad or sd.n_rows, 1))
        if self.gstep is None or self.gstep.numel() < arr.size:
            if self.use_graphs:
                self.gstep = torch.zeros(max(1 << 16, 1 << (arr.size - 1).bit_length()),
                                         dtype=torch.int32, device=self.dev)
                self.graphs = {}
                self.graph_pool = torch.cuda.graph_pool_handle()
        if self.recording is not None:
            self.recording.append((sd, arr, forward))
            return None
        return self._execute(sd, self.upload(arr), forward)

    def _execute(self, sd: StepDesc, step: torch.Tensor, forward: bool):
        st = stream_handle()
        tstride = self.tables.shape[1]
        pev = self.prologue_events
        if pev is not None:
            p0 = torch.cuda.Event(enable_timing=True)
            p0.record()
        if sd.jobs:
            L.call("tim_prune_compact", step.data_ptr(), len(sd.jobs), self.live.data_ptr(),
                   self.live.shape[1], self.logical.data_ptr(), self.logical.shape[1],
                   self.row_tokens.data_ptr(), self.pool.err.data_ptr(), st)
            self.launches += 1
        if sd.ops:
            self.pool.run_ops(step, self.tables)
            self.launches += 1
        if sd.new or sd.n_rows:
            L.call("tim_stage_rows", step.data_ptr(), self.tables.data_ptr(), tstride,
                   self.live.data_ptr(), self.live.shape[1], self.logical.data_ptr(),
                   self.logical.shape[1], self.row_tokens.data_ptr(), self.row_pages.data_ptr(),
                   self.row_pos.data_ptr(), st)
            self.launches += 2
        if sd.ops or sd.new or sd.n_rows:
            self.pool.account(step, self.slot_acct if self.max_slots > 0 else None,
                              self.reports if self.max_slots > 0 else None)
            self.launches += 1
        if pev is not None:
            p1 = torch.cuda.Event(enable_timing=True)
            p1.record()
            pev.append((p0, p1, sd))
        if not forward or sd.n_rows == 0 or self.model is None or not self.model.has_weights:
            return None
        return self.model.forward_rows(self, step, sd)

    def replay_upload(self, records) -> list:
        """Make recorded descriptors device-resident (one buffer, one copy)."""
        offs, total = [], 0
        for _, arr, _ in records:
            offs.append(total)
            total += (arr.size + 31) // 32 * 32
        host = np.zeros(max(total, 1), dtype=np.int32)
        for (_, arr, _), o in zip(records, offs):
            host[o:o + arr.size] = arr
        dev = torch.from_numpy(host).to(self.dev)
        return [(sd, dev[o:o + arr.size], fw) for (sd, arr, fw), o in zip(records, offs)]

    def replay(self, resident) -> None:
        for sd, step, fw in resident:
            self._execute(sd, step, fw)

    def check(self) -> None:
        self.pool.check()

    def device_reports(self) -> list[dict]:
        """The device's per-descriptor records still in the ring, oldest first:
        {serial, pages_free, flops_units, slots: [(table_len, decoded, max_cache)]}."""
        acct = self.pool.acct.cpu().tolist()
        n = acct[1]
        ring = self.reports.cpu().numpy()
        out = []
        for k in range(max(0, n - self.REPORT_RING), n):
            r = ring[k % self.REPORT_RING]
            S = (r.size - 4) // 3
            out.append({"serial": int(r[0]), "pages_free": int(r[1]),
                        "flops_units": int(r[2]) & 0xFFFFFFFF | (int(r[3]) << 32),
                        "slots": r[4:4 + 3 * S].reshape(S, 3).tolist()})
        return out


class B200Transformer:
    """TinyTransformer-compatible backend running on libtimrun + cuBLAS."""

    has_weights = True

    def __init__(self, config: ModelConfig, device: str = "cuda"):
        if config.precision not in ("float32", "bfloat16"):
            raise NotImplementedError(f"precision {config.precision!r} is not supported on the B200 path")
        L.load()
        self.config = cfg = config
        self.dev = torch.device(device)
        dt = cfg.torch_dtype
        dm, D, hq, hkv = cfg.model_dim, cfg.head_dim, cfg.heads, cfg.n_kv
        if cfg.precision == "float32":
            torch.backends.cuda.matmul.allow_tf32 = False
            torch.backends.cudnn.allow_tf32 = False
        # Projection weights are stored transposed ([out, in], K contiguous): an
        # output-column block is then one contiguous slab for the decode GEMM's
        # TMA weight stream; `wqkv[li]` etc. remain the reference's [in, out].
        if cfg.weight_init == "reference":
            emb, layers = _reference_weights(cfg)
            self.emb = torch.from_numpy(emb).to(self.dev, dt)
            self.wqkv_t, self.wo_t, self.w1_t, self.w2_t = [], [], [], []
            for wq, wk, wv, wo, w1, w2 in layers:
                qkv = np.concatenate([wq, wk, wv], axis=1)
                self.wqkv_t.append(torch.from_numpy(np.ascontiguousarray(qkv.T)).to(self.dev, dt))
                self.wo_t.append(torch.from_numpy(np.ascontiguousarray(wo.T)).to(self.dev, dt))
                self.w1_t.append(torch.from_numpy(np.ascontiguousarray(w1.T)).to(self.dev, dt))
                self.w2_t.append(torch.from_numpy(np.ascontiguousarray(w2.T)).to(self.dev, dt))
        else:
            g = torch.Generator(device=self.dev).manual_seed(cfg.seed)
            sc = 1.0 / math.sqrt(dm)

            def mat(*shape):
                return (torch.randn(*shape, generator=g, device=self.dev, dtype=torch.float32) * sc).to(dt)

            self.emb = mat(cfg.vocab, dm)
            W = (hq + 2 * hkv) * D
            self.wqkv_t = [mat(W, dm) for _ in range(cfg.layers)]
            self.wo_t = [mat(dm, dm) for _ in range(cfg.layers)]
            self.w1_t = [mat(cfg.n_mlp, dm) for _ in range(cfg.layers)]
            self.w2_t = [mat(dm, cfg.n_mlp) for _ in range(cfg.layers)]
        self.wqkv = [w.t() for w in self.wqkv_t]
        self.wo = [w.t() for w in self.wo_t]
        self.w1 = [w.t() for w in self.w1_t]
        self.w2 = [w.t() for w in self.w2_t]
        self.emb_t = self.emb.t().contiguous()     # tied LM head (model.py:164)
        cos, sin = _rope_tables(cfg)
        self.cos = torch.from_numpy(cos).to(self.dev)
        self.sin = torch.from_numpy(sin).to(self.dev)
        self.scale = 1.0 / math.sqrt(D)
        self.tensor_cores = (cfg.precision == "bfloat16" and L.load().tim_extend_queries_per_item(
            hq, hkv, D, L.DTYPE_BF16) < (1 << 30))
        self.tile_q = 16 // (hq // hkv) if self.tensor_cores else 0   # queries per mode-0 tile
        # multi-token rows go to the tcgen05 kernel (mode 1) when the shape has
        # one: an item = ext_q queries x the q heads of one kv head (two 128-row
        # MMA tiles sharing each K/V block)
        qpi = L.load().tim_extend_queries_per_item(hq, hkv, D, L.DTYPE_BF16) if self.tensor_cores else 0
        self.ext_q = qpi if self.tensor_cores and qpi * (hq // hkv) in (128, 256) else 0
        self.ext_groups = L.load().tim_extend_head_groups(hq, hkv, D) if self.ext_q else 0
        self._runtimes: dict[int, StepRuntime] = {}

    # Diagnostics only (bench ablation of kernel classes; results are garbage):
    # TIMRUN_DIAG_SKIP=gemm,rope,silu,attn drops those launches from the step.
    _DIAG_SKIP = frozenset(x for x in os.environ.get("TIMRUN_DIAG_SKIP", "").split(",") if x)

    def _gemm(self, rt, li: int, which: int, x, y, res, T: int) -> int:
        """y (+)= x @ W for projection `which` (0 qkv, 1 o, 2 up, 3 down) on
        cuBLAS (a tcgen05 weight-streaming kernel for <= 64 rows was measured
        slower)."""
        if "gemm" in self._DIAG_SKIP:
            return 0
        wt = (self.wqkv_t, self.wo_t, self.w1_t, self.w2_t)[which][li]
        if res is None:
            torch.matmul(x[:T], wt.t(), out=y[:T])
        else:
            y[:T].addmm_(x[:T], wt.t())
        return 0

    # ------------------------------------------------------- protocol
    @property
    def vocab_size(self) -> int:
        return self.config.vocab

    @property
    def position_limit(self) -> int:
        return self.config.position_limit

    def make_pool(self, capacity: int) -> DevicePagePool:
        return DevicePagePool(capacity, kv_shape=self.config.kv_shape(),
                              dtype=self.config.torch_dtype, device=self.dev)

    def runtime(self, pool: DevicePagePool, max_slots: int, logical_cap: int) -> StepRuntime:
        return StepRuntime(self, pool, max_slots, logical_cap)

    def weight_bytes(self) -> int:
        t = [self.emb] + self.wqkv_t + self.wo_t + self.w1_t + self.w2_t
        return sum(x.numel() * x.element_size() for x in t)

    def _protocol_runtime(self, pool: DevicePagePool) -> StepRuntime:
        rt = self._runtimes.get(id(pool))
        if rt is None or rt.pool is not pool:
            rt = StepRuntime(self, pool, 0, 1)
            self._runtimes[id(pool)] = rt
        return rt

    def _forward(self, tokens, positions, table: PageTable, pool: DevicePagePool):
        cfg = self.config
        n = len(tokens)
        for p in positions:
            if p >= cfg.position_limit:
                raise PositionOverflow(int(p), cfg.position_limit)
        new_pages = pool.alloc(table.request_id, n)
        rt = self._protocol_runtime(pool)
        m = len(table.pages)
        pages = list(table.pages) + new_pages
        rt._ensure_rows(n)
        rt.tables[rt.scratch_slot, : m + n] = torch.tensor(pages, dtype=torch.int32, device=self.dev)
        rt.row_tokens[:n] = torch.tensor(tokens, dtype=torch.int32, device=self.dev)
        rt.row_pages[:n] = torch.tensor(new_pages, dtype=torch.int32, device=self.dev)
        rt.row_pos[:n] = torch.tensor([int(p) for p in positions], dtype=torch.int32, device=self.dev)
        sd = StepDesc()
        sd.n_rows = n
        self.plan_attention(sd, rt.scratch_slot, m, n, 0)
        sd.last.append(n - 1)
        sd.ctas = rt.sms
        rt.serial = (rt.serial % 0x7FFFFFFF) + 1
        sd.serial = rt.serial
        step = rt.upload(sd.pack())
        self.forward_rows(rt, step, sd)
        table.append(new_pages)
        return rt.last_logits[0].cpu().numpy()

    def prefill(self, tokens, positions, table, pool):
        if len(tokens) != len(positions):
            raise ValueError("tokens and positions must align")
        if not tokens:
            raise EmptyExtend("nothing to prefill")
        return self._forward(list(tokens), list(positions), table, pool)

    def extend(self, tokens, start_position, table, pool):
        if not tokens:
            raise EmptyExtend("nothing to extend")
        return self._forward(list(tokens), list(range(start_position, start_position + len(tokens))),
                             table, pool)

    def decode_step(self, last_token, position, table, pool):
        return self._forward([last_token], [position], table, pool)

    # ------------------------------------------------------ batched path
    EXT_MIN_ROWS = 8

    def plan_attention(self, sd: StepDesc, slot: int, m: int, n: int, row_off: int) -> None:
        """Attention work records for one segment: decode tiles (mode 0) for
        single rows and short segments, tcgen05 items (mode 1) for longer ones."""
        sd.segs.append((slot, m, n, row_off))
        if not self.tensor_cores:
            return
        if self.ext_q and n >= self.EXT_MIN_ROWS:
            # re-encode / tool / prefill segment: tcgen05 items of ext_q queries
            # x one kv head (K/V slice streamed once per ext_q queries)
            for q0 in range(0, n, self.ext_q):
                nq = min(self.ext_q, n - q0)
                for g in range(self.ext_groups):
                    sd.ext.append((row_off + q0, slot, m + q0 + nq, nq, m, g))
            return
        # Decode rows and short segments: the split-K decode-tile kernel (mode 0),
        # tiles of tile_q consecutive queries x all kv heads.
        tq = self.tile_q
        for q0 in range(0, n, tq):
            nq = min(tq, n - q0)
            sd.dec.append((row_off + q0, slot, m + q0 + nq, nq, m, 0))

    def alloc_activations(self, rt: StepRuntime, R: int) -> None:
        cfg = self.config
        dt, d = cfg.torch_dtype, self.dev
        dm, D = cfg.model_dim, cfg.head_dim
        W = (cfg.heads + 2 * cfg.n_kv) * D
        rt.h = torch.zeros(R, dm, dtype=dt, device=d)
        rt.qkv = torch.zeros(R, W, dtype=dt, device=d)
        rt.q = torch.zeros(R, cfg.heads * D, dtype=dt, device=d)
        rt.ctx = torch.zeros(R, cfg.heads * D, dtype=dt, device=d)
        rt.u = torch.zeros(R, cfg.n_mlp, dtype=dt, device=d)
        n_ctas = max(rt.sms, 1)
        rt.n_ctas = n_ctas
        rt.max_dec = R
        rt.ws = torch.zeros(L.load().tim_decode_ws_floats(n_ctas, R, cfg.n_kv, D), device=d)
        rt.counters = torch.zeros(R * 8, dtype=torch.int32, device=d)

    # The forward is split in three phases so that a decode step can run as
    # two captured CUDA graphs around one eagerly launched layer-0 attention
    # (which bench.py brackets with CUDA events for the live roofline figure).
    def _pre(self, rt: StepRuntime, sp: int, T: int) -> int:
        cfg, st, td = self.config, stream_handle(), self.config.tim_dtype
        dm = cfg.model_dim
        h = rt.h[:T]
        if self.tensor_cores:   # decode-tile partition of this step, shared by all layers
            L.call("tim_attn_plan", sp, rt.tables.data_ptr(), rt.tables.shape[1], rt.n_ctas, rt.max_dec,
                   cfg.head_dim, rt.ws.data_ptr(), st)
        L.call("tim_embed", rt.row_tokens.data_ptr(), T, self.emb.data_ptr(), dm, h.data_ptr(), td, st)
        return (2 if self.tensor_cores else 1) + self._layer_head(rt, 0, T)

    def _layer_head(self, rt, li, T) -> int:
        """QKV GEMM on the raw residual + fused RMSNorm-scale/RoPE/page store."""
        cfg, st, td = self.config, stream_handle(), self.config.tim_dtype
        dm, D = cfg.model_dim, cfg.head_dim
        n = self._gemm(rt, li, 0, rt.h, rt.qkv, None, T)
        if "rope" in self._DIAG_SKIP:
            return n
        L.call("tim_rope_kv_store", rt.qkv.data_ptr(), rt.h.data_ptr(), dm, 1e-6, T,
               rt.row_pos.data_ptr(), rt.row_pages.data_ptr(), self.cos.data_ptr(),
               self.sin.data_ptr(), cfg.heads, cfg.n_kv, D, rt.q.data_ptr(),
               self.pool_layer(rt.pool.K_layers, li), self.pool_layer(rt.pool.V_layers, li), td, st)
        return 1 + n

    def _attn(self, rt, sp: int, li: int, T: int, has_ext: bool, timed=None) -> int:
        """Attention of one layer: the split-K tile kernel over the decode tiles
        (mode 0) and, when the step has multi-token rows, over its multi-token
        tiles (mode 1) on the tensor-core path; else the fp32 kernel."""
        cfg, st, td = self.config, stream_handle(), self.config.tim_dtype
        D, hq, hkv = cfg.head_dim, cfg.heads, cfg.n_kv
        kl = self.pool_layer(rt.pool.K_layers, li)
        vl = self.pool_layer(rt.pool.V_layers, li)
        tstride = rt.tables.shape[1]
        if not self.tensor_cores:
            L.call("tim_attn_extend", sp, T, rt.q.data_ptr(), rt.ctx.data_ptr(), kl, vl,
                   rt.tables.data_ptr(), tstride, hq, hkv, D, self.scale, td, st)
            return 1
        if timed is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        # mode 2: decode tiles and multi-token items in one launch, CTAs split
        # per the descriptor's cost model (falls back to two launches when the
        # shape has no tcgen05 multi-token kernel)
        if "attn" in self._DIAG_SKIP:
            return 0
        L.call("tim_attn_decode", sp, 2 if has_ext else 0, rt.q.data_ptr(), rt.ctx.data_ptr(), kl, vl,
               rt.tables.data_ptr(), tstride, hq, hkv, D, self.scale, rt.ws.data_ptr(),
               rt.counters.data_ptr(), rt.n_ctas, rt.max_dec, td, st)
        n = 1 if has_ext and self.ext_q else (2 if has_ext else 1)
        if timed is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            timed.append((e0, e1))
        return n

    def _layer_tail(self, rt, li, T) -> int:
        """h += ctx @ wo; u = silu(rms(h) @ w1) (scale fused); h += u @ w2."""
        cfg, st, td = self.config, stream_handle(), self.config.tim_dtype
        dm = cfg.model_dim
        n = self._gemm(rt, li, 1, rt.ctx, rt.h, rt.h, T)
        n += self._gemm(rt, li, 2, rt.h, rt.u, None, T)
        if "silu" not in self._DIAG_SKIP:
            L.call("tim_silu_rms", rt.u.data_ptr(), T, cfg.n_mlp, rt.h.data_ptr(), dm, 1e-6, td, st)
        n += self._gemm(rt, li, 3, rt.u, rt.h, rt.h, T)
        return 1 + n

    def _post(self, rt, sp: int, step: torch.Tensor, T: int, n_last: int, has_ext: bool,
              mask_off: int | None = None):
        cfg, st, td = self.config, stream_handle(), self.config.tim_dtype
        dm = cfg.model_dim
        n = self._layer_tail(rt, 0, T)
        for li in range(1, cfg.layers):
            n += self._layer_head(rt, li, T)
            n += self._attn(rt, sp, li, T, has_ext)
            n += self._layer_tail(rt, li, T)
        off = L.HEADER_INTS                     # `last` is packed first (stepdesc.pack)
        idx = step[off: off + n_last].long()
        hl = rt.h.index_select(0, idx)
        xl = torch.empty_like(hl)
        L.call("tim_rmsnorm", hl.data_ptr(), dm, xl.data_ptr(), dm, n_last, dm, 1e-6, td, st)
        logits = torch.matmul(xl, self.emb_t).float()
        toks = torch.empty(n_last, dtype=torch.int32, device=self.dev)
        # masked greedy pick (model.py:186-192): mask ids follow `last` in the descriptor
        mask_ids = step.data_ptr() + (off + n_last if mask_off is None else mask_off) * 4
        L.call("tim_masked_argmax", logits.data_ptr(), n_last, cfg.vocab, mask_ids, rt.masks.data_ptr(),
               rt.mask_words, toks.data_ptr(), L.DTYPE_F32, st)
        return n + 2, logits, toks

    def forward_rows(self, rt: StepRuntime, step: torch.Tensor, sd: StepDesc):
        """The batched forward over staged rows (model.py:137-164 for every segment).
        Graph mode replays the captured graphs of (row bucket, has multi-token rows)."""
        timed = rt.attn_events
        ev = [] if timed is not None else None
        has_ext = bool(sd.ext)
        if rt.graph_bucket(sd.n_rows) is not None and sd.rows_pad:
            Tb = sd.rows_pad
            if step.data_ptr() != rt.gstep.data_ptr():
                rt.gstep[: step.numel()].copy_(step)
            key = (Tb, has_ext)
            g = rt.graphs.get(key)
            if g is None:
                g = self._capture(rt, Tb, sd.last_pad, has_ext)
                rt.graphs[key] = g
            pe = rt.phase_events
            if pe is not None:
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                evs[0].record()
            g["pre"].replay()
            if pe is not None:
                evs[1].record()
            n_att = self._attn(rt, rt.gstep.data_ptr(), 0, Tb, has_ext, ev)
            if pe is not None:
                evs[2].record()
            g["post"].replay()
            if pe is not None:
                evs[3].record()
                pe.append((key, len(sd.dec), sum(sg[1] + sg[2] for sg in sd.segs), evs))
            rt.launches += g["launches"] + n_att
            logits, toks = g["logits"][: len(sd.last)].clone(), g["toks"]
        else:
            T = sd.n_rows
            sp = step.data_ptr()
            n = self._pre(rt, sp, T)
            n += self._attn(rt, sp, 0, T, has_ext, ev)
            m, logits, toks = self._post(rt, sp, step, T, len(sd.last), has_ext,
                                         sd.offsets["off_last_mask"])
            rt.launches += n + m
        if ev:
            timed.append((ev[0][0], ev[0][1], sd))
        rt.last_logits = logits
        rt.last_tokens = toks
        return toks

    def _capture(self, rt: StepRuntime, Tb: int, n_last: int, has_ext: bool) -> dict:
        """Capture the pre (embed + layer-0 head) and post (rest) phases for a row
        bucket; the descriptor is read from the fixed rt.gstep buffer."""
        sp = rt.gstep.data_ptr()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):          # warm-up (cuBLAS handles, heuristics)
            self._pre(rt, sp, Tb)
            self._attn(rt, sp, 0, Tb, has_ext)
            self._post(rt, sp, rt.gstep, Tb, n_last, has_ext)
        torch.cuda.current_stream().wait_stream(side)
        pre, post = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(pre):
            n_pre = self._pre(rt, sp, Tb)
        with torch.cuda.graph(post):
            n_post, logits, toks = self._post(rt, sp, rt.gstep, Tb, n_last, has_ext)
        return {"pre": pre, "post": post, "logits": logits, "toks": toks,
                "launches": n_pre + n_post}

    @staticmethod
    def pool_layer(t: torch.Tensor, li: int) -> int:
        return t.data_ptr() + li * t.stride(0) * t.element_size()


# Reference-compatible name for the numeric backend.
TinyTransformer = B200Transformer


class ScriptedModel:
    """Replay backend: device page accounting (K4/K5) without arithmetic
    (model.py:195-233).  Logits are None; the engine pops the script."""

    has_weights = False

    def __init__(self, vocab: int = 512, position_limit: int = 256):
        self.vocab = vocab
        self.position_limit = position_limit
        self.config = None

    @property
    def vocab_size(self) -> int:
        return self.vocab

    def make_pool(self, capacity: int) -> DevicePagePool:
        return DevicePagePool(capacity)

    def runtime(self, pool, max_slots: int, logical_cap: int) -> StepRuntime:
        return StepRuntime(self, pool, max_slots, logical_cap)

    def plan_attention(self, sd, slot, m, n, row_off) -> None:
        sd.segs.append((slot, m, n, row_off))

    def _forward(self, n, positions, table, pool):
        for p in positions:
            if p >= self.position_limit:
                raise PositionOverflow(int(p), self.position_limit)
        table.append(pool.alloc(table.request_id, n))
        return None

    def prefill(self, tokens, positions, table, pool):
        if not tokens:
            raise EmptyExtend("nothing to prefill")
        return self._forward(len(tokens), positions, table, pool)

    def extend(self, tokens, start_position, table, pool):
        if not tokens:
            raise EmptyExtend("nothing to extend")
        return self._forward(len(tokens), range(start_position, start_position + len(tokens)),
                             table, pool)

    def decode_step(self, last_token, position, table, pool):
        return self._forward(1, [position], table, pool)


def sample(logits, mask) -> int:
    """Greedy pick among admitted ids, lowest id on ties (model.py:186-192)."""
    logits = np.asarray(logits)
    if hasattr(mask, "as_array"):
        allowed = mask.as_array(len(logits))
    else:
        allowed = np.zeros(len(logits), dtype=bool)
        allowed[list(mask)] = True
    if not allowed.any():
        raise EmptyMask("no admissible token")
    return int(np.argmax(np.where(allowed, logits, -np.inf)))
