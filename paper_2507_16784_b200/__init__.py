"""B200-native TIMRUN working-memory decode path (arXiv 2507.16784).

Drop-in for the hot-path subset of the reference package `threadrun`
(/root/reference/pkg/src/threadrun/__init__.py:35-81): the engine/step API,
the page pool, the prune entry points and the model-backend protocol keep
their names, arguments and exceptions.  Compute runs in libtimrun.so
(hand-written sm_100a kernels, include/timrun.h) plus cuBLAS GEMMs; there is
no CPU fallback.
"""

__version__ = "0.1.0"

from .tokenizer import ByteTokenizer, build_tokenizer
from .spans import TokenSpan
from .grammar import Grammar, TokenMask, Tracker
from .structure import Rejected, StructureEvent
from .paging import DevicePagePool, DoubleFree, KvPage, OutOfPages, PagePool, PageTable, gather
from .pruning import (PruneBuffer, PrunePlan, RequestMetrics, SpanOutOfRange, ZeroLength, apply,
                      coalesce, kv_pruned_pct, oracle_evictions)
from .model import (B200Transformer, EmptyExtend, EmptyMask, ModelConfig, PositionOverflow,
                    ScriptedModel, TinyTransformer, qwen3_8b_shape, sample)
from .tools import ToolCall, ToolHub, ToolResponse, ToolSpec
from .scheduler import (BatchConfig, Deadline, Engine, PromptTooLong, QueueFull, ScriptError,
                        Status, StepReport, TokenLimit, attention_flops_estimate)
from .traces import Trace, make_trace_from_text

__all__ = [
    "ByteTokenizer", "build_tokenizer", "TokenSpan", "Rejected", "StructureEvent",
    "Grammar", "TokenMask", "Tracker", "DevicePagePool", "DoubleFree", "KvPage", "OutOfPages", "PagePool",
    "PageTable", "gather", "PruneBuffer", "PrunePlan", "RequestMetrics", "SpanOutOfRange",
    "ZeroLength", "apply", "coalesce", "kv_pruned_pct", "oracle_evictions", "B200Transformer",
    "EmptyExtend", "EmptyMask", "ModelConfig", "PositionOverflow", "ScriptedModel",
    "TinyTransformer", "qwen3_8b_shape", "sample", "ToolCall", "ToolHub", "ToolResponse",
    "ToolSpec", "BatchConfig", "Deadline", "Engine", "PromptTooLong", "QueueFull", "ScriptError",
    "Status", "StepReport", "TokenLimit", "attention_flops_estimate", "Trace",
    "make_trace_from_text",
]
