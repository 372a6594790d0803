"""ctypes binding of libtimrun.so (include/timrun.h).

There is no fallback: if the library is missing or a call fails, an exception
is raised.  Error codes map onto the reference exception types.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libtimrun.so"

TIM_OK = 0
TIM_OUT_OF_PAGES = 1
TIM_DOUBLE_FREE = 2
TIM_POSITION_OVERFLOW = 3
TIM_SPAN_OUT_OF_RANGE = 4
TIM_BAD_ARGUMENT = 5
TIM_CUDA_ERROR = 6
TIM_UNSUPPORTED = 7
TIM_REJECTED = 8

DTYPE_F32 = 0
DTYPE_BF16 = 1

OP_ALLOC = 0
OP_FREE = 1

HEADER_INTS = 32
NEW_FIELDS, SEG_FIELDS, DEC_FIELDS, EXT_FIELDS, JOB_FIELDS, OP_FIELDS = 5, 4, 6, 6, 8, 6

# Every exported symbol with its ctypes signature (checked by tests/test_abi.py).
_i32, _i64, _f32, _p, _cp = C.c_int32, C.c_int64, C.c_float, C.c_void_p, C.c_char_p
SIGNATURES = {
    "tim_abi_version": (_i32, []),
    "tim_last_error": (_cp, []),
    "tim_sm_count": (_i32, []),
    "tim_read_error": (_i32, [_p, _p, _p, _p]),
    "tim_pool_init": (_i32, [_p, _p, _i32, _p]),
    "tim_page_ops": (_i32, [_p, _p, _p, _i32, _p, _i64, _p, _p]),
    "tim_prune_compact": (_i32, [_p, _i32, _p, _i64, _p, _i64, _p, _p, _p]),
    "tim_stage_rows": (_i32, [_p, _p, _i64, _p, _i64, _p, _i64, _p, _p, _p, _p]),
    "tim_embed": (_i32, [_p, _i32, _p, _i32, _p, _i32, _p]),
    "tim_rmsnorm": (_i32, [_p, _i64, _p, _i64, _i32, _i32, _f32, _i32, _p]),
    "tim_silu": (_i32, [_p, _i64, _i32, _p]),
    "tim_rope_kv_store": (_i32, [_p, _p, _i32, _f32, _i32, _p, _p, _p, _p, _i32, _i32, _i32, _p, _p,
                                 _p, _i32, _p]),
    "tim_silu_rms": (_i32, [_p, _i32, _i32, _p, _i32, _f32, _i32, _p]),
    "tim_decode_ws_floats": (_i64, [_i32, _i32, _i32, _i32]),
    "tim_attn_decode": (_i32, [_p, _i32, _p, _p, _p, _p, _p, _i64, _i32, _i32, _i32, _f32, _p, _p,
                               _i32, _i32, _i32, _p]),
    "tim_attn_extend": (_i32, [_p, _i32, _p, _p, _p, _p, _p, _i64, _i32, _i32, _i32, _f32, _i32, _p]),
    "tim_extend_queries_per_item": (_i32, [_i32, _i32, _i32, _i32]),
    "tim_extend_head_groups": (_i32, [_i32, _i32, _i32]),
    "tim_argmax": (_i32, [_p, _i32, _i32, _p, _i32, _p]),
    "tim_set_trace": (_i32, [_p]),
    "tim_tc_trace": (_i32, [_p]),
    "tim_noop": (_i32, [_i32, _i32, _i32, _p]),
    "tim_attn_plan": (_i32, [_p, _p, _i64, _i32, _i32, _i32, _p, _p]),
    "tim_step_account": (_i32, [_p, _p, _p, _i32, _p, _i32, _p, _p]),
    "tim_masked_argmax": (_i32, [_p, _i32, _i32, _p, _p, _i32, _p, _i32, _p]),
    # grammar tracker (host)
    "tim_grammar_create": (_p, [_p, _p, _i32, _p, _p, _i32, _i32]),
    "tim_grammar_destroy": (None, [_p]),
    "tim_grammar_mask_count": (_i32, [_p]),
    "tim_grammar_mask_words": (_i32, [_p]),
    "tim_grammar_mask": (_i32, [_p, _i32, _p, _p, _p]),
    "tim_tracker_create": (_p, [_p]),
    "tim_tracker_clone": (_p, [_p]),
    "tim_tracker_destroy": (None, [_p]),
    "tim_tracker_feed": (_i32, [_p, _i32, _p]),
    "tim_tracker_feed_many": (_i32, [_p, _p, _i32, _p]),
    "tim_tracker_event": (_i32, [_p, _i32, _p, _p, _p, _p, _p]),
    "tim_tracker_mask": (_i32, [_p, _p, _p, _p]),
    "tim_tracker_state": (_i32, [_p, _p, _p, _p, _p]),
    "tim_tracker_context": (_cp, [_p]),
}


class TimrunError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"libtimrun {what} failed with code {code}")


_lib = None


def load(path: Path | None = None):
    """Load the shared library (once).  Raises if it is absent: no CPU fallback."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("TIMRUN_LIB") or LIB_PATH)   # TIMRUN_LIB: diagnostics builds
    if not p.exists():
        raise RuntimeError(
            f"libtimrun.so not found at {p}; build it with `python -m paper_2507_16784_b200.build` "
            "(the CUDA path has no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().tim_last_error().decode(errors="replace")


def call(name: str, *args) -> int:
    """Invoke an ABI entry point, raising TimrunError on a non-zero return code."""
    fn = getattr(load(), name)
    rc = fn(*args)
    if SIGNATURES[name][0] is _i32 and name not in ("tim_abi_version", "tim_sm_count",
                                                    "tim_extend_queries_per_item",
                                                    "tim_extend_head_groups") and rc != TIM_OK:
        raise TimrunError(rc, f"{name}: {last_error()}")
    return rc
