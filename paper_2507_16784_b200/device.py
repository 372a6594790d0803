"""Single-call device helpers for the per-call (reference-shaped) APIs."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .stepdesc import StepDesc


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def prune_compact_one(live, tokens, s0: int, reencode_from: int, spans):
    """Run K4 for one request held in host lists; returns (new suffix, suffix tokens)."""
    L.load()
    n = len(live)
    live_d = torch.tensor(np.asarray(live, dtype=np.int32).reshape(1, -1) if n else
                          np.zeros((1, 1), np.int32), device="cuda")
    tok_d = torch.tensor(np.asarray(tokens, dtype=np.int32).reshape(1, -1) if tokens else
                         np.zeros((1, 1), np.int32), device="cuda")
    keep = sum(1 for i in live[s0:] if not any(a <= i < b for a, b in spans))
    sd = StepDesc()
    sd.job(0, n, s0, reencode_from, spans, 0, keep)
    step = torch.from_numpy(sd.pack()).cuda()
    rows = torch.zeros(max(keep, 1), dtype=torch.int32, device="cuda")
    err = torch.zeros(2, dtype=torch.int32, device="cuda")
    L.call("tim_prune_compact", step.data_ptr(), 1, live_d.data_ptr(), live_d.shape[1],
           tok_d.data_ptr(), tok_d.shape[1], rows.data_ptr(), err.data_ptr(), _stream())
    code = int(err[0].item())
    if code:
        from .paging import raise_device_error
        raise_device_error(code, int(err[1].item()))
    suffix = live_d[0, s0:s0 + keep].cpu().tolist()
    return suffix, rows[:keep].cpu().tolist()
