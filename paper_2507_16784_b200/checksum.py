"""Order-sensitive checksums of the engine's paging state (block tables, live
lists, free stack), computed on the device without copying the state back.

The same definition, restated in numpy, is what oracle/gen_golden.py records
per step from the REFERENCE Engine (scheduler.py:274-335 with ScriptedModel),
so a long device run can be compared with the reference bit-exactly at every
step for a few microseconds of GPU work instead of a full readback:

    w(i)            = ((i * 2654435761) mod 2**32 >> 16) + 1          (1..65536)
    table_hash      = sum_k sum_{i < len_k} (table_k[i] + 1) * w(i + 7919 k)
    live_hash       = sum_k sum_{i < len_k} (live_k[i]  + 1) * w(i + 7919 k)
    free_hash       = sum_{i < free_count} (free_list[i] + 1) * w(i)

k is the request's submission index (rid "r<k>"), table_k its block table
(paging.py:86-107), live_k its retained logical indices (scheduler.py:136),
free_list the LIFO free list bottom-to-top (paging.py:40,57,62-67).  Every
term is < 2**37, so the int64 sums cannot overflow below 2**26 entries.
"""

from __future__ import annotations

import numpy as np
import torch

MUL = 2654435761
STRIDE = 7919


def weights_np(idx: np.ndarray) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.int64)
    return (((idx * MUL) & 0xFFFFFFFF) >> 16) + 1


def weights_torch(idx: torch.Tensor) -> torch.Tensor:
    return (((idx * MUL) & 0xFFFFFFFF) >> 16) + 1


def seq_hash_np(values, k: int = 0) -> int:
    v = np.asarray(values, dtype=np.int64)
    if v.size == 0:
        return 0
    w = weights_np(np.arange(v.size, dtype=np.int64) + STRIDE * k)
    return int(((v + 1) * w).sum())


def host_hash(live_lens: dict, pending_lens: dict, decoded: dict) -> int:
    """Hash of the per-request host counters (rid -> int), order-independent
    over the dicts, sensitive to which request holds which value."""
    h = 0
    for rid, n in live_lens.items():
        k = int(rid[1:])
        h += (n + 1) * int(weights_np(3 * k)) + (pending_lens.get(rid, 0) + 1) * int(weights_np(3 * k + 1))
    for rid, n in decoded.items():
        k = int(rid[1:])
        h += (n + 1) * int(weights_np(3 * k + 2))
    return h & 0x7FFFFFFFFFFFFFFF


def device_hashes(engine) -> tuple[int, int, int]:
    """(table_hash, live_hash, free_hash) of a B200 Engine's device state.
    One small reduction per array; a single device->host read of 3 int64."""
    rt, pool = engine.runtime, engine.pool
    dev = rt.tables.device
    reqs = [r for r in engine.requests.values() if r.slot is not None and r.table_len > 0]
    out = torch.zeros(3, dtype=torch.int64, device=dev)
    if reqs:
        n = max(r.table_len for r in reqs)
        slots = torch.tensor([r.slot for r in reqs], dtype=torch.long, device=dev)
        ks = torch.tensor([int(r.rid[1:]) for r in reqs], dtype=torch.int64, device=dev)
        lens = torch.tensor([r.table_len for r in reqs], dtype=torch.int64, device=dev)
        idx = torch.arange(n, dtype=torch.int64, device=dev)
        mask = idx[None, :] < lens[:, None]
        w = weights_torch(idx[None, :] + STRIDE * ks[:, None]) * mask
        out[0] = ((rt.tables[slots, :n].long() + 1) * w).sum()
        out[1] = ((rt.live[slots, :n].long() + 1) * w).sum()
    sp = pool.free_count
    if sp:
        i = torch.arange(sp, dtype=torch.int64, device=dev)
        out[2] = ((pool.free_stack[:sp].long() + 1) * weights_torch(i)).sum()
    a, b, c = out.cpu().tolist()
    return int(a), int(b), int(c)
