"""Oracle restatement of the reference rotary transformer (threadrun/model.py).  Test-only.

Follows model.py:39-192 line for line.  The only additions are two config
fields the reference lacks, `kv_heads` (GQA, q head h reads kv head
h // (heads // kv_heads), the HF repeat_kv convention) and `mlp_dim`; with
kv_heads == heads and mlp_dim == 4*model_dim the weights and arithmetic are
exactly the reference's (same RNG stream: emb, then per layer wq, wk, wv, wo,
w1, w2 — model.py:91-103).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .paging import PagePool


class PositionOverflow(RuntimeError):
    """model.py:24-28"""

    def __init__(self, position: int, limit: int):
        super().__init__(f"position {position} >= limit {limit}")
        self.position, self.limit = position, limit


@dataclass
class Config:
    """model.py:39-66 (+ kv_heads, mlp_dim)."""
    layers: int = 2
    heads: int = 4
    head_dim: int = 16
    vocab: int = 512
    position_limit: int = 256
    rope_base: float = 10000.0
    seed: int = 0
    precision: str = "float32"
    kv_heads: int = 0
    mlp_dim: int = 0

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


def rmsnorm(x):
    """model.py:69-70"""
    return x / np.sqrt(np.mean(np.square(x), axis=-1, keepdims=True) + 1e-6)


def silu(x):
    """model.py:73-74"""
    return x / (1.0 + np.exp(-x))


def init_weights(cfg: Config) -> dict:
    """model.py:87-105: seeded N(0, 1/dm) weights in the reference draw order."""
    dt, dm = cfg.dtype, cfg.model_dim
    rng = np.random.default_rng(cfg.seed)
    scale = 1.0 / np.sqrt(dm)

    def mat(*shape):
        return (rng.standard_normal(shape) * scale).astype(dt)

    w = {"emb": mat(cfg.vocab, dm), "layers": []}
    kvd = cfg.n_kv * cfg.head_dim
    for _ in range(cfg.layers):
        w["layers"].append({
            "wq": mat(dm, dm), "wk": mat(dm, kvd), "wv": mat(dm, kvd), "wo": mat(dm, dm),
            "w1": mat(dm, cfg.n_mlp), "w2": mat(cfg.n_mlp, dm),
        })
    half = cfg.head_dim // 2
    w["inv_freq"] = (cfg.rope_base ** (-np.arange(half) / half)).astype(dt)
    return w


def rope(x, positions, inv_freq):
    """model.py:118-125, rotate-half; x: (n, heads, D)."""
    half = x.shape[-1] // 2
    ang = positions[:, None] * inv_freq[None, :]
    cos = np.cos(ang)[:, None, :]
    sin = np.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * cos - x2 * sin, x1 * sin + x2 * cos], axis=-1)


def attend(q, k_all, v_all, m: int):
    """model.py:149-159 for one layer: q (n, Hq, D) over k/v (m+n, Hkv, D), prefix
    fully visible, causal inside the new block.  Returns ctx (n, Hq, D)."""
    n, hq, d = q.shape
    hkv = k_all.shape[1]
    if hkv != hq:
        k_all = np.repeat(k_all, hq // hkv, axis=1)
        v_all = np.repeat(v_all, hq // hkv, axis=1)
    col = np.arange(m + n)
    causal = col[None, :] > (m + np.arange(n))[:, None]
    scores = np.einsum("qhd,khd->hqk", q, k_all) / np.sqrt(d)
    scores = np.where(causal[None, :, :], -np.inf, scores)
    scores = scores - scores.max(axis=-1, keepdims=True)
    w = np.exp(scores)
    w = w / w.sum(axis=-1, keepdims=True)
    return np.einsum("hqk,khd->qhd", w, v_all)


class Model:
    """model.py:78-183: one forward path writing one page per token."""

    def __init__(self, cfg: Config, weights: dict | None = None):
        self.config = cfg
        self.w = weights if weights is not None else init_weights(cfg)

    @property
    def position_limit(self) -> int:
        return self.config.position_limit

    def make_pool(self, capacity: int) -> PagePool:
        c = self.config
        return PagePool(capacity, (c.layers, c.n_kv, c.head_dim), c.dtype)

    def forward(self, tokens, positions, table, pool, return_ctx: bool = False):
        """model.py:127-164"""
        cfg = self.config
        n = len(tokens)
        for p in positions:
            if p >= cfg.position_limit:
                raise PositionOverflow(int(p), cfg.position_limit)
        new_pages = pool.alloc(table.request_id, n)
        pos = np.asarray(positions, dtype=cfg.dtype)
        prefix = table.pages
        m = len(prefix)
        h = self.w["emb"][np.asarray(tokens, dtype=np.int64)]
        ctxs = []
        for li, layer in enumerate(self.w["layers"]):
            x = rmsnorm(h)
            q = rope((x @ layer["wq"]).reshape(n, cfg.heads, cfg.head_dim), pos, self.w["inv_freq"])
            k = rope((x @ layer["wk"]).reshape(n, cfg.n_kv, cfg.head_dim), pos, self.w["inv_freq"])
            v = (x @ layer["wv"]).reshape(n, cfg.n_kv, cfg.head_dim)
            pool.K[new_pages, li] = k
            pool.V[new_pages, li] = v
            if m:
                k_all = np.concatenate([pool.K[prefix, li], k], axis=0)
                v_all = np.concatenate([pool.V[prefix, li], v], axis=0)
            else:
                k_all, v_all = k, v
            ctx = attend(q, k_all, v_all, m).reshape(n, cfg.model_dim)
            ctxs.append(ctx)
            h = h + ctx.astype(cfg.dtype) @ layer["wo"]
            h = h + silu(rmsnorm(h) @ layer["w1"]) @ layer["w2"]
        table.append(new_pages)
        logits = rmsnorm(h[-1]) @ self.w["emb"].T
        return (logits, ctxs) if return_ctx else logits

    def prefill(self, tokens, positions, table, pool):
        if len(tokens) != len(positions):
            raise ValueError("tokens and positions must align")
        if not tokens:
            raise ValueError("nothing to prefill")
        return self.forward(tokens, positions, table, pool)

    def extend(self, tokens, start, table, pool):
        if not tokens:
            raise ValueError("nothing to extend")
        return self.forward(tokens, list(range(start, start + len(tokens))), table, pool)

    def decode_step(self, token, position, table, pool):
        return self.forward([token], [position], table, pool)


def masked_argmax(logits, allowed) -> int:
    """oracles.py:105-115"""
    best, best_v = None, None
    for tid in sorted(allowed):
        v = float(logits[tid])
        if best_v is None or v > best_v:
            best, best_v = tid, v
    if best is None:
        raise ValueError("empty mask")
    return best
