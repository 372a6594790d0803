"""Kernel-level parity of libtimrun against the CPU oracle (GPU only).

Tolerances (BASELINE.json north_star): fp32 runs <= 1e-5 relative
(max|d| / max|ref|, verify.py:116-117); bf16 KV <= 2e-2 max-abs against the
fp32 oracle evaluated on the same (bf16-rounded) inputs.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import model as om
from oracle import paging as op
from oracle import pruning as opr
from paper_2507_16784_b200 import _lib as L
from paper_2507_16784_b200.stepdesc import StepDesc

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
F32_REL = 1e-5


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _dev(arr):
    return torch.from_numpy(np.ascontiguousarray(arr)).cuda()


def _ptr(t):
    return t.data_ptr()


def _pool(cap, hkv, d, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    k = torch.randn(cap, hkv, d, device="cuda", generator=g).to(dtype)
    v = torch.randn(cap, hkv, d, device="cuda", generator=g).to(dtype)
    return k, v


def _tables(lengths, cap, stride, seed):
    rng = np.random.default_rng(seed)
    perm = rng.permutation(cap)
    tab = np.full((len(lengths), stride), -1, dtype=np.int32)
    off = 0
    for i, n in enumerate(lengths):
        tab[i, :n] = perm[off:off + n]
        off += n
    return tab


@pytest.mark.parametrize("planned", [False, True])
@pytest.mark.parametrize("n_ctas", [None, 3, 1])
@pytest.mark.parametrize("hq,hkv", [(32, 8), (16, 4), (8, 8), (32, 2)])
def test_decode_bf16_matches_oracle(n_ctas, hq, hkv, planned):
    """Decode tiles (K1), with and without the per-step plan (tim_attn_plan)."""
    _decode_case([1, 2, 15, 16, 17, 100, 777, 1500, 33, 4096], n_ctas, hq, hkv, planned)


@pytest.mark.parametrize("planned", [False, True])
@pytest.mark.parametrize("n_ctas", [None, 7])
def test_decode_bf16_long_horizon_lengths(n_ctas, planned):
    """C4 retained lengths (12K-token prompt + working memory, up to the 16,384
    position limit) on the C2 head shape."""
    _decode_case([13378, 16384, 12001, 3, 16383, 9000, 12500, 64], n_ctas, 32, 8, planned)


def _decode_case(lengths, n_ctas, hq, hkv, planned):
    d = 128
    cap = sum(lengths) + 7
    stride = max(lengths)
    kp, vp = _pool(cap, hkv, d, torch.bfloat16, 1)
    tab = _tables(lengths, cap, stride, 2)
    g = torch.Generator(device="cuda").manual_seed(3)
    q = torch.randn(len(lengths), hq, d, device="cuda", generator=g).to(torch.bfloat16)
    sd = StepDesc()
    for i, n in enumerate(lengths):
        sd.dec.append((i, i, n, 1, n - 1, 0))
    sd.serial = 7 if planned else 0
    step = _dev(sd.pack())
    out = torch.zeros(len(lengths), hq, d, device="cuda", dtype=torch.bfloat16)
    sms = L.load().tim_sm_count()
    ctas = sms if n_ctas is None else n_ctas
    ws = torch.zeros(L.load().tim_decode_ws_floats(ctas, len(lengths), hkv, d), device="cuda")
    if planned:
        L.call("tim_attn_plan", _ptr(step), _ptr(_dev(tab)), stride, ctas, len(lengths), d, _ptr(ws), _stream())
    cnt = torch.zeros(len(lengths) * 8, device="cuda", dtype=torch.int32)
    tab_d = _dev(tab)
    for _ in range(2):  # twice: counters must self-reset
        L.call("tim_attn_decode", _ptr(step), 0, _ptr(q), _ptr(out), _ptr(kp), _ptr(vp), _ptr(tab_d),
               stride, hq, hkv, d, 1.0 / np.sqrt(d), _ptr(ws), _ptr(cnt), ctas, len(lengths),
               L.DTYPE_BF16, _stream())
        torch.cuda.synchronize()
        assert int(cnt.abs().sum()) == 0
        kf, vf, qf = kp.float().cpu().numpy(), vp.float().cpu().numpy(), q.float().cpu().numpy()
        got = out.float().cpu().numpy()
        for i, n in enumerate(lengths):
            pages = tab[i, :n]
            ref = om.attend(qf[i:i + 1], kf[pages], vf[pages], n - 1)[0]
            err = np.abs(got[i] - ref).max()
            assert err <= BF16_TOL, (i, n, err)


def _extend_case(hq, hkv, d, dtype, segs_mn, seed):
    """segs_mn: list of (m, n).  Returns tensors + oracle outputs."""
    lengths = [m + n for m, n in segs_mn]
    cap = sum(lengths) + 5
    stride = max(lengths)
    kp, vp = _pool(cap, hkv, d, dtype, seed)
    tab = _tables(lengths, cap, stride, seed + 1)
    rows = sum(n for _, n in segs_mn)
    g = torch.Generator(device="cuda").manual_seed(seed + 2)
    q = torch.randn(rows, hq, d, device="cuda", generator=g).to(dtype)
    sd = StepDesc()
    row = 0
    for i, (m, n) in enumerate(segs_mn):
        sd.segs.append((i, m, n, row))
        row += n
    sd.n_rows = rows
    return kp, vp, tab, stride, q, sd, rows


SEGSETS = {
    "mixed": [(0, 1), (0, 7), (5, 33), (100, 64), (700, 150), (0, 200), (1200, 3), (40, 1)],
    # C4: re-encodes / decode rows behind a 12K-16K retained prefix
    "long": [(13000, 150), (12000, 1), (16000, 64), (9000, 33), (14000, 1), (5, 1)],
}


@pytest.mark.parametrize("segset", ["mixed", "long"])
@pytest.mark.parametrize("one_launch", [False, True])
@pytest.mark.parametrize("n_ctas", [None, 5])
@pytest.mark.parametrize("hq,hkv", [(32, 8), (16, 4), (4, 4), (32, 2)])
def test_extend_tiles_bf16_matches_oracle(hq, hkv, n_ctas, one_launch, segset):
    """Multi-query tiles (re-encode / prefill / tool rows) through the unified
    split-K kernel: paged prefix fully visible + causal new block."""
    if segset == "long" and (hq, hkv) != (32, 8):
        pytest.skip("long prefixes only at the C2/C4 head shape")
    d = 128
    segs = SEGSETS[segset]
    kp, vp, tab, stride, q, sd, rows = _extend_case(hq, hkv, d, torch.bfloat16, segs, 11)
    qpi = L.load().tim_extend_queries_per_item(hq, hkv, d, L.DTYPE_BF16)
    ngr = L.load().tim_extend_head_groups(hq, hkv, d)
    assert qpi >= 1 and 1 <= ngr <= hkv
    row = 0
    for i, (m, n) in enumerate(segs):
        if n == 1:
            sd.dec.append((row, i, m + 1, 1, m, 0))
        for q0 in range(0, n if n > 1 else 0, qpi):
            nq = min(qpi, n - q0)
            for gi in range(ngr):
                sd.ext.append((row + q0, i, m + q0 + nq, nq, m, gi))
        row += n
    ctas = n_ctas or L.load().tim_sm_count()
    sd.ctas = ctas
    step = _dev(sd.pack())
    out = torch.zeros(rows, hq, d, device="cuda", dtype=torch.bfloat16)
    ntiles = len(sd.dec) + len(sd.ext)
    ws = torch.zeros(L.load().tim_decode_ws_floats(ctas, ntiles, hkv, d), device="cuda")
    cnt = torch.zeros(ntiles * 8, device="cuda", dtype=torch.int32)
    tab_d = _dev(tab)
    for mode in ((2,) if one_launch else (0, 1)):
        L.call("tim_attn_decode", _ptr(step), mode, _ptr(q), _ptr(out), _ptr(kp), _ptr(vp),
               _ptr(tab_d), stride, hq, hkv, d, 1.0 / np.sqrt(d), _ptr(ws), _ptr(cnt), ctas,
               ntiles, L.DTYPE_BF16, _stream())
    torch.cuda.synchronize()
    assert int(cnt.abs().sum()) == 0
    kf, vf, qf = kp.float().cpu().numpy(), vp.float().cpu().numpy(), q.float().cpu().numpy()
    got = out.float().cpu().numpy()
    row = 0
    for i, (m, n) in enumerate(segs):
        pages = tab[i, :m + n]
        ref = om.attend(qf[row:row + n], kf[pages], vf[pages], m)
        err = np.abs(got[row:row + n] - ref).max()
        assert err <= BF16_TOL, (i, m, n, err)
        row += n


@pytest.mark.parametrize("hq,hkv,d", [(4, 4, 32), (4, 4, 16), (8, 2, 64)])
def test_generic_fp32_matches_oracle(hq, hkv, d):
    segs = [(0, 1), (0, 9), (13, 1), (40, 20), (3, 70)]
    kp, vp, tab, stride, q, sd, rows = _extend_case(hq, hkv, d, torch.float32, segs, 21)
    step = _dev(sd.pack())
    out = torch.zeros(rows, hq, d, device="cuda", dtype=torch.float32)
    tab_d = _dev(tab)
    L.call("tim_attn_extend", _ptr(step), rows, _ptr(q), _ptr(out), _ptr(kp), _ptr(vp),
           _ptr(tab_d), stride, hq, hkv, d, 1.0 / np.sqrt(d), L.DTYPE_F32, _stream())
    torch.cuda.synchronize()
    kf, vf, qf = kp.cpu().numpy(), vp.cpu().numpy(), q.cpu().numpy()
    got = out.cpu().numpy()
    row = 0
    for i, (m, n) in enumerate(segs):
        pages = tab[i, :m + n]
        ref = om.attend(qf[row:row + n], kf[pages], vf[pages], m)
        rel = np.abs(got[row:row + n] - ref).max() / np.abs(ref).max()
        assert rel <= F32_REL, (i, m, n, rel)
        row += n


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_rope_kv_store_matches_oracle(dtype):
    hq, hkv, d, P = 8, 2, 64, 512
    n = 37
    cap = 64
    half = d // 2
    inv = (1e4 ** (-np.arange(half) / half)).astype(np.float32)
    ang = np.arange(P, dtype=np.float32)[:, None] * inv[None, :]
    cos_t, sin_t = _dev(np.cos(ang).astype(np.float32)), _dev(np.sin(ang).astype(np.float32))
    g = torch.Generator(device="cuda").manual_seed(5)
    qkv = torch.randn(n, (hq + 2 * hkv) * d, device="cuda", generator=g).to(dtype)
    rng = np.random.default_rng(0)
    pos = rng.integers(0, P, n).astype(np.int32)
    pages = rng.permutation(cap)[:n].astype(np.int32)
    pages[3] = -1  # padding row: no store
    kl = torch.zeros(cap, hkv, d, device="cuda", dtype=dtype)
    vl = torch.zeros_like(kl)
    qo = torch.zeros(n, hq, d, device="cuda", dtype=dtype)
    pos_d, pages_d = _dev(pos), _dev(pages)
    L.call("tim_rope_kv_store", _ptr(qkv), None, 0, 0.0, n, _ptr(pos_d), _ptr(pages_d), _ptr(cos_t),
           _ptr(sin_t), hq, hkv, d, _ptr(qo), _ptr(kl), _ptr(vl),
           L.DTYPE_F32 if dtype == torch.float32 else L.DTYPE_BF16, _stream())
    torch.cuda.synchronize()
    x = qkv.float().cpu().numpy()
    qr = om.rope(x[:, :hq * d].reshape(n, hq, d), pos.astype(np.float32), inv)
    kr = om.rope(x[:, hq * d:(hq + hkv) * d].reshape(n, hkv, d), pos.astype(np.float32), inv)
    vr = x[:, (hq + hkv) * d:].reshape(n, hkv, d)
    tol = 1e-6 if dtype == torch.float32 else 1e-2
    assert np.abs(qo.float().cpu().numpy() - qr).max() <= tol * max(1, np.abs(qr).max())
    kg, vg = kl.float().cpu().numpy(), vl.float().cpu().numpy()
    for i in range(n):
        if pages[i] < 0:
            continue
        assert np.abs(kg[pages[i]] - kr[i]).max() <= tol * max(1, np.abs(kr).max())
        assert np.array_equal(vg[pages[i]], vr[i]) if dtype == torch.float32 else \
            np.abs(vg[pages[i]] - vr[i]).max() <= tol
    untouched = np.setdiff1d(np.arange(cap), pages[pages >= 0])
    assert np.all(kg[untouched] == 0)


def test_page_ops_match_lifo_oracle():
    """Random interleavings of alloc/free in reference order give identical ids."""
    cap, slots, stride = 300, 6, 300
    rng = np.random.default_rng(7)
    pool = op.PagePool(cap)
    tables = [op.PageTable(s) for s in range(slots)]
    stack = torch.empty(cap, dtype=torch.int32, device="cuda")
    owner = torch.empty(cap, dtype=torch.int32, device="cuda")
    tab_d = torch.full((slots, stride), -1, dtype=torch.int32, device="cuda")
    err = torch.zeros(2, dtype=torch.int32, device="cuda")
    L.call("tim_pool_init", _ptr(stack), _ptr(owner), cap, _stream())
    for step_i in range(200):
        sd = StepDesc()
        for _ in range(rng.integers(1, 12)):
            s = int(rng.integers(slots))
            t = tables[s]
            if rng.random() < 0.6:
                nn = int(rng.integers(0, 9))
                if nn > pool.free_count:
                    continue
                sp = pool.free_count
                off = len(t)
                t.append(pool.alloc(s, nn))
                sd.op(L.OP_ALLOC, s, off, nn, sp, s)
            elif len(t):
                cut = int(rng.integers(0, len(t)))
                sp = pool.free_count
                freed = t.truncate_from(cut)
                pool.free(freed)
                sd.op(L.OP_FREE, s, cut, len(freed), sp, s)
        step = _dev(sd.pack())
        L.call("tim_page_ops", _ptr(step), _ptr(stack), _ptr(owner), cap, _ptr(tab_d), stride,
               _ptr(err), _stream())
        torch.cuda.synchronize()
        assert err.cpu().tolist() == [0, 0]
        tg = tab_d.cpu().numpy()
        for s in range(slots):
            assert tg[s, :len(tables[s])].tolist() == tables[s].pages
        sp = pool.free_count
        assert stack[:sp].cpu().tolist() == pool.free_list
        own = owner.cpu().numpy()
        assert {int(p): int(own[p]) for p in np.nonzero(own >= 0)[0]} == pool.allocated


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_rms_folding_matches_rmsnorm_then_gemm(dtype):
    """rope_kv_store/silu_rms with h: rms(h) @ W == (h @ W) * inv_rms (model.py:69-70)."""
    n, dm, hq, hkv, d, P = 9, 256, 4, 2, 32, 64
    half = d // 2
    g = torch.Generator(device="cuda").manual_seed(8)
    h = (torch.randn(n, dm, device="cuda", generator=g) * 3).to(dtype)
    W = (torch.randn(dm, (hq + 2 * hkv) * d, device="cuda", generator=g) / 16).to(dtype)
    inv = (1e4 ** (-np.arange(half) / half)).astype(np.float32)
    ang = np.arange(P, dtype=np.float32)[:, None] * inv[None, :]
    cos_t, sin_t = _dev(np.cos(ang).astype(np.float32)), _dev(np.sin(ang).astype(np.float32))
    pos = _dev(np.arange(n, dtype=np.int32))
    pages = _dev(np.arange(n, dtype=np.int32))
    qkv = h @ W
    kl = torch.zeros(n, hkv, d, device="cuda", dtype=dtype)
    vl = torch.zeros_like(kl)
    qo = torch.zeros(n, hq, d, device="cuda", dtype=dtype)
    td = L.DTYPE_F32 if dtype == torch.float32 else L.DTYPE_BF16
    L.call("tim_rope_kv_store", _ptr(qkv), _ptr(h), dm, 1e-6, n, _ptr(pos), _ptr(pages), _ptr(cos_t),
           _ptr(sin_t), hq, hkv, d, _ptr(qo), _ptr(kl), _ptr(vl), td, _stream())
    hf = h.float().cpu().numpy()
    x = om.rmsnorm(hf) @ W.float().cpu().numpy()
    tol = 1e-5 if dtype == torch.float32 else 3e-2
    qr = om.rope(x[:, :hq * d].reshape(n, hq, d), np.arange(n, dtype=np.float32), inv)
    vr = x[:, (hq + hkv) * d:].reshape(n, hkv, d)
    assert np.abs(qo.float().cpu().numpy() - qr).max() <= tol * max(1, np.abs(qr).max())
    assert np.abs(vl.float().cpu().numpy() - vr).max() <= tol * max(1, np.abs(vr).max())
    u = (h @ W[:, :64]).contiguous()
    ur = om.silu(om.rmsnorm(hf) @ W[:, :64].float().cpu().numpy())
    L.call("tim_silu_rms", _ptr(u), n, 64, _ptr(h), dm, 1e-6, td, _stream())
    assert np.abs(u.float().cpu().numpy() - ur).max() <= tol * max(1, np.abs(ur).max())


def test_prune_compact_matches_apply():
    rng = np.random.default_rng(9)
    slots, stride = 8, 400
    live_h = np.zeros((slots, stride), dtype=np.int32)
    logical_h = np.zeros((slots, 1000), dtype=np.int32)
    sd = StepDesc()
    expect = {}
    out_row = 0
    for s in range(slots):
        n_log = int(rng.integers(20, 900))
        tokens = rng.integers(0, 265, n_log).tolist()
        logical_h[s, :n_log] = tokens
        applied = []
        for _ in range(int(rng.integers(0, 3))):
            a = int(rng.integers(0, n_log - 1))
            applied.append(opr.Span(a, min(n_log, a + int(rng.integers(1, 60)))))
        live = opr.surgery(list(range(n_log)), applied)[:stride]
        enc = len(live)
        live_h[s, :enc] = live
        plans = []
        for _ in range(int(rng.integers(1, 4))):
            a = int(rng.integers(0, n_log - 1))
            b = min(n_log, a + int(rng.integers(1, 120)))
            plans.append(opr.Plan([opr.Span(a, b)], a, b - a))
        plan = opr.coalesce(plans)
        tab = op.PageTable(s)
        tab.append(list(range(enc)))
        _, suffix_tokens, s0, new_live = opr.apply(plan, tab, list(live), tokens)
        sd.job(s, enc, s0, plan.reencode_from, [(x.start, x.end) for x in plan.spans], out_row,
               len(new_live) - s0)
        expect[s] = (new_live, suffix_tokens, out_row)
        out_row += len(suffix_tokens)
    step = _dev(sd.pack())
    live_d, logical_d = _dev(live_h), _dev(logical_h)
    row_tokens = torch.full((max(out_row, 1),), -1, dtype=torch.int32, device="cuda")
    err = torch.zeros(2, dtype=torch.int32, device="cuda")
    L.call("tim_prune_compact", _ptr(step), slots, _ptr(live_d), stride, _ptr(logical_d), 1000,
           _ptr(row_tokens), _ptr(err), _stream())
    torch.cuda.synchronize()
    assert err.cpu().tolist() == [0, 0]
    lg, rt = live_d.cpu().numpy(), row_tokens.cpu().numpy()
    for s, (new_live, suffix_tokens, orow) in expect.items():
        assert lg[s, :len(new_live)].tolist() == new_live
        assert rt[orow:orow + len(suffix_tokens)].tolist() == suffix_tokens


def test_prune_compact_flags_desync():
    sd = StepDesc()
    sd.job(0, 5, 1, 3, [(3, 4)], 0, 3)  # suffix_start 1 is wrong: live[1] = 1 < 3
    step = _dev(sd.pack())
    live = _dev(np.arange(5, dtype=np.int32)[None, :])
    logical = _dev(np.arange(5, dtype=np.int32)[None, :])
    rt = torch.zeros(8, dtype=torch.int32, device="cuda")
    err = torch.zeros(2, dtype=torch.int32, device="cuda")
    L.call("tim_prune_compact", _ptr(step), 1, _ptr(live), 5, _ptr(logical), 5, _ptr(rt), _ptr(err),
           _stream())
    torch.cuda.synchronize()
    assert int(err[0]) == L.TIM_SPAN_OUT_OF_RANGE
