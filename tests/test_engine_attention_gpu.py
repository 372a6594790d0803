"""Attention outputs INSIDE the batched engine at the C2 shape (GPU).

The kernel tests (test_kernels_gpu.py) feed synthetic tables; here the
engine's own step does the work: 64 tool_chain_tree(32) requests (the bench's
C2 request set), T=2, Qwen3-8B head shape (32 q / 8 kv heads x 128) in bf16,
so the decode tiles (K1), the tcgen05 multi-token items (K2) and the
one-launch split see the real mix of decode rows, re-encoded suffixes and tool
responses.  After sampled steps the last layer's RoPE'd queries (rt.q) and
attention outputs (rt.ctx) are compared, segment by segment, with the fp32
oracle attention (oracle/model.py attend, model.py:149-159 + GQA) over the
bf16 K/V the engine stored in its pool pages:

    max |ctx - attend(q, K[pages], V[pages], m)| <= 2e-2   (BASELINE north_star)
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2507_16784_b200 as tr
from oracle import model as om
from paper_2507_16784_b200.traces import load_corpus, make_trace_from_text

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def _check_step(eng, cfg):
    sd, rt, pool = eng._sd, eng.runtime, eng.pool
    li = cfg.layers - 1
    T = sd.n_rows
    q = rt.q[:T].float().view(T, cfg.heads, cfg.head_dim)
    ctx = rt.ctx[:T].float().view(T, cfg.heads, cfg.head_dim)
    worst = 0.0
    for slot, m, n, row in sd.segs:
        pages = rt.tables[slot, : m + n].long()
        k = pool.K_layers[li].index_select(0, pages).float().cpu().numpy()
        v = pool.V_layers[li].index_select(0, pages).float().cpu().numpy()
        ref = om.attend(q[row:row + n].cpu().numpy(), k, v, m)
        err = float(np.abs(ctx[row:row + n].cpu().numpy() - ref).max())
        assert err <= BF16_TOL, (eng.step_index, slot, m, n, err)
        worst = max(worst, err)
    return worst


def test_engine_attention_outputs_c2_shape(golden):
    cfg = tr.ModelConfig(layers=2, heads=32, kv_heads=8, head_dim=128, mlp_dim=12288, vocab=512,
                         position_limit=40960, rope_base=1e6, precision="bfloat16",
                         weight_init="device")
    model = tr.B200Transformer(cfg)
    docs = load_corpus(golden / "corpus_tool_chain32.json.gz")[:64]
    eng = tr.Engine(model, tr.BatchConfig(max_batch=64, buffer_threshold=2, position_limit=40960,
                                          pool_pages=64 * 1600, max_queue=64, check_masks=False,
                                          max_output_tokens=20000, check_device=True))
    for i, d in enumerate(docs):
        t = make_trace_from_text(d)
        eng.submit(f"q{i}:", [tr.ToolSpec(n) for n in t.tool_names], script=t.script,
                   tool_responses=t.tool_responses)
    n_dec = n_mixed = 0
    worst = 0.0
    rows_seen = []
    for step in range(1400):
        eng.step()
        sd = eng._sd
        if sd.n_rows == 0:
            continue
        if sd.ext and n_mixed < 16:
            worst = max(worst, _check_step(eng, cfg))
            n_mixed += 1
            rows_seen.append(sd.n_rows)
        elif not sd.ext and step % 97 == 5:
            worst = max(worst, _check_step(eng, cfg))
            n_dec += 1
    assert n_mixed >= 8 and n_dec >= 8, (n_mixed, n_dec)
    assert max(rows_seen) > 64 + 100          # a re-encode / tool response of >100 rows was checked
    print(f"checked {n_dec} decode and {n_mixed} mixed steps, worst |d ctx| {worst:.3g}")
