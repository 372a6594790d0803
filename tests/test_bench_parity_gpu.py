"""Paging parity at the benchmark's own configurations (BASELINE configs 2-4).

oracle/gen_golden.py ran the REFERENCE Engine (scheduler.py:274-335, with
ScriptedModel, model.py:195-233) on exactly the request sets bench.py and
tools/bench_configs.py build, and recorded per step the StepReport fields plus
order-sensitive checksums of every request's block table and live list and of
the pool's free list (paper_2507_16784_b200/checksum.py).  Here the B200
Engine replays the same requests; its K4 (prune compaction) and K5 (page ops)
kernels own the tables, live lists and free stack on the device, and every
recorded step must match bit-exactly:
  c2_g1_r0 : 64 x tool_chain_tree(32), T=2, P=40960, pool 64x1600 (C2, 4381 steps)
  c3_g8_r0 : shard 0 of the 512 requests dealt round-robin over 8 GPUs (C3)
  c3_g2_r1 : shard 1 of 2 (C3)
  c4_slice : 4 x deep_recursion_tree(8,3,text_chars=16) after a 12,000-token
             prompt, T=2, P=16384, to completion (C4: 134,480 tokens each,
             max_cache 13,378 < 16K), checked every 16th step
"""

import gzip
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2507_16784_b200 as tr
from paper_2507_16784_b200.checksum import device_hashes, host_hash, seq_hash_np
from paper_2507_16784_b200.traces import load_corpus, make_trace_from_text

pytestmark = pytest.mark.gpu


def _meta(golden):
    with gzip.open(golden / "bench_runs.json.gz", "rt", encoding="utf-8") as f:
        return json.load(f)


def _docs(golden, name):
    if name.startswith("c4"):
        return load_corpus(golden / "corpus_deep8_3_16.json.gz")
    return load_corpus(golden / "corpus_tool_chain32.json.gz")


def replay_and_check(golden, name, backend=None):
    meta = next(s for s in _meta(golden)["scenarios"] if s["name"] == name)
    rows = np.load(golden / "bench_runs.npz")[name]
    docs = _docs(golden, name)
    P = meta["position_limit"]
    eng = tr.Engine(backend or tr.ScriptedModel(position_limit=P), tr.BatchConfig(**meta["config"]))
    prompts = ["a" * 12000] * 4 if name.startswith("c4") else meta["prompts"]
    for d, prompt in zip(meta["docs"], prompts):
        t = make_trace_from_text(docs[d])
        eng.submit(prompt, [tr.ToolSpec(n) for n in t.tool_names], script=t.script,
                   tool_responses=t.tool_responses or None)
    by_step = {int(r[0]): r for r in rows}
    checked = 0
    while not eng.all_terminal():
        rep = eng.step()
        g = by_step.get(rep.step)
        if g is None:
            continue
        pend = {rid: len(eng.requests[rid].pending) for rid in rep.request_live}
        mine = [rep.step, rep.active, rep.awaiting_tool, rep.finished, rep.failed, rep.pages_free,
                rep.flops_units, host_hash(rep.request_live, pend, rep.decoded), *device_hashes(eng)]
        assert mine == [int(x) for x in g], (name, rep.step, mine, g.tolist())
        checked += 1
        if checked % 512 == 0:
            eng.runtime.check()          # device error word (K4/K5 faults)
    eng.runtime.check()
    assert eng.step_index == meta["n_steps"]
    for rid, g in meta["requests"].items():
        r = eng.requests[rid]
        assert r.status.value == g["status"]
        m = eng.result(rid)["metrics"]
        for k in ("output_len", "max_cache", "position_high_water", "tool_calls", "pruned_tokens"):
            assert m[k] == g["metrics"][k], (name, rid, k)
        assert len(r.eviction_log) == g["evictions"]
        assert seq_hash_np([x for s in r.eviction_log for x in (s.start, s.end)]) == g["eviction_hash"]
        assert seq_hash_np([x for s in r.applied_spans for x in (s.start, s.end)]) == g["applied_hash"]
        assert seq_hash_np(r.logical) == g["logical_hash"]
    assert eng.pool.free_count == eng.pool.capacity
    return eng, checked


@pytest.mark.parametrize("name", ["c2_g1_r0", "c3_g8_r0", "c3_g2_r1"])
def test_bench_config_paging_bit_exact(golden, name):
    _, checked = replay_and_check(golden, name)
    assert checked > 4000


def test_c4_long_horizon_paging_bit_exact(golden):
    """>128K generated tokens per request with < 16K retained: every 16th
    step's tables / live lists / free stack match the reference, no page leaks."""
    eng, checked = replay_and_check(golden, "c4_slice")
    assert checked > 8000
    for r in eng.requests.values():
        assert r.metrics.output_len == 134480 and r.metrics.max_cache < 16384
