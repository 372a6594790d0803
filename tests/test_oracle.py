"""Pin the CPU oracle to the reference (CPU-only).

Golden data: tests/golden/*, produced by oracle/gen_golden.py from the
reference's own code (tokenizer.py, tracker.py, scheduler.py with
ScriptedModel / TinyTransformer).  Known-answer vectors are the reference
unit tests' (file:line cited per test).
"""

import gzip
import json
import random
import zlib

import numpy as np
import pytest

from oracle import engine as oe
from oracle import model as om
from oracle import paging as op
from oracle import pruning as opr
from paper_2507_16784_b200.tokenizer import build_tokenizer


def _load(golden, name):
    with gzip.open(golden / name, "rt", encoding="utf-8") as f:
        return json.load(f)


def crc(ids):
    return zlib.crc32(np.asarray(ids, dtype=np.int32).tobytes())


# ---------------------------------------------------------------- known answers
def test_apply_worked_example():
    """tests/test_pruning.py:107-118 (paper §3.1)."""
    pool = op.PagePool(12)
    t = op.PageTable("r")
    t.append(pool.alloc("r", 6))
    freed, suffix, start, new_live = opr.apply(opr.Plan([opr.Span(1, 3)], 1, 2), t, list(range(6)),
                                               [101, 111, 112, 102, 121, 999])
    assert len(freed) == 5 and suffix == [102, 121, 999] and start == 1
    assert new_live == [0, 3, 4, 5] and len(t) == 1


def test_apply_overlap_and_suffix_final():
    """tests/test_pruning.py:120-138."""
    pool = op.PagePool(20)
    t = op.PageTable("r")
    t.append(pool.alloc("r", 10))
    _, suffix, start, new_live = opr.apply(opr.Plan([opr.Span(6, 10)], 6, 4), t, list(range(10)),
                                           list(range(10)))
    assert suffix == [] and start == 6 and new_live == list(range(6))
    t2 = op.PageTable("q")
    t2.append(pool.alloc("q", 10))
    live = [0, 1, 2, 3, 6, 7, 8, 9, 10, 11]
    _, suffix, start, new_live = opr.apply(opr.Plan([opr.Span(2, 9)], 2, 7), t2, live, list(range(12)))
    assert new_live == [0, 1, 9, 10, 11] and suffix == [9, 10, 11] and start == 2


def test_buffer_semantics():
    """tests/test_pruning.py:25-58."""
    b = opr.Buffer(0)
    p = b.on_list_closed(opr.Span(5, 9))
    assert p.spans == [opr.Span(5, 9)] and p.reencode_from == 5 and p.freed == 4
    b = opr.Buffer(1)
    assert b.on_list_closed(opr.Span(2, 6)) is None
    assert b.on_list_closed(opr.Span(10, 14)).spans == [opr.Span(2, 6)]
    b = opr.Buffer(2)
    b.on_list_closed(opr.Span(4, 8))
    b.on_list_closed(opr.Span(2, 12))
    assert b.entries == [opr.Span(2, 12)]
    b = opr.Buffer(2, subsume=False)
    b.on_list_closed(opr.Span(4, 8))
    b.on_list_closed(opr.Span(2, 12))
    assert b.on_list_closed(opr.Span(20, 24)).spans == [opr.Span(4, 8)]


def test_coalesce_random_union():
    """tests/test_pruning.py:74-93."""
    rng = random.Random(1)
    for _ in range(200):
        plans = []
        for _ in range(rng.randint(1, 5)):
            a = rng.randrange(0, 50)
            b = a + rng.randrange(1, 10)
            plans.append(opr.Plan([opr.Span(a, b)], a, b - a))
        out = opr.coalesce(plans)
        expect = set().union(*[set(range(s.start, s.end)) for p in plans for s in p.spans])
        got = set()
        for s in out.spans:
            ids = set(range(s.start, s.end))
            assert not (ids & got)
            got |= ids
        assert got == expect and out.reencode_from == min(expect)


def test_kv_pruned_pct_paper_rows():
    """tests/test_acceptance.py:56-60."""
    assert opr.kv_pruned_pct(1569.2, 3362.2) == pytest.approx(0.533, abs=1e-3)
    assert opr.kv_pruned_pct(3218.6, 8974.7) == pytest.approx(0.641, abs=1e-3)
    assert opr.kv_pruned_pct(4096, 4096) == 0.0


def test_lifo_pool_interleaving():
    """SURVEY appendix A3 shape: pops 0,1,2,...; frees come back reversed."""
    pool = op.PagePool(8)
    a = pool.alloc("a", 3)
    b = pool.alloc("b", 2)
    assert a == [0, 1, 2] and b == [3, 4]
    pool.free(a)
    assert pool.alloc("c", 3) == [2, 1, 0]


# ------------------------------------------------------------- oracle engine
def _events_for(trace):
    if trace["script"] and not trace["events"]:
        return {0: "reject"}
    return oe.event_table(trace["events"])


def _run_oracle(scen):
    cfg = scen["config"]
    P = scen["position_limit"]
    tok = build_tokenizer()
    eng = oe.Engine(oe.Accounting(P), max_batch=cfg["max_batch"], threshold=cfg["buffer_threshold"],
                    position_limit=P, pool_pages=cfg["pool_pages"], max_queue=cfg["max_queue"],
                    starvation_steps=cfg["starvation_steps"], subsume=cfg["subsume"],
                    max_output_tokens=cfg["max_output_tokens"], tokenize=tok.tokenize)
    rids = []
    for i, tr in enumerate(scen["traces"]):
        th = None if scen["thresholds"] is None else scen["thresholds"][i]
        rids.append(eng.submit(tok.tokenize(scen["prompts"][i]), tr["script"],
                               {int(k): v for k, v in tr["tool_responses"].items()},
                               _events_for(tr), threshold=th, subsume=scen["subsume"]))
    return eng, rids


def test_oracle_engine_matches_reference_runs(golden):
    scens = _load(golden, "engine_runs.json.gz")
    assert len(scens) >= 15
    for scen in scens:
        eng, rids = _run_oracle(scen)
        assert rids == scen["rids"]
        for i, gs in enumerate(scen["steps"]):
            rep = eng.step()
            where = (scen["name"], i)
            assert rep["report"] == gs["report"], where
            assert rep["request_live"] == gs["request_live"], where
            assert rep["decoded"] == gs["decoded"], where
            for rid, g in gs["reqs"].items():
                r = eng.requests[rid]
                assert [r.status, len(r.live), len(r.pending), len(r.table), r.pruned_tokens] == \
                    [g["status"], g["live"], g["pending"], g["n_pages"], g["pruned"]], where
                assert crc(r.table.pages) == g["crc"], where
                if "pages" in g:
                    assert r.table.pages == g["pages"], where
            assert [eng.pool.free_count, crc(eng.pool.free_list)] == gs["free"], where
        assert eng.all_terminal(), scen["name"]
        for rid, g in scen["requests"].items():
            r = eng.requests[rid]
            assert [[s.start, s.end] for s in r.eviction_log] == g["eviction_log"], (scen["name"], rid)
            assert [[s.start, s.end] for s in r.applied_spans] == g["applied_spans"]
            assert r.logical == g["logical"]
            res = g["result"]
            assert eng.results[rid]["status"] == res["status"]
            m = eng.results[rid]["metrics"]
            for k in ("output_len", "max_cache", "position_high_water", "tool_calls", "pruned_tokens"):
                assert m[k] == res["metrics"][k], (scen["name"], rid, k)
            if res["status"] == "failed":
                assert eng.results[rid]["failure"].split(":")[0] == res["failure"].split(":")[0]


# -------------------------------------------------------------- oracle model
def _ref_arrays(golden):
    return np.load(golden / "model_ref.npz")


@pytest.mark.parametrize("tag,cfg", [
    ("d16", om.Config()),
    ("c1", om.Config(layers=2, heads=4, head_dim=32, vocab=512, position_limit=2048)),
])
def test_oracle_model_matches_reference(golden, tag, cfg):
    ref = _ref_arrays(golden)
    m = om.Model(cfg)
    assert np.array_equal(m.w["emb"][:4], ref[f"{tag}_emb"])
    assert np.array_equal(m.w["layers"][0]["wq"][:2], ref[f"{tag}_wq0"])
    assert np.array_equal(m.w["layers"][-1]["w2"][-2:], ref[f"{tag}_w2_last"])
    seq = [3, 99, 260, 45, 7, 123, 264, 10, 11, 500]
    pool, t = m.make_pool(64), op.PageTable("t")
    logits = m.prefill(seq, list(range(len(seq))), t, pool)
    k, v = op.gather(pool, t)
    for got, key in ((logits, "prefill_logits"), (k, "prefill_k"), (v, "prefill_v")):
        r = ref[f"{tag}_{key}"]
        assert np.abs(got - r).max() / np.abs(r).max() < 1e-6, key
    seq6 = [5, 6, 7, 8, 9, 10]
    pool, t = m.make_pool(64), op.PageTable("t")
    m.prefill(seq6, list(range(6)), t, pool)
    pool.free(t.truncate_from(1))
    lg = m.extend(seq6[3:], 1, t, pool)
    k, v = op.gather(pool, t)
    for got, key in ((lg, "reencode_logits"), (k, "reencode_k"), (v, "reencode_v")):
        r = ref[f"{tag}_{key}"]
        assert np.abs(got - r).max() / np.abs(r).max() < 1e-6, key


def test_gqa_reduces_to_reference_when_kv_equals_heads():
    a = om.init_weights(om.Config(layers=1, heads=4, head_dim=8))
    b = om.init_weights(om.Config(layers=1, heads=4, head_dim=8, kv_heads=4, mlp_dim=128))
    for k in ("wq", "wk", "wv", "wo", "w1", "w2"):
        assert np.array_equal(a["layers"][0][k], b["layers"][0][k])


def test_oracle_engine_matches_reference_bench_config(golden):
    """The oracle engine pinned at the C2 bench configuration (64 x
    tool_chain_tree(32), T=2, P=40960): the first 600 steps' reports and
    table / live / free-list checksums equal the reference run's
    (tests/golden/bench_runs.*, oracle/gen_golden.py gen_bench)."""
    import gzip as _gz
    import json as _json
    from paper_2507_16784_b200.checksum import host_hash, seq_hash_np
    from paper_2507_16784_b200.grammar import Grammar
    from paper_2507_16784_b200.traces import load_corpus, make_trace_from_text
    with _gz.open(golden / "bench_runs.json.gz", "rt") as f:
        meta = next(s for s in _json.load(f)["scenarios"] if s["name"] == "c2_g1_r0")
    rows = np.load(golden / "bench_runs.npz")["c2_g1_r0"]
    docs = load_corpus(golden / "corpus_tool_chain32.json.gz")
    cfg = meta["config"]
    tok = build_tokenizer()
    eng = oe.Engine(oe.Accounting(40960), max_batch=64, threshold=cfg["buffer_threshold"],
                    position_limit=40960, pool_pages=cfg["pool_pages"], max_queue=cfg["max_queue"],
                    max_output_tokens=cfg["max_output_tokens"], tokenize=tok.tokenize)
    for d, prompt in zip(meta["docs"], meta["prompts"]):
        t = make_trace_from_text(docs[d])
        sc, evs, stream, call = Grammar(t.tool_names, 16, tok).tracker(), [], [], 0
        for tid in t.script:
            for e in sc.feed(tid):
                evs.append([e.kind, len(stream), e.depth, e.payload])
            stream.append(tid)
            if any(e[0] == "ToolResultSlotOpened" and e[1] == len(stream) - 1 for e in evs[-3:]):
                text = _json.dumps(t.tool_responses[call], separators=(",", ":"), ensure_ascii=False)
                for rt_ in tok.tokenize(text):
                    for e in sc.feed(rt_):
                        evs.append([e.kind, len(stream), e.depth, e.payload])
                    stream.append(rt_)
                call += 1
        eng.submit(tok.tokenize(prompt), t.script, t.tool_responses, oe.event_table(evs))
    for g in rows[:600]:
        rep = eng.step()
        live = rep["request_live"]
        pend = {rid: len(eng.requests[rid].pending) for rid in live}
        th = lh = 0
        for rid, r in eng.requests.items():
            if r.table.pages:
                th += seq_hash_np(r.table.pages, int(rid[1:]))
                lh += seq_hash_np(r.live, int(rid[1:]))
        mine = list(rep["report"]) + [host_hash(live, pend, rep["decoded"]), th, lh,
                                      seq_hash_np(eng.pool.free_list)]
        assert mine == [int(x) for x in g], (int(g[0]), mine, g.tolist())
