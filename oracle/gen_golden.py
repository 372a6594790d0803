"""Generate golden fixtures by running the REFERENCE (threadrun) in the build container.

Usage (needs /root/reference; never runs on the GPU box):
    PYTHONDONTWRITEBYTECODE=1 python -m oracle.gen_golden

Writes tests/golden/*.json.gz / *.npz.  Everything the B200 path must match
bit-exactly (token ids, structure events, eviction logs, page ids per step,
metrics) or within tolerance (fp32 logits / K / V) is dumped here from the
reference's own code paths:
  tokenizer.py ByteTokenizer.tokenize, tracker.py Tracker.feed,
  scheduler.py Engine.step with model.py ScriptedModel / TinyTransformer.
"""

from __future__ import annotations

import gzip
import zlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("THREADRUN_SRC", "/root/reference/pkg/src"))
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF))

from threadrun.model import ModelConfig, ScriptedModel, TinyTransformer  # noqa: E402
from threadrun.paging import PageTable, gather  # noqa: E402
from threadrun.scheduler import BatchConfig, Engine  # noqa: E402
from threadrun.schema import (ToolSpec, deep_recursion_tree, random_tree,  # noqa: E402
                              tool_chain_tree)
from threadrun.tokenizer import build_tokenizer  # noqa: E402
from threadrun.tracker import ThreadGrammar, TOOL_RESULT_SLOT_OPENED  # noqa: E402
from threadrun.traces import make_trace  # noqa: E402

TOK = build_tokenizer()
TOOLS = (ToolSpec("search"), ToolSpec("calc"))


def dump(name: str, obj) -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    with gzip.open(OUT / name, "wt", encoding="utf-8") as f:
        json.dump(obj, f, separators=(",", ":"))


def trace_record(tree, tools=None):
    trace = make_trace(tree, TOK)
    names = list(trace.tool_names)
    tools = tools if tools is not None else [ToolSpec(n) for n in names]
    grammar = ThreadGrammar(list(tools), 16, TOK)
    tr = grammar.tracker()
    stream, events = [], []
    call = 0
    script = list(trace.script)
    i = 0
    while i < len(script):
        tid = script[i]
        i += 1
        evs = tr.feed(tid)
        stream.append(tid)
        slot_opened = False
        for e in evs:
            events.append([e.kind, e.offset, e.depth, e.payload])
            if e.kind == TOOL_RESULT_SLOT_OPENED:
                slot_opened = True
        if slot_opened:
            # scheduler.py:469-472 override, then _integrate (477-499) feeds the response
            value = trace.tool_responses.get(call)
            call += 1
            text = json.dumps(value, separators=(",", ":"), ensure_ascii=False)
            for rt in TOK.tokenize(text):
                for e in tr.feed(rt):
                    events.append([e.kind, e.offset, e.depth, e.payload])
                stream.append(rt)
    return {
        "script": script,
        "tool_responses": {str(k): v for k, v in trace.tool_responses.items()},
        "tool_names": names,
        "text": trace.text,
        "stream": stream,
        "events": events,
    }


def gen_tokenizer():
    texts = ["", "p:", "task:", "hello world", '[{"thought":"a","conclusion":"b"}]',
             '{"q":"café \\"hi\\"","k":3}', '}]},{"thought":', '[[{{}}]]', "é中\n\t"]
    for s in range(6):
        texts.append(make_trace(random_tree(s, 3, 3, tool_prob=0.5), TOK).text)
    dump("tokenizer.json.gz", [[t, TOK.tokenize(t)] for t in texts])


def gen_events():
    recs = []
    for seed in range(150):
        r = trace_record(random_tree(seed, 4, 3, tool_prob=0.3))
        r["gen"] = ["random_tree", seed, 4, 3, 0.3]
        recs.append(r)
    for args in [(3, 2, 0), (4, 2, 1), (6, 2, 0), (3, 3, 5)]:
        r = trace_record(deep_recursion_tree(args[0], args[1], seed=args[2]))
        r["gen"] = ["deep_recursion_tree", *args]
        recs.append(r)
    for n in (1, 4, 8):
        r = trace_record(tool_chain_tree(n, seed=n))
        r["gen"] = ["tool_chain_tree", n]
        recs.append(r)
    dump("events.json.gz", recs)


def crc(ids) -> int:
    return zlib.crc32(np.asarray(ids, dtype=np.int32).tobytes())


def _snap(engine, rids, full):
    reqs = {}
    for rid in rids:
        r = engine.requests[rid]
        reqs[rid] = {"status": r.status.value, "live": len(r.live), "pending": len(r.pending),
                     "n_pages": len(r.table.pages), "crc": crc(r.table.pages),
                     "pruned": r.metrics.pruned_tokens}
        if full:
            reqs[rid]["pages"] = list(r.table.pages)
    return reqs


def run_scenario(name, traces, cfg, prompts=None, thresholds=None, position_limit=4096,
                 subsume=None, full_pages=True):
    engine = Engine(ScriptedModel(position_limit=position_limit), cfg)
    rids = []
    for i, tr in enumerate(traces):
        prompt = prompts[i] if prompts else f"p{i}:"
        tools = [ToolSpec(n) for n in tr["tool_names"]]
        rids.append(engine.submit(
            prompt, tools, script=tr["script"],
            tool_responses={int(k): v for k, v in tr["tool_responses"].items()} or None,
            threshold=None if thresholds is None else thresholds[i],
            subsume=subsume))
    steps = []
    guard = 0
    while not engine.all_terminal():
        rep = engine.step()
        guard += 1
        assert guard < 100000
        steps.append({
            "report": [rep.step, rep.active, rep.awaiting_tool, rep.finished, rep.failed,
                       rep.pages_free, rep.flops_units],
            "request_live": rep.request_live, "decoded": rep.decoded,
            "reqs": _snap(engine, rids, full_pages and len(steps) % 25 == 0),
            "free": [len(engine.pool.free_list), crc(engine.pool.free_list)],
        })
    out = {"name": name, "config": cfg.__dict__, "position_limit": position_limit,
           "prompts": [prompts[i] if prompts else f"p{i}:" for i in range(len(traces))],
           "thresholds": thresholds, "subsume": subsume, "traces": traces, "rids": rids,
           "steps": steps, "requests": {}}
    for rid in rids:
        r = engine.requests[rid]
        out["requests"][rid] = {
            "result": engine.result(rid),
            "eviction_log": [[s.start, s.end] for s in r.eviction_log],
            "applied_spans": [[s.start, s.end] for s in r.applied_spans],
            "transitions": r.transitions,
            "logical": r.logical,
        }
    return out


def gen_engine():
    ev = {}
    def rt(*a):
        key = a
        if key not in ev:
            fn = {"random": random_tree, "deep": deep_recursion_tree, "chain": tool_chain_tree}[a[0]]
            if a[0] == "random":
                tree = fn(a[1], a[2], a[3], tool_prob=a[4])
            elif a[0] == "deep":
                tree = fn(a[1], a[2], seed=a[3])
            else:
                tree = fn(a[1], seed=a[2])
            ev[key] = trace_record(tree)
        return ev[key]

    scen = []
    deep32 = rt("deep", 3, 2, 0)
    for t in (0, 1, 2):
        scen.append(run_scenario(f"deep32_T{t}", [deep32], BatchConfig(
            buffer_threshold=t, position_limit=256, pool_pages=256), prompts=["p:"], position_limit=256))
    scen.append(run_scenario("two_requests_T0", [deep32, deep32], BatchConfig(
        max_batch=2, buffer_threshold=0, position_limit=256, pool_pages=512),
        prompts=["a:", "b:"], position_limit=256))
    mix = [rt("random", s, 4, 3, 0.3) for s in (1, 5, 9, 12)]
    for t in (0, 1, 2, 5):
        scen.append(run_scenario(f"mix4_T{t}_b2", mix, BatchConfig(
            max_batch=2, buffer_threshold=t, position_limit=4096, pool_pages=8192)))
        scen.append(run_scenario(f"mix4_T{t}_b4", mix, BatchConfig(
            max_batch=4, buffer_threshold=t, position_limit=4096, pool_pages=8192)))
    scen.append(run_scenario("mix4_T1_nosubsume", mix, BatchConfig(
        max_batch=4, buffer_threshold=1, position_limit=4096, pool_pages=8192, subsume=False)))
    scen.append(run_scenario("mix4_per_request_T", mix, BatchConfig(
        max_batch=4, buffer_threshold=1, position_limit=4096, pool_pages=8192),
        thresholds=[0, 2, 1, 1 << 30]))
    chain = [rt("chain", 6, s) for s in (0, 1, 2)]
    for t in (1, 2):
        scen.append(run_scenario(f"chain3_T{t}", chain, BatchConfig(
            max_batch=3, buffer_threshold=t, position_limit=4096, pool_pages=8192)))
    # out of pages: parks, starves (tests/test_scheduler.py:187-200)
    deep72 = rt("deep", 7, 2, 0)
    scen.append(run_scenario("oop_starve", [deep72, deep72], BatchConfig(
        buffer_threshold=1 << 30, position_limit=4096, pool_pages=120, max_batch=2,
        starvation_steps=10), prompts=["a:", "b:"]))
    # position overflow (tests/test_scheduler.py:170-185 shape)
    scen.append(run_scenario("pos_overflow", [rt("random", 2, 2, 2, 0.0), rt("random", 3, 3, 3, 0.0)],
                             BatchConfig(buffer_threshold=1, position_limit=128, pool_pages=512,
                                         max_batch=4), prompts=["ok:", "p:"], position_limit=128))
    # rejected first token (tests/test_scheduler.py:137-146), empty prompt
    bad = {"script": [ord("x")], "tool_responses": {}, "tool_names": [], "text": "x", "stream": [],
           "events": []}
    scen.append(run_scenario("reject_and_ok", [rt("random", 2, 3, 2, 0.0), bad], BatchConfig(
        buffer_threshold=0, max_batch=4, position_limit=4096, pool_pages=8192), prompts=["a:", "b:"]))
    scen.append(run_scenario("empty_prompt", [rt("random", 2, 2, 2, 0.0)], BatchConfig(
        buffer_threshold=1 << 30, position_limit=4096, pool_pages=8192), prompts=[""]))
    # beyond-limit generation (acceptance 3 shape, smaller): deep(7,2) at P=128, T=1
    scen.append(run_scenario("beyond_limit", [deep72], BatchConfig(
        buffer_threshold=1, position_limit=128, pool_pages=512), prompts=["g:"], position_limit=128))
    dump("engine_runs.json.gz", scen)


def gen_model():
    arrays = {}
    for tag, cfg in [("d16", ModelConfig()),
                     ("c1", ModelConfig(layers=2, heads=4, head_dim=32, vocab=512,
                                        position_limit=2048))]:
        m = TinyTransformer(cfg)
        seq = [3, 99, 260, 45, 7, 123, 264, 10, 11, 500][: 10]
        pool = m.make_pool(64)
        t = PageTable("t")
        logits = m.prefill(seq, list(range(len(seq))), t, pool)
        k, v = gather(pool, t)
        arrays[f"{tag}_prefill_logits"] = logits
        arrays[f"{tag}_prefill_k"] = k
        arrays[f"{tag}_prefill_v"] = v
        # extend after prune (tests/test_model.py:115-131)
        seq6 = [5, 6, 7, 8, 9, 10]
        pool = m.make_pool(64)
        t = PageTable("t")
        m.prefill(seq6, list(range(6)), t, pool)
        pool.free(t.truncate_from(1))
        lg = m.extend(seq6[3:], 1, t, pool)
        k, v = gather(pool, t)
        arrays[f"{tag}_reencode_logits"] = lg
        arrays[f"{tag}_reencode_k"] = k
        arrays[f"{tag}_reencode_v"] = v
        arrays[f"{tag}_emb"] = m.emb[:4]
        arrays[f"{tag}_wq0"] = m.layers[0]["wq"][:2]
        arrays[f"{tag}_w2_last"] = m.layers[-1]["w2"][-2:]
    # C1 numeric replay: deep(3,2,seed 0) prompt "p:" T=1; logits after every step
    cfg = ModelConfig(layers=2, heads=4, head_dim=32, vocab=512, position_limit=2048)
    tr = trace_record(deep_recursion_tree(3, 2, seed=0))
    engine = Engine(TinyTransformer(cfg), BatchConfig(buffer_threshold=1, position_limit=2048,
                                                      pool_pages=4096))
    rid = engine.submit("p:", [], script=tr["script"])
    req = engine.requests[rid]
    logits, kv_after = [], None
    while not engine.all_terminal():
        engine.step()
        if req.last_logits is not None and req.status.value == "decoding":
            logits.append(np.asarray(req.last_logits))
        if req.metrics.pruned_tokens and kv_after is None and req.status.value == "decoding":
            kv_after = gather(engine.pool, req.table)
    arrays["c1_replay_logits"] = np.stack(logits)
    arrays["c1_replay_k_after_prune"] = kv_after[0]
    arrays["c1_replay_v_after_prune"] = kv_after[1]
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / "model_ref.npz", **arrays)


def gen_corpus():
    """Bench/parity corpora: the reference generators' exact documents."""
    c2 = [make_trace(tool_chain_tree(32, seed=i), TOK).text for i in range(512)]
    dump("corpus_tool_chain32.json.gz", c2)
    c1 = [make_trace(random_tree(s, 3, 3, tool_prob=0.3), TOK).text for s in range(100)]
    dump("corpus_random_3_3.json.gz", c1)
    # acceptance criterion 1 (tests/test_acceptance.py:40-53): verify.suite_prune_extend's trees
    a1 = [make_trace(random_tree(s, 4, 2, tool_prob=0.25), TOK).text for s in range(100)]
    dump("corpus_random_4_2_025.json.gz", a1)


# ------------------------------------------------------------------------------
# Bench-configuration runs (BASELINE configs 2-4): per-step checksums of the
# reference Engine's paging state, in the definition of
# paper_2507_16784_b200/checksum.py (restated here in numpy so the generator
# does not depend on the product package).
_MUL, _STRIDE = 2654435761, 7919


def _w(idx):
    idx = np.asarray(idx, dtype=np.int64)
    return (((idx * _MUL) & 0xFFFFFFFF) >> 16) + 1


def _seq_hash(values, k=0):
    v = np.asarray(values, dtype=np.int64)
    if v.size == 0:
        return 0
    return int(((v + 1) * _w(np.arange(v.size, dtype=np.int64) + _STRIDE * k)).sum())


def _host_hash(live_lens, pending_lens, decoded):
    h = 0
    for rid, n in live_lens.items():
        k = int(rid[1:])
        h += (n + 1) * int(_w(3 * k)) + (pending_lens.get(rid, 0) + 1) * int(_w(3 * k + 1))
    for rid, n in decoded.items():
        k = int(rid[1:])
        h += (n + 1) * int(_w(3 * k + 2))
    return h & 0x7FFFFFFFFFFFFFFF


BENCH_COLS = ["step", "active", "awaiting_tool", "finished", "failed", "pages_free", "flops_units",
              "host_hash", "table_hash", "live_hash", "free_hash"]


class _WorkRecorder(ScriptedModel):
    """ScriptedModel that logs every forward the reference Engine asks for:
    (step, request index, start = prefix length m, n rows)."""

    def __init__(self, position_limit):
        super().__init__(position_limit=position_limit)
        self.engine = None
        self.calls = []

    def _log(self, table, start, n):
        self.calls.append((self.engine.step_index + 1, int(table.request_id[1:]), start, n))

    def prefill(self, tokens, positions, table, pool):
        self._log(table, len(table.pages), len(tokens))
        return super().prefill(tokens, positions, table, pool)

    def extend(self, tokens, start_position, table, pool):
        self._log(table, start_position, len(tokens))
        return super().extend(tokens, start_position, table, pool)


def run_bench_scenario(name, docs, prompts, cfg, position_limit, every=1, record_work=False):
    """Reference scripted Engine over `docs`; one checksum row per `every` steps
    (and the last step).  Returns (rows int64 [n, 11], meta)."""
    backend = _WorkRecorder(position_limit) if record_work else ScriptedModel(position_limit=position_limit)
    engine = Engine(backend, cfg)
    if record_work:
        backend.engine = engine
    rids = []
    for doc, prompt in zip(docs, prompts):
        tr = make_trace_from_doc(doc)
        rids.append(engine.submit(prompt, [ToolSpec(n) for n in tr.tool_names], script=tr.script,
                                  tool_responses=tr.tool_responses or None))
    rows = []
    decoded = []
    while not engine.all_terminal():
        rep = engine.step()
        decoded.append(sum(rep.decoded.values()))
        if rep.step % every and not engine.all_terminal():
            continue
        pend = {rid: len(engine.requests[rid].pending) for rid in rep.request_live}
        th = lh = 0
        for rid in rids:
            r = engine.requests[rid]
            k = int(rid[1:])
            if r.table.pages:
                th += _seq_hash(r.table.pages, k)
                lh += _seq_hash(r.live, k)
        rows.append([rep.step, rep.active, rep.awaiting_tool, rep.finished, rep.failed,
                     rep.pages_free, rep.flops_units, _host_hash(rep.request_live, pend, rep.decoded),
                     th, lh, _seq_hash(engine.pool.free_list)])
    meta = {"name": name, "config": cfg.__dict__, "position_limit": position_limit, "every": every,
            "prompts": prompts, "rids": rids, "n_steps": engine.step_index, "requests": {}}
    for rid in rids:
        r = engine.requests[rid]
        meta["requests"][rid] = {
            "status": r.status.value,
            "metrics": r.metrics.to_dict(),
            "evictions": len(r.eviction_log),
            "eviction_hash": _seq_hash([x for s in r.eviction_log for x in (s.start, s.end)]),
            "applied_hash": _seq_hash([x for s in r.applied_spans for x in (s.start, s.end)]),
            "logical_hash": _seq_hash(r.logical),
        }
    if record_work:
        meta["work"] = np.asarray(backend.calls, dtype=np.int32)
        meta["decoded"] = np.asarray(decoded, dtype=np.int32)
    return np.asarray(rows, dtype=np.int64), meta


def make_trace_from_doc(doc):
    from threadrun.schema import parse_tree_text
    return make_trace(parse_tree_text(doc), TOK)


def gen_bench():
    """C2 (64 x tool_chain_tree(32), T=2, P=40960, pool 64x1600), C3 shards
    (512 documents dealt round-robin over G GPUs) and a C4 slice (4 x
    deep_recursion_tree(8,3,text_chars=16) after a 12,000-token prompt, P=16384,
    to completion): exactly the engines bench.py / tools/bench_configs.py build."""
    import time
    chain = [make_trace(tool_chain_tree(32, seed=i), TOK).text for i in range(512)]
    arrays, metas = {}, []

    def c23(name, G, r):
        idx = [i for i in range(64 * G) if i % G == r]
        cfg = BatchConfig(max_batch=64, buffer_threshold=2, position_limit=40960, pool_pages=64 * 1600,
                          max_queue=64, check_masks=False, max_output_tokens=20000)
        t0 = time.time()
        rows, meta = run_bench_scenario(name, [chain[i] for i in idx], [f"q{i}:" for i in idx], cfg, 40960,
                                        record_work=(G == 1))
        if "work" in meta:
            # every forward of the C2 run: the CPU baseline's per-step work list
            arrays["c2_work"] = meta.pop("work")
            arrays["c2_decoded"] = meta.pop("decoded")      # first-encoded tokens per step
        meta["docs"] = idx
        print(name, rows.shape, f"{time.time() - t0:.0f}s")
        arrays[name] = rows
        metas.append(meta)

    c23("c2_g1_r0", 1, 0)
    c23("c3_g8_r0", 8, 0)
    c23("c3_g2_r1", 2, 1)
    deep = [make_trace(deep_recursion_tree(8, 3, seed=i, text_chars=16), TOK).text for i in range(4)]
    dump("corpus_deep8_3_16.json.gz", deep)
    cfg = BatchConfig(max_batch=4, buffer_threshold=2, position_limit=16384, pool_pages=4 * 16384,
                      max_queue=64, check_masks=False, max_output_tokens=140_000)
    prompt = "a" * 12000
    t0 = time.time()
    rows, meta = run_bench_scenario("c4_slice", deep, [prompt] * 4, cfg, 16384, every=16)
    meta["prompts"] = ["a*12000"] * 4
    meta["docs"] = list(range(4))
    print("c4_slice", rows.shape, f"{time.time() - t0:.0f}s")
    arrays["c4_slice"] = rows
    metas.append(meta)
    np.savez_compressed(OUT / "bench_runs.npz", **arrays)
    dump("bench_runs.json.gz", {"columns": BENCH_COLS, "scenarios": metas})


def gen_masks():
    """tracker.py allowed_mask at every position of documents, plus Rejected
    messages: the C++ grammar tracker (csrc/grammar.cpp) must reproduce them.
    Documents: 40 event-golden streams (depth limit 16, their tools) and
    random mask walks (traces.random_mask_walk) under tools/no tools and depth
    limits 16/2/1."""
    import random
    from threadrun.tracker import Rejected
    from threadrun.traces import random_mask_walk
    with gzip.open(OUT / "events.json.gz", "rt") as f:
        ev = json.load(f)
    docs = []
    for r in ev[:40]:
        docs.append({"tools": r["tool_names"], "depth": 16, "stream": r["stream"]})
    for seed in range(72):
        # unusual tool names (multi-byte UTF-8, shared prefixes) in the last 12 walks
        tools = (["search", "search_web", "calc2", "s"] if seed >= 60 else
                 ([] if seed % 3 == 0 else ["search", "calc"]))
        depth = (16, 2, 1)[seed % 3 if seed % 5 else 0]
        g = ThreadGrammar([ToolSpec(n) for n in tools], depth, TOK)
        docs.append({"tools": tools, "depth": depth,
                     "stream": random_mask_walk(g.tracker(), TOK, seed, budget=60 + 5 * seed)})
    distinct: dict = {}
    V = TOK.vocab_size
    rng = random.Random(0)
    for d in docs:
        g = ThreadGrammar([ToolSpec(n) for n in d["tools"]], d["depth"], TOK)
        tr = g.tracker()
        idx, rejects = [], []
        for pos, tid in enumerate(d["stream"] + [None]):
            m = tr.allowed_mask()
            bits = np.zeros(V, dtype=np.uint8)
            bits[list(m.ids)] = 1
            key = np.packbits(bits, bitorder="little").tobytes().hex()
            idx.append(distinct.setdefault(key, len(distinct)))
            if pos % 7 == 0:
                # a few inadmissible tokens: the exception text (byte index + context)
                bad = [t for t in range(V) if not m.admits(t)]
                for t in rng.sample(bad, min(3, len(bad))):
                    probe = tr.deep_copy()
                    try:
                        probe.feed(t)
                        rejects.append([pos, t, None])
                    except Rejected as e:
                        rejects.append([pos, t, str(e)])
            if tid is not None:
                tr.feed(tid)
        d["mask_idx"] = idx
        d["rejects"] = rejects
    dump("masks.json.gz", {"vocab": V, "masks": list(distinct), "docs": docs})


SCRIPTED: dict = {}


def gen_unscripted():
    """Unscripted (grammar-masked greedy) runs of the reference Engine +
    TinyTransformer (fp32, reference weights): per step the report, every
    request's page-table / live-list CRC and the free-list CRC; per request the
    token stream, status and result.  Requests hit their max_output_tokens at
    different steps, so each TokenLimit failure frees pages between two other
    requests' allocations (scheduler.py:304-316, 536-548)."""
    scens = []
    # seed 5 mixes scripted requests (deep(3,2): subtask lists close, prunes
    # and re-encodes at T=1) with unscripted ones in the same steps
    SCRIPTED.clear()
    SCRIPTED[5] = {0: make_trace(deep_recursion_tree(3, 2, seed=0), TOK).script,
                   2: make_trace(deep_recursion_tree(3, 2, seed=3), TOK).script}
    for seed, prompts, tools, limits, T in [
            (3, ["task:", "q:", "x"], [[], ["search"], []], [60, 200, 130], 1),
            (0, ["task:"], [[]], [150], 0),
            (1, ["a:", "b:", "c:", "d:"], [[], [], ["calc", "search"], []], [45, 90, 120, 75], 2),
            (5, ["p:", "u1:", "s:", "u2:"], [[], [], [], []], [400, 70, 400, 110], 1)]:
        m = TinyTransformer(ModelConfig(layers=2, heads=4, head_dim=32, vocab=512, position_limit=512,
                                        seed=seed))
        e = Engine(m, BatchConfig(max_batch=len(prompts), buffer_threshold=T, position_limit=512,
                                  pool_pages=2048, max_output_tokens=400))
        scripts = SCRIPTED.get(seed, {})
        rids = [e.submit(p, [ToolSpec(n) for n in tl], max_output_tokens=lim, script=scripts.get(i))
                for i, (p, tl, lim) in enumerate(zip(prompts, tools, limits))]
        steps = []
        while not e.all_terminal():
            rep = e.step()
            steps.append([rep.step, rep.active, rep.finished, rep.failed, rep.pages_free, rep.flops_units,
                          [crc(e.requests[r].table.pages) for r in rids],
                          [crc(e.requests[r].live) for r in rids], crc(e.pool.free_list)])
        scens.append({"seed": seed, "prompts": prompts, "tools": tools, "limits": limits, "threshold": T,
                      "scripts": {str(k): v for k, v in scripts.items()},
                      "rids": rids, "steps": steps,
                      "requests": {r: {"logical": e.requests[r].logical, "status": e.requests[r].status.value,
                                       "result": e.result(r), "evictions": [[s.start, s.end] for s in
                                                                            e.requests[r].eviction_log]}
                                   for r in rids}})
    dump("unscripted_runs.json.gz", scens)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tokenizer", "events", "engine", "model", "corpus"]
    for w in which:
        globals()[f"gen_{w}"]()
        print("generated", w)
