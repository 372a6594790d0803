"""N>1 host path on CPU (gloo, world_size 2): request sharding is a partition
of the corpus with no data-path collective, and the bench's reduction takes
the max time / summed tokens over ranks.  Each rank also replays its shard
through the reference-exact oracle accounting engine and checks that the
shards' page accounting is independent (every request finishes, pools drain)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import engine as oe
    from paper_2507_16784_b200.grammar import Grammar
    from paper_2507_16784_b200.tokenizer import build_tokenizer
    from paper_2507_16784_b200.traces import make_trace_from_text
    from paper_2507_16784_b200.traces import load_corpus
    per = 4
    corpus = load_corpus(bench.ROOT / "tests" / "golden" / "corpus_tool_chain32.json.gz")
    idx = bench.shard_docs(rank, world, per)          # round-robin: document i -> rank i % world
    assert idx == [i for i in range(per * world) if i % world == rank]
    docs = [corpus[i] for i in idx]
    tok = build_tokenizer()
    eng = oe.Engine(oe.Accounting(4096), max_batch=per, threshold=2, position_limit=4096,
                    pool_pages=per * 1600, tokenize=tok.tokenize)
    for i, d in enumerate(docs):
        t = make_trace_from_text(d)
        sc = Grammar(t.tool_names, 16, tok).tracker()
        evs, stream, call = {}, [], 0
        for tid in t.script:
            for e in sc.feed(tid):
                evs.setdefault(len(stream), []).append((e.kind, e.payload))
            stream.append(tid)
            if any(k == "ToolResultSlotOpened" for k, _ in evs.get(len(stream) - 1, [])):
                import json
                for r in tok.tokenize(json.dumps(t.tool_responses[call], separators=(",", ":"))):
                    for e in sc.feed(r):
                        evs.setdefault(len(stream), []).append((e.kind, e.payload))
                    stream.append(r)
                call += 1
        eng.submit(tok.tokenize(f"q{idx[i]}:"), t.script, t.tool_responses, evs)
    steps = tokens = 0
    while not eng.all_terminal():
        rep = eng.step()
        tokens += sum(rep["decoded"].values())
        steps += 1
    assert all(r["status"] == "finished" for r in eng.results.values())
    assert eng.pool.free_count == eng.pool.capacity
    t_max, t_max2, c_sum, c_sum2 = bench.reduce_over_ranks(dist, [float(steps), 1.0 + rank],
                                                           [float(tokens), 1.0])
    gathered = [None] * world
    dist.all_gather_object(gathered, [hash(d) for d in docs])
    if rank == 0:
        out.put((t_max, t_max2, c_sum, c_sum2, gathered, tokens))
    dist.destroy_process_group()


def test_two_rank_sharding_and_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t_max, t_max2, c_sum, c_sum2, gathered, tok0 = res
    assert t_max2 == 2.0 and c_sum2 == 2.0          # max over ranks / sum over ranks
    assert c_sum > tok0 > 0                           # both shards contributed tokens
    assert not set(gathered[0]) & set(gathered[1])    # shards are disjoint
