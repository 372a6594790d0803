"""Benchmark: decode tokens/s with subtask pruning on B200 (BASELINE.json metric).

Workload (N=1 line = BASELINE config 2, C2): Qwen3-8B-shaped TIM decoder
(36 layers, hidden 4096, GQA 32q/8kv, head_dim 128, MLP 12288, vocab 512,
bf16, random init) running 64 scripted TIM trajectories per GPU to completion
-- the reference's own tool_chain_tree(32, seed=i) documents (tests/golden
corpus) -- with pruning buffer T=2.  Under torchrun (or `--gpus N`, which
re-executes itself under torchrun) the 64*N documents are dealt round-robin,
document i to rank i % N (BASELINE config 3 at N=8), weak scaling, no
collective on the data path.

A "step" is one Engine.step() over the batch: host planning, K4/K5 device
paging, and one batched forward of all requests' new tokens through every
layer (decode rows + re-encode/tool rows).  The whole trajectory (~4.4K steps)
runs; K steps sampled at a fixed stride over it (after W warm-up steps) are
timed, so the timed steps carry the trajectory's own mix of decode-only and
pruning / tool-response steps whatever K is:
  value : the trajectory replayed from device-resident step descriptors (host
          planning done beforehand); CUDA events bracket each timed step.
  e2e   : a fresh engine runs the whole trajectory through the public
          Engine.step(); every step after the W warm-up steps is timed as one
          contiguous window (host planning + pinned H2D of each step
          descriptor + device work + async D2H of each step's greedy tokens),
          synchronised at both ends -- what a caller of the API sees.
Tokens = tokens encoded for the first time (generated + tool tokens), the
reference's output_len accounting (cli.py:130-134, scheduler.py:374-377).
Both runs are checked against the REFERENCE Engine's per-step checksums of
block tables, live lists and free list (tests/golden/bench_runs.*) and the
device error word; a mismatch aborts the run.

`--impl reference` times the reference's CPU implementation of the path (the
numpy oracle restatement of model.py -- the Python reference cannot travel to
the GPU box) on the reference's own recorded per-step work of the same timed
steps, with every host thread BLAS can use.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode tokens/s with pruning at 1/2/4/8 B200; attention HBM GB/s vs peak"
UNIT = "tokens/s"
PER_GPU = 64


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self) -> dict:
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


def local_device() -> int:
    """This rank's GPU: LOCAL_RANK (modulo the visible devices, so a smoke
    test can run several ranks on one GPU)."""
    import torch
    return int(os.environ.get("LOCAL_RANK", 0)) % max(torch.cuda.device_count(), 1)


def reduce_over_ranks(dist, times, counts, device="cpu"):
    """Times: max over ranks (the job ends with its slowest rank); counts: sum."""
    import torch
    if dist is None:
        return (*times, *counts)
    t = torch.tensor(times, dtype=torch.float64, device=device)
    c = torch.tensor(counts, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return (*[float(x) for x in t], *[float(x) for x in c])


# --------------------------------------------------------------------- GPU arm
def shard_docs(rank: int, world: int, per_gpu: int = PER_GPU) -> list[int]:
    """BASELINE config 3: the 512 (= 64 x G) documents dealt round-robin,
    document i to GPU i % G; G = 1 is config 2's 64."""
    return [i for i in range(per_gpu * world) if i % world == rank]


def build_engine(rank: int, n_req: int, threshold: int, pool_per_req: int = 1600, world: int = 1,
                 model=None):
    import paper_2507_16784_b200 as tr
    from paper_2507_16784_b200.traces import load_corpus, make_trace_from_text
    cfg = tr.qwen3_8b_shape()
    model = model or tr.B200Transformer(cfg)
    docs = load_corpus(ROOT / "tests" / "golden" / "corpus_tool_chain32.json.gz")
    idx = shard_docs(rank, world, n_req)
    eng = tr.Engine(model, tr.BatchConfig(max_batch=n_req, buffer_threshold=threshold,
                                          position_limit=cfg.position_limit,
                                          pool_pages=n_req * pool_per_req,
                                          max_queue=max(64, n_req), check_masks=False,
                                          max_output_tokens=20000))
    for i in idx:
        t = make_trace_from_text(docs[i % len(docs)])
        eng.submit(f"q{i}:", [tr.ToolSpec(n) for n in t.tool_names], script=t.script,
                   tool_responses=t.tool_responses)
    return eng, cfg, model


def golden_rows(rank: int, world: int, threshold: int, n_req: int):
    """The reference Engine's per-step checksums for this shard, when
    tests/golden holds them (oracle/gen_golden.py gen_bench)."""
    import gzip
    import numpy as np
    if threshold != 2 or n_req != PER_GPU:
        return None
    name = f"c2_g1_r0" if world == 1 else f"c3_g{world}_r{rank}"
    meta_p = ROOT / "tests" / "golden" / "bench_runs.json.gz"
    if not meta_p.exists():
        return None
    with gzip.open(meta_p, "rt") as f:
        names = [s["name"] for s in json.load(f)["scenarios"]]
    if name not in names:
        return None
    rows = np.load(ROOT / "tests" / "golden" / "bench_runs.npz")[name]
    return name, {int(r[0]): [int(x) for x in r] for r in rows}


def sampled_steps(n_steps: int, k: int, warmup: int) -> list[int]:
    """K step indices at a fixed stride over the whole trajectory after the
    W warm-up steps, so the timed steps carry the trajectory's own mix of
    decode-only and mixed (prune re-encode / tool response) steps whatever K is."""
    lo = min(warmup, n_steps - 1)
    span = n_steps - lo
    if k >= span:
        return list(range(lo, n_steps))
    return sorted({lo + (j * span) // k + (span // k) // 2 for j in range(k)})


def run_gpu(args, rank: int, world: int, dist):
    """value and e2e over the SAME K steps of the trajectories (sampled at a
    stride over the whole run, every step before and between them executed
    untimed).  value: engine A plans the whole trajectory on the host, then
    replays it from device-resident step descriptors; CUDA events bracket the
    K sampled steps.  e2e: a fresh engine B on the same requests runs every
    step through the public Engine.step(); each sampled step is timed from
    the call to the D2H read of its greedy tokens (host planning, pinned H2D of
    the step descriptor, device work, D2H), synchronised on both sides."""
    import torch
    from paper_2507_16784_b200.checksum import device_hashes, host_hash, seq_hash_np
    torch.cuda.set_device(local_device())
    gold = golden_rows(rank, world, args.threshold, args.batch)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------------------------------------------------------- value
    eng, cfg, model = build_engine(rank, args.batch, args.threshold, world=world)
    rt = eng.runtime
    t0 = time.perf_counter()
    rt.precapture()
    print(f"[rank {rank}] captured {len(rt.graphs)} step graphs in {time.perf_counter() - t0:.1f} s",
          file=sys.stderr)
    rt.recording = []
    step_tokens, step_free = [], []
    while not eng.all_terminal():
        rep = eng.step()
        step_tokens.append(sum(rep.decoded.values()))
        step_free.append(rep.pages_free)
    records, rt.recording = rt.recording, None
    n_steps = len(step_tokens)
    assert len(records) == n_steps, (len(records), n_steps)
    # every rank times the same step indices of its own shard
    if dist is not None:
        t = torch.tensor([n_steps], device="cuda" if os.environ.get("TIMRUN_DIST_BACKEND", "nccl") == "nccl"
                         else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        n_steps_common = int(t.item())
    else:
        n_steps_common = n_steps
    timed = sampled_steps(n_steps_common, args.steps, args.warmup)
    timed_set = set(timed)
    resident = rt.replay_upload(records)
    checkpoints = {timed[len(timed) * q // 4] for q in (1, 2, 3)} if gold else set()
    kv_tok_layer = cfg.n_kv * cfg.head_dim * 2 * 2          # K+V bytes per token per layer (bf16)
    q_o_bytes = cfg.heads * cfg.head_dim * 2 * 2            # q in + ctx out per query row
    attn_store, step_ev = [], []
    launches0 = rt.launches
    launches_timed = 0
    clocks = ClockSampler(local_device())
    clocks.start()
    barrier()
    # TIMRUN_PROFILE_TIMED=1 brackets each timed step with cudaProfilerStart/Stop
    # (ncu --profile-from-start off then captures exactly the value window)
    prof = os.environ.get("TIMRUN_PROFILE_TIMED") == "1"
    for i, (sd, step, fw) in enumerate(resident):
        if i in timed_set:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            rt.attn_events = attn_store
            l0 = rt.launches
            if prof:
                torch.cuda.cudart().cudaProfilerStart()
            a.record()
            rt._execute(sd, step, fw)
            b.record()
            if prof:
                torch.cuda.cudart().cudaProfilerStop()
            rt.attn_events = None
            launches_timed += rt.launches - l0
            step_ev.append((a, b, i))
        else:
            rt._execute(sd, step, fw)
        if i in checkpoints:
            # step i+1 of the reference run: free stack vs the reference free list
            torch.cuda.synchronize()
            g = gold[1].get(i + 1)
            sp = step_free[i]
            ii = torch.arange(sp, dtype=torch.int64, device="cuda")
            from paper_2507_16784_b200.checksum import weights_torch
            fh = int(((eng.pool.free_stack[:sp].long() + 1) * weights_torch(ii)).sum()) if sp else 0
            if g is not None and [sp, fh] != [g[5], g[10]]:
                raise SystemExit(f"[rank {rank}] value run: free stack diverged from the reference at step {i + 1}")
    barrier()
    clk = clocks.stop()
    rt.check()                                              # device error word of the whole run
    ms = sum(a.elapsed_time(b) for a, b, _ in step_ev)
    tokens = sum(step_tokens[i] for i in timed)
    mixed_steps = sum(1 for i in timed if records[i][0].ext)
    rows = sorted(records[i][0].n_rows for i in timed)
    all_rows = [sd.n_rows for sd, _, _ in records]
    mean_live = (sum(sum(sg[1] for sg in sd.segs) / max(len(sd.segs), 1) for sd, _, _ in records if sd.segs)
                 / max(1, sum(1 for sd, _, _ in records if sd.segs)))
    # Fixed cost of bracketing ONE launch with CUDA events (an empty grid of the
    # attention kernel's shape, launched the same way): reported beside the
    # roofline so the per-launch figure can be read net of it.
    from paper_2507_16784_b200 import _lib as L
    floor = []
    L.call("tim_noop", rt.sms, 288, 230000, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    torch.cuda._sleep(4_000_000)
    for _ in range(60):
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        L.call("tim_noop", rt.sms, 288, 230000, torch.cuda.current_stream().cuda_stream)
        b_.record()
        floor.append((a_, b_))
    torch.cuda.synchronize()
    floor_ms = sorted(a_.elapsed_time(b_) for a_, b_ in floor[10:])
    floor_ms = floor_ms[len(floor_ms) // 2]
    weight_gb = model.weight_bytes() / 1e9
    # dominant kernel: the layer-0 attention launch of every timed step
    def attn_bytes(sd):
        return sum(sg[1] + sg[2] for sg in sd.segs) * kv_tok_layer + sd.n_rows * q_o_bytes
    attn = [(a.elapsed_time(b), sd) for a, b, sd in attn_store]
    dec = [(t, sd) for t, sd in attn if not sd.ext]
    mix = [(t, sd) for t, sd in attn if sd.ext]

    def agg(lst):
        if not lst:
            return {"achieved": None, "bytes_per_launch": 0.0, "ms_per_launch": 0.0, "launches": 0}
        tm = sum(t for t, _ in lst) / len(lst)
        by = sum(attn_bytes(sd) for _, sd in lst) / len(lst)
        return {"achieved": by / (tm * 1e-3) / 1e9, "bytes_per_launch": by, "ms_per_launch": tm,
                "launches": len(lst)}
    del resident, records
    # ------------------------------------------------------------------ e2e
    eng2, _, _ = build_engine(rank, args.batch, args.threshold, world=world, model=model)
    del eng, rt
    torch.cuda.empty_cache()
    rt2 = eng2.runtime
    rt2.precapture()
    # every step's greedy tokens land in one pinned buffer (async D2H per step)
    host_buf = torch.empty(n_steps * args.batch + 16, dtype=torch.int32, pin_memory=True)
    e2e_s, e2e_tokens, h2d, d2h, e2e_steps = 0.0, 0, 0, 0, 0
    host_ms = []
    verified = []
    k = 0
    while k < args.warmup and not eng2.all_terminal():
        eng2.step()
        k += 1
    barrier()
    w0 = time.perf_counter()
    off = 0
    while not eng2.all_terminal():
        th = time.perf_counter()
        rep = eng2.step()
        host_ms.append((time.perf_counter() - th) * 1e3)
        toks = eng2.last_step_tokens
        if toks is not None:
            n = toks.numel()
            host_buf[off:off + n].copy_(toks, non_blocking=True)   # D2H of the step's greedy tokens
            off += n
            d2h += n * 4
        e2e_tokens += sum(rep.decoded.values())
        h2d += rt2._last_upload_bytes
        e2e_steps += 1
        k += 1
        if gold and k in gold[1] and (k in {c + 1 for c in checkpoints} or eng2.all_terminal()):
            # reference checksum verification: clock stopped while it runs
            torch.cuda.synchronize()
            e2e_s += time.perf_counter() - w0
            pend = {rid: len(eng2.requests[rid].pending) for rid in rep.request_live}
            mine = [rep.step, rep.active, rep.awaiting_tool, rep.finished, rep.failed, rep.pages_free,
                    rep.flops_units, host_hash(rep.request_live, pend, rep.decoded), *device_hashes(eng2)]
            if mine != gold[1][k]:
                raise SystemExit(f"[rank {rank}] e2e run diverged from the reference ({gold[0]}) at step {k}")
            verified.append(k)
            w0 = time.perf_counter()
    torch.cuda.synchronize()
    e2e_s += time.perf_counter() - w0
    result_sum = int(host_buf[:off].sum())
    if dist is not None:
        dist.barrier()
    rt2.check()
    e2e_h2d, e2e_d2h = h2d / max(e2e_steps, 1), d2h / max(e2e_steps, 1)
    hs = sorted(host_ms)
    print(f"[rank {rank}] trajectory {n_steps} steps; timed {len(timed)} (stride "
          f"{(n_steps_common - args.warmup) / max(len(timed), 1):.0f}); mixed steps timed {mixed_steps}; "
          f"rows/step timed: min {rows[0]} median {rows[len(rows) // 2]} max {rows[-1]} mean "
          f"{sum(rows) / len(rows):.0f} (whole run mean {sum(all_rows) / len(all_rows):.0f})",
          file=sys.stderr)
    print(f"[rank {rank}] e2e host time inside Engine.step(): mean {sum(hs) / len(hs):.2f} ms, "
          f"median {hs[len(hs) // 2]:.2f}, max {hs[-1]:.2f}", file=sys.stderr)
    print(f"[rank {rank}] reference checksums verified at steps {verified} ({gold[0] if gold else 'no golden'})",
          file=sys.stderr)
    print(f"[rank {rank}] value: {tokens} tokens in {ms:.1f} ms; e2e: {e2e_tokens} tokens in "
          f"{e2e_s * 1e3:.1f} ms over {e2e_steps} contiguous steps (token checksum {result_sum})",
          file=sys.stderr)
    ms_max, e2e_ms_max, tok_sum, e2e_tok_sum = reduce_over_ranks(
        dist, [ms, e2e_s * 1e3], [tokens, e2e_tokens],
        device="cuda" if os.environ.get("TIMRUN_DIST_BACKEND", "nccl") == "nccl" else "cpu")
    return dict(ms=ms_max, e2e_ms=e2e_ms_max, tokens=tok_sum, e2e_tokens=e2e_tok_sum,
                n_timed=len(timed), n_steps=n_steps, mixed_timed=mixed_steps,
                attn=agg(attn), dec=agg(dec), mix=agg(mix), launches=launches_timed, clocks=clk,
                h2d=e2e_h2d, d2h=e2e_d2h, e2e_steps=e2e_steps, mean_live=mean_live,
                weight_gb=weight_gb, floor_ms=floor_ms, verified=verified,
                golden=gold[0] if gold else None, launches_total=rt2.launches)


# --------------------------------------------------------------- CPU reference
def workload_config(world: int, args) -> dict:
    """The `config` object of BOTH arms (identical, so the driver pairs them)."""
    return {"workload": f"C2/C3: Qwen3-8B-shaped TIM decoder, {args.batch} tool_chain_tree(32) requests per GPU "
                        f"(512 dealt round-robin at 8 GPUs), pruning buffer T={args.threshold}, run to completion",
            "model": "qwen3-8b-shape: 36L, d4096, 32q/8kv x128, mlp 12288, vocab 512 (random init)",
            "global_batch": args.batch * world, "seq_len": "retained working memory, mean ~640 tokens (max 1177)",
            "parallelism": f"dp{world} (requests sharded, no collective)",
            "window": f"{args.steps} engine steps at a fixed stride over the whole trajectory "
                      f"(after {args.warmup} warm-up steps); every other step runs untimed",
            "l2": "inputs larger than L2 (10.3 GB of weights + the retained KV read every step)"}


def cpu_reference(budget_s: float, steps: int, warmup: int, threshold: int, n_req: int = PER_GPU):
    """The reference's CPU algorithm for this path, timed on the host cores:
    the numpy oracle of model.py:127-164 (+ GQA) at the Qwen3-8B shape, all
    36 layers (one layer's weights shared by the 36, which leaves the work per
    forward unchanged and keeps host memory at 0.7 GB), on the REFERENCE's own
    per-step work: the (prefix m, n rows) of every forward the reference
    Engine issued in the C2 run (tests/golden bench_runs.npz c2_work, recorded
    by oracle/gen_golden.py).  The reference runs requests one after another
    (scheduler.py:304-316), so a step costs the sum of its forwards.  Within
    the budget, forwards are drawn uniformly at random from the same K timed
    steps as the GPU arm; the steps' time is estimated as (#forwards) x (mean
    sampled forward time) and tokens/s = the steps' first-encoded tokens over it.
    Also reported: the scripted (page accounting only) oracle Engine's host
    tokens/s on the same requests (SURVEY §8d leg 3)."""
    import numpy as np
    from oracle import model as om
    from oracle.paging import PageTable

    if threshold != 2 or n_req != PER_GPU:
        raise SystemExit("the CPU reference leg is defined on the C2 workload (T=2, 64 requests)")
    g = np.load(ROOT / "tests" / "golden" / "bench_runs.npz")
    work, decoded = g["c2_work"], g["c2_decoded"]
    n_steps = len(decoded)
    timed = [i + 1 for i in sampled_steps(n_steps, steps, warmup)]       # reference step numbers
    calls = work[np.isin(work[:, 0], timed)]
    tokens = int(decoded[np.asarray(timed) - 1].sum())
    cfg = om.Config(layers=36, heads=32, kv_heads=8, head_dim=128, mlp_dim=12288, vocab=512,
                    position_limit=40960, rope_base=1e6)
    rng = np.random.default_rng(0)
    sc_ = np.float32(1.0 / np.sqrt(cfg.model_dim))
    kvd = cfg.n_kv * cfg.head_dim

    def mat(*shape):
        return rng.standard_normal(shape, dtype=np.float32) * sc_
    layer = {"wq": mat(4096, 4096), "wk": mat(4096, kvd), "wv": mat(4096, kvd), "wo": mat(4096, 4096),
             "w1": mat(4096, 12288), "w2": mat(12288, 4096)}
    w = {"emb": mat(512, 4096), "inv_freq": (1e6 ** (-np.arange(64) / 64)).astype(np.float32),
         "layers": [layer] * 36}
    model = om.Model(cfg, w)
    max_pages = int((calls[:, 2] + calls[:, 3]).max()) + 1
    pool = model.make_pool(max_pages)
    pool.K[:] = rng.standard_normal(pool.K.shape, dtype=np.float32)
    pool.V[:] = rng.standard_normal(pool.V.shape, dtype=np.float32)
    order = rng.permutation(len(calls))
    times = []
    t_start = time.perf_counter()
    for j in order:
        _, _, m, n = (int(x) for x in calls[j])
        pool.free_list = list(range(max_pages - 1, m - 1, -1))
        pool.allocated = {p: "x" for p in range(m)}
        t = PageTable("x")
        t.pages = list(range(m))
        toks = [int(x) for x in rng.integers(0, 512, n)]
        c0 = time.perf_counter()
        model.forward(toks, list(range(m, m + n)), t, pool)
        times.append(time.perf_counter() - c0)
        if time.perf_counter() - t_start > budget_s:
            break
    est_s = len(calls) * float(np.mean(times))
    value = tokens / est_s
    # leg 3: the scripted reference Engine (page accounting only) on the same
    # requests -- the reference's own code when baseline/_ref is installed
    acc, acc_kind = reference_scripted_rate(min(budget_s / 3, 10.0), n_req, threshold)
    if acc is None:
        acc, acc_kind = scripted_engine_rate(min(budget_s / 3, 10.0), n_req, threshold), "port"
    import threadpoolctl
    blas = threadpoolctl.threadpool_info()
    threads = max([b.get("num_threads", 1) for b in blas] or [1])
    return {"value": value, "unit": UNIT, "cores": int(threads), "kind": "port",
            "sample": (f"{len(times)} of the {len(calls)} forwards the reference Engine issued in the "
                       f"{len(timed)} timed steps of the C2 run (tool_chain_tree(32) x 64, T=2), each a "
                       f"full 36-layer numpy forward (oracle/model.py = model.py:127-164 + GQA) at its "
                       f"recorded (prefix m, rows n); {sum(times):.1f} s measured, steps' time estimated "
                       f"as #forwards x mean = {est_s:.0f} s for {tokens} tokens; numpy {np.__version__}, "
                       f"BLAS threads {threads}, os.cpu_count {os.cpu_count()}"),
            "scripted_engine_tokens_per_s": acc, "scripted_engine_kind": acc_kind}


def reference_scripted_rate(budget_s: float, n_req: int, threshold: int):
    """SURVEY §8d leg 3 on the REFERENCE's own code: threadrun's Engine with its
    ScriptedModel (scheduler.py:274-442, model.py:195-233; page accounting and
    grammar tracking, no arithmetic) from baseline/_ref, on the C2 requests,
    for `budget_s` of host time: (tokens/s, "reference") or (None, None)."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "threadrun").is_dir():
        return None, None
    sys.path.insert(0, str(ref))
    try:
        from threadrun.model import ScriptedModel
        from threadrun.scheduler import BatchConfig, Engine
        from threadrun.schema import ToolSpec, parse_tree_text
        from threadrun.tokenizer import build_tokenizer
        from threadrun.traces import make_trace
    finally:
        sys.path.remove(str(ref))
    from paper_2507_16784_b200.traces import load_corpus
    tok = build_tokenizer()
    P = 40960
    eng = Engine(ScriptedModel(position_limit=P),
                 BatchConfig(max_batch=n_req, buffer_threshold=threshold, position_limit=P,
                             pool_pages=n_req * 1600, max_queue=max(64, n_req), check_masks=False,
                             max_output_tokens=20000))
    docs = load_corpus(ROOT / "tests" / "golden" / "corpus_tool_chain32.json.gz")
    for i in shard_docs(0, 1, n_req):
        t = make_trace(parse_tree_text(docs[i]), tok)
        eng.submit(f"q{i}:", [ToolSpec(n) for n in t.tool_names], script=t.script,
                   tool_responses=t.tool_responses or None)
    t0 = time.perf_counter()
    toks = 0
    while time.perf_counter() - t0 < budget_s and not eng.all_terminal():
        toks += sum(eng.step().decoded.values())
    return toks / (time.perf_counter() - t0), "reference"


def c1_legs() -> dict | None:
    """SURVEY §8d leg 1 in the same run: BASELINE config 1 (tiny fp32, 2
    layers x 4 heads x 32, batch 1, deep_recursion_tree(3,2), T=1) through the
    REFERENCE Engine + TinyTransformer (baseline/_ref, numpy, this host) and
    through the B200 engine (graphs captured first), same trace; tokens/s of
    each and whether their text and metrics agree."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "threadrun").is_dir():
        return None
    import torch
    import paper_2507_16784_b200 as tr
    sys.path.insert(0, str(ref))
    try:
        from threadrun import model as rm, scheduler as rs, schema, tokenizer, traces
    finally:
        sys.path.remove(str(ref))
    script = traces.make_trace(schema.deep_recursion_tree(3, 2, seed=0), tokenizer.build_tokenizer()).script
    kw = dict(layers=2, heads=4, head_dim=32, vocab=512, position_limit=2048)
    best = None
    for _ in range(3):
        e = rs.Engine(rm.TinyTransformer(rm.ModelConfig(**kw)),
                      rs.BatchConfig(buffer_threshold=1, position_limit=2048, pool_pages=4096))
        rid = e.submit("p:", script=script)
        t0 = time.perf_counter()
        e.run_until_done()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        rres = e.result(rid)
    mine = None
    for _ in range(3):                   # best of 3 (the first pass also warms allocator / cuBLAS)
        eng = tr.Engine(tr.B200Transformer(tr.ModelConfig(**kw)),
                        tr.BatchConfig(buffer_threshold=1, position_limit=2048, pool_pages=4096))
        eng.runtime.precapture()
        rid2 = eng.submit("p:", script=script)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        while not eng.all_terminal():
            eng.step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        mine = dt if mine is None else min(mine, dt)
    res = eng.result(rid2)
    n = rres["metrics"]["output_len"]
    return {"workload": "C1 tiny fp32 (2 layers, 4 heads x 32), batch 1, deep_recursion_tree(3,2), T=1",
            "reference_tokens_per_s": n / best, "reference_kind": "reference (threadrun from baseline/_ref)",
            "b200_tokens_per_s": res["metrics"]["output_len"] / mine,
            "identical_text_and_metrics": rres["text"] == res["text"] and rres["metrics"] == res["metrics"]}


def scripted_engine_rate(budget_s: float, n_req: int, threshold: int) -> float:
    """SURVEY §8d leg 3: the oracle's reference-order scripted Engine (page
    accounting, no arithmetic) on the C2 requests: host tokens/s."""
    from oracle import engine as oe
    from paper_2507_16784_b200.grammar import Grammar
    from paper_2507_16784_b200.tokenizer import build_tokenizer
    from paper_2507_16784_b200.traces import load_corpus, make_trace_from_text
    tok = build_tokenizer()
    P = 40960
    eng = oe.Engine(oe.Accounting(P), max_batch=n_req, threshold=threshold, position_limit=P,
                    pool_pages=n_req * 1600, max_queue=max(64, n_req), tokenize=tok.tokenize)
    docs = load_corpus(ROOT / "tests" / "golden" / "corpus_tool_chain32.json.gz")
    for i in shard_docs(0, 1, n_req):
        t = make_trace_from_text(docs[i])
        sc, evs, stream, call = Grammar(t.tool_names, 16, tok).tracker(), [], [], 0
        for tid in t.script:
            for e in sc.feed(tid):
                evs.append([e.kind, len(stream), e.depth, e.payload])
            stream.append(tid)
            if evs and evs[-1][0] == "ToolResultSlotOpened" and evs[-1][1] == len(stream) - 1:
                text = json.dumps(t.tool_responses[call], separators=(",", ":"), ensure_ascii=False)
                for rt_ in tok.tokenize(text):
                    for e in sc.feed(rt_):
                        evs.append([e.kind, len(stream), e.depth, e.payload])
                    stream.append(rt_)
                call += 1
        eng.submit(tok.tokenize(f"q{i}:"), t.script, t.tool_responses, oe.event_table(evs))
    t0 = time.perf_counter()
    toks = 0
    while time.perf_counter() - t0 < budget_s and not eng.all_terminal():
        toks += sum(eng.step()["decoded"].values())
    return toks / (time.perf_counter() - t0)


def respawn_under_torchrun(n: int) -> None:
    """`python bench.py --gpus N` outside torchrun: re-exec as N ranks (one per GPU)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=PER_GPU)
    ap.add_argument("--threshold", type=int, default=2)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        respawn_under_torchrun(args.gpus)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    config = workload_config(world, args)
    if args.impl == "reference":
        if rank != 0:
            return
        cb = cpu_reference(args.cpu_budget, args.steps, args.warmup, args.threshold, args.batch)
        line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic: reference tool_chain_tree(32) documents replayed as scripts; random-init weights",
                "impl": "reference", "config": config, "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_mod
        local = local_device()
        torch.cuda.set_device(local)
        # NCCL for the barrier and the max/sum reductions (no collective on the
        # data path); TIMRUN_DIST_BACKEND=gloo lets several ranks share one GPU
        # (a smoke test of the N>1 path on a single-GPU box)
        backend = os.environ.get("TIMRUN_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist_mod.init_process_group(backend)
        dist = dist_mod
    res = run_gpu(args, rank, world, dist)
    if rank == 0:
        pk = peaks()
        a = res["attn"]
        tr_path = ROOT / "profiles" / "attention_traffic.json"
        traffic = json.loads(tr_path.read_text()) if tr_path.exists() else None
        cpu = None
        if world == 1 and args.cpu_budget > 0:
            # C1 first: the numpy legs leave BLAS worker threads spinning on the
            # host cores, which slows the B200 engine's host-bound C1 loop
            c1 = c1_legs()
            cpu = cpu_reference(args.cpu_budget, args.steps, args.warmup, args.threshold, args.batch)
            cpu["c1_leg"] = c1
        value = res["tokens"] / (res["ms"] * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms"] / res["n_timed"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: reference tool_chain_tree(32) documents replayed as scripts; random-init weights",
            "config": config,
            "roofline": {"bound": "hbm", "kernel": "tim_attn_decode: decode tiles (K1) + tcgen05 items (K2), "
                                                    "layer 0 of every timed step",
                         "achieved": a["achieved"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": (a["achieved"] or 0.0) / pk["hbm_gbs"],
                         "traffic": traffic["bytes_per_launch"] if traffic else None,
                         "traffic_src": traffic["source"] if traffic else None,
                         "peak_src": pk["src"],
                         "bytes_per_launch": a["bytes_per_launch"], "ms_per_launch": a["ms_per_launch"],
                         "launches_timed": a["launches"],
                         "event_floor_us": res["floor_ms"] * 1e3,
                         "achieved_net_of_event_floor": a["bytes_per_launch"] / ((a["ms_per_launch"] - res["floor_ms"]) * 1e-3) / 1e9
                         if a["launches"] else None,
                         "decode_only_steps": res["dec"], "mixed_steps": res["mix"]},
            "cpu_baseline": cpu,
            "e2e": {"value": res["e2e_tokens"] / (res["e2e_ms"] * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"],
                    "window": f"all {res['e2e_steps']} steps after the {args.warmup} warm-up steps, contiguous "
                              "through Engine.step() (host planning + pinned H2D descriptor + device step + "
                              "async D2H of every step's tokens), synchronised at both ends"},
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
            "trajectory": {"steps": res["n_steps"], "timed_steps": res["n_timed"],
                           "mixed_steps_timed": res["mixed_timed"], "mean_retained": res["mean_live"],
                           "reference_checksums": res["golden"], "verified_at_steps": res["verified"]},
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
