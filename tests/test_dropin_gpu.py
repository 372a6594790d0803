"""Drop-in proof: the REFERENCE's own Engine (threadrun.scheduler.Engine,
scheduler.py:187-608) driving B200Transformer over the device page pool.

The reference package is installed unmodified into baseline/_ref (DESIGN.md §7:
`pip install --no-index --no-deps --target baseline/_ref <copy of
/root/reference/pkg>`); it travels to the GPU box with the repo snapshot.  Each
scenario runs twice in the same process -- the reference Engine with the
reference TinyTransformer (numpy, fp32) and the reference Engine with
B200Transformer(weight_init="reference") -- and must agree on:

* every step's page table, live list and pending list (bit-exact; the device
  pool's LIFO free stack reproduces paging.py:40-67 through the per-call API);
* eviction logs, applied spans, metrics and the final text;
* every step's last-position logits within 1e-5 relative (verify.py:116-117);
* unscripted (grammar-masked greedy, the reference's own sample() on our
  logits): the same token stream, or a divergence only at a logit near-tie.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2507_16784_b200 as tr

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module")
def threadrun():
    if not (REF / "threadrun").is_dir():
        pytest.skip("reference not installed in baseline/_ref (see DESIGN.md §7)")
    sys.path.insert(0, str(REF))
    import threadrun  # noqa: F401
    from threadrun import model as rm, scheduler as rs, schema, tokenizer, traces

    def script(seed):
        tree = schema.deep_recursion_tree(3, 2, seed=seed)
        return traces.make_trace(tree, tokenizer.build_tokenizer()).script
    return rm, rs, script


def _cfg_pair(rm, **kw):
    ref = rm.ModelConfig(**kw)
    ours = tr.ModelConfig(**kw, weight_init="reference")
    return ref, ours


def _run(rs, backend, prompts, scripts, threshold, pool_pages, max_batch, max_output=None):
    """Step a reference Engine to completion, recording per-step state."""
    eng = rs.Engine(backend, rs.BatchConfig(max_batch=max_batch, buffer_threshold=threshold,
                                            position_limit=backend.position_limit,
                                            pool_pages=pool_pages,
                                            max_output_tokens=max_output or 8192))
    rids = [eng.submit(p, script=s) for p, s in zip(prompts, scripts)]
    steps = []
    while not eng.all_terminal():
        eng.step()
        rec = {}
        for rid in rids:
            r = eng.requests[rid]
            lg = None if r.last_logits is None else np.asarray(r.last_logits, dtype=np.float64)
            rec[rid] = (list(r.table.pages), list(r.live), list(r.pending), lg)
        steps.append(rec)
        assert len(steps) < 20000
    return eng, rids, steps


def _compare(ref_run, our_run, logit_tol=1e-5):
    (re_, rids, rsteps), (oe, orids, osteps) = ref_run, our_run
    assert rids == orids
    assert len(rsteps) == len(osteps)
    worst = 0.0
    for a, b in zip(rsteps, osteps):
        for rid in rids:
            pa, la, qa, ga = a[rid]
            pb, lb, qb, gb = b[rid]
            assert pa == pb and la == lb and qa == qb
            if ga is not None:
                rel = np.abs(ga - gb).max() / np.abs(ga).max()
                assert rel <= logit_tol, rel
                worst = max(worst, rel)
    for rid in rids:
        ra, rb = re_.requests[rid], oe.requests[rid]
        assert ra.eviction_log == rb.eviction_log
        assert ra.applied_spans == rb.applied_spans
        assert re_.result(rid) == oe.result(rid)
    assert re_.pool.free_count == oe.pool.free_count == oe.pool.capacity
    return worst


@pytest.mark.parametrize("threshold", [0, 1, 2])
def test_reference_engine_drives_b200_backend(threadrun, threshold):
    rm, rs, script = threadrun
    ref_cfg, our_cfg = _cfg_pair(rm, layers=2, heads=4, head_dim=32, vocab=512, position_limit=512)
    scripts = [script(0), script(1)]
    prompts = ["p:", "q:"]
    ref_run = _run(rs, rm.TinyTransformer(ref_cfg), prompts, scripts, threshold, 1024, 2)
    our_run = _run(rs, tr.B200Transformer(our_cfg), prompts, scripts, threshold, 1024, 2)
    worst = _compare(ref_run, our_run)
    assert worst < 1e-5


def test_reference_engine_unscripted_masked_greedy(threadrun):
    """No script: the reference Engine computes its grammar masks and calls its
    own sample(logits, mask) on OUR logits.  Greedy streams must agree unless
    the reference's top-2 admitted logits are within fp32 noise."""
    rm, rs, _ = threadrun
    ref_cfg, our_cfg = _cfg_pair(rm, layers=2, heads=4, head_dim=32, vocab=512, position_limit=256)
    ref_run = _run(rs, rm.TinyTransformer(ref_cfg), ["task:"], [None], 1, 512, 1, max_output=120)
    our_run = _run(rs, tr.B200Transformer(our_cfg), ["task:"], [None], 1, 512, 1, max_output=120)
    (re_, rids, rsteps), (oe, _, osteps) = ref_run, our_run
    a = re_.requests[rids[0]].logical
    b = oe.requests[rids[0]].logical
    n = min(len(a), len(b))
    div = next((i for i in range(n) if a[i] != b[i]), None)
    if div is None:
        assert len(a) == len(b)
        assert re_.result(rids[0]) == oe.result(rids[0])
        _compare(ref_run, our_run)
    else:
        # a divergence is only legal at a near-tie of the reference's logits
        step = div - len(re_.requests[rids[0]].prompt_tokens)
        lg = rsteps[max(step - 1, 0)][rids[0]][3]
        top = np.sort(lg)[-2:]
        assert top[1] - top[0] <= 1e-5 * np.abs(lg).max(), (div, top)
