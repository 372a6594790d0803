"""Unscripted decoding: grammar-masked greedy picks on the
device must reproduce the REFERENCE Engine + TinyTransformer run bit-exactly.

tests/golden/unscripted_runs.json.gz (oracle/gen_golden.py gen_unscripted) holds
four reference runs (fp32, reference weights, T = 1 / 0 / 2 / 1, tools and no
tools; the fourth mixes two scripted deep(3,2) requests -- subtask lists
close, prune, re-encode and finish -- with two unscripted ones in the same
steps).  Each request samples under the tracker's admissible-token mask
(scheduler.py:413-442, model.py:186-192) until its own max_output_tokens, so
the TokenLimit failures land on different steps and free their pages between
other requests' allocations.  The B200 Engine (native grammar tracker, masks
in a device table, tim_masked_argmax after the batched forward, the step split
at picks that may free pages) must match every step's report, every request's
page-table and live-list CRC and the free-list CRC, and the final token
streams and results.
"""

import gzip
import json
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2507_16784_b200 as tr

pytestmark = pytest.mark.gpu


def crc(ids):
    return zlib.crc32(np.asarray(ids, dtype=np.int32).tobytes())


def _scenarios(golden):
    with gzip.open(golden / "unscripted_runs.json.gz", "rt", encoding="utf-8") as f:
        return json.load(f)


@pytest.mark.parametrize("which", [0, 1, 2, 3])
def test_unscripted_masked_greedy_matches_reference(golden, which):
    sc = _scenarios(golden)[which]
    cfg = tr.ModelConfig(layers=2, heads=4, head_dim=32, vocab=512, position_limit=512, seed=sc["seed"])
    eng = tr.Engine(tr.B200Transformer(cfg),
                    tr.BatchConfig(max_batch=len(sc["prompts"]), buffer_threshold=sc["threshold"],
                                   position_limit=512, pool_pages=2048, max_output_tokens=400,
                                   check_device=True))
    scripts = {int(k): v for k, v in sc.get("scripts", {}).items()}
    rids = [eng.submit(p, [tr.ToolSpec(n) for n in tl], max_output_tokens=lim, script=scripts.get(i))
            for i, (p, tl, lim) in enumerate(zip(sc["prompts"], sc["tools"], sc["limits"]))]
    assert rids == sc["rids"]
    for g in sc["steps"]:
        rep = eng.step()
        mine = [rep.step, rep.active, rep.finished, rep.failed, rep.pages_free, rep.flops_units,
                [crc(eng.requests[r].table.pages) for r in rids],
                [crc(eng.requests[r].live) for r in rids], crc(eng.pool.free_list)]
        assert mine == g, (rep.step, mine, g)
    assert eng.all_terminal()
    for r in rids:
        want = sc["requests"][r]
        assert eng.requests[r].logical == want["logical"], r
        assert eng.requests[r].status.value == want["status"]
        assert eng.result(r) == want["result"]
        assert [[x.start, x.end] for x in eng.requests[r].eviction_log] == want["evictions"]
    assert eng.pool.free_count == eng.pool.capacity


def test_masked_argmax_kernel_matches_numpy():
    """tim_masked_argmax == np.argmax(np.where(mask, logits, -inf)) (model.py:186-192),
    lowest id on ties, -1 for an empty mask, -1 ids = unmasked rows."""
    from paper_2507_16784_b200 import _lib as L
    rng = np.random.default_rng(0)
    V, R, W = 512, 37, 16
    logits = rng.standard_normal((R, V)).astype(np.float32)
    logits[3, 10] = logits[3, 200] = 50.0            # tie -> lowest admitted id
    masks = rng.integers(0, 2**32, size=(8, W), dtype=np.uint64).astype(np.uint32)
    masks[5] = 0                                      # empty
    masks[6] = 0
    masks[6, 6] = 1 << 8                              # only id 200
    mids = rng.integers(-1, 8, size=R).astype(np.int32)
    mids[3] = 7
    masks[7] = 0xFFFFFFFF
    mids[4] = 5
    mids[9] = 6
    d_logits = torch.from_numpy(logits).cuda()
    d_masks = torch.from_numpy(masks.view(np.int32)).cuda()
    d_mids = torch.from_numpy(mids).cuda()
    out = torch.empty(R, dtype=torch.int32, device="cuda")
    L.call("tim_masked_argmax", d_logits.data_ptr(), R, V, d_mids.data_ptr(), d_masks.data_ptr(), W,
           out.data_ptr(), L.DTYPE_F32, torch.cuda.current_stream().cuda_stream)
    got = out.cpu().numpy()
    for r in range(R):
        if mids[r] < 0:
            want = int(np.argmax(logits[r]))
        else:
            bits = np.unpackbits(masks[mids[r]].view(np.uint8), bitorder="little")[:V].astype(bool)
            want = int(np.argmax(np.where(bits, logits[r], -np.inf))) if bits.any() else -1
        assert got[r] == want, (r, got[r], want)
    assert got[3] == 10 and got[4] == -1 and got[9] == 200
