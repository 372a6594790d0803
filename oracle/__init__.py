"""CPU oracle for the TIMRUN working-memory decode path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy / Python, the reference algorithms of
`threadrun` (/root/reference/pkg/src/threadrun) that the B200 path replaces:

* paging.py   — LIFO page pool, page tables, gather          (ref paging.py:27-127)
* pruning.py  — FIFO prune buffer, coalesce, apply, metric   (ref pruning.py:29-168)
* model.py    — seeded rotary transformer (+ GQA fields)     (ref model.py:39-192)
* engine.py   — continuous-batching scripted step loop       (ref scheduler.py:132-581)

Each function cites the reference file:line it follows.  The oracle is pinned
against golden vectors generated from the reference itself
(tests/golden/, made by oracle/gen_golden.py which imports the reference in
the build container) and against the reference tests' known-answer vectors.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` arm may import this package, and only as the checker or
the timed CPU baseline — never as the product path.  The product path
(`paper_2507_16784_b200`) runs on the CUDA library and fails loudly without it.
"""
