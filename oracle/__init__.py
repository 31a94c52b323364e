"""CPU oracle for the Ulysses hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything here, and
only as the checker (or the timed CPU baseline).  The product path in
``paper_2309_14509_b200`` never imports this package and has no CPU
fallback.

``ulysses_oracle`` restates, in float64 NumPy, the reference ``seqlab``
functions on the DistributedAttention path (every function cites the
reference ``file:line`` it follows; paths are relative to
``/root/reference/pkg/src/seqlab``).  Parity of the restatement is pinned
against golden vectors produced by the unmodified reference
(``oracle/gen_golden.py`` -> ``tests/golden/*.npz``) and against the
reference's own known-answer tests (``tests/test_oracle_golden.py``).

Two restatements have no reference counterpart and are therefore only
pinned indirectly:
  * GQA (the reference is MHA-only): K/V heads are replicated across their
    query-head group and dK/dV are summed over the group.  Pinned by
    reduction to MHA (H_kv == H_q reproduces the golden vectors).
  * LSE (the reference recomputes probabilities and never stores it):
    ``m + log(sum(exp(s - m)))`` over the reference's own score rows.
    Checked only through O and the gradients it feeds.
"""
