"""Oracle for the RollPacker tail-batching rollout path (arXiv 2509.21009).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2509_21009_b200``) never imports it, and
this package never imports the product path: the two share no code.  Inputs
come from ``synth/`` (seeded generators that hold none of the method's
arithmetic).

Contents (each function cites the passage it follows; ``P:n`` =
/root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n, ``Zk`` = the
reading numbered k in DESIGN.md §3):

* ``philox``  — Philox4x32-10 counter-based generator (Z10, Z12).
* ``weights`` — the random-init weight formula (Z12), widened bf16 -> fp64.
* ``decoder`` — plain fp64 Qwen2-shaped decoder, teacher-forced logits
  (C-2 in SURVEY.md §8(c)).
* ``sampler`` — Gumbel-max sampling with Philox noise (Z9-Z11).
* ``sched``   — the tail-batching schedule: closed form, literal step loop,
  round planner and the DP cutoff protocol (
  S:271-306).

Parity status: ``sched`` is pinned by brute force, SPEC examples and
invariants; ``philox`` by Random123 KATs; ``sampler`` by the Gumbel-max
law (chi-square) and special cases; ``decoder`` pieces by closed forms and
the whole decoder by a library cross-check (transformers Qwen2).  The
whole-decoder VALUES are otherwise *parity unpinned* (the paper prints no
logits) -- see DESIGN.md §3.
"""
