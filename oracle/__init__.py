"""fp64 CPU oracle for the PTD-P hot path (arXiv 2104.04473).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2104_04473_b200`` and its CUDA library)
never imports, links or executes anything here, and this package imports
nothing from the product path: the two share no code.  The only shared module
is ``gen`` (seeded input generation, no arithmetic of the method).

Citation convention: ``P:n`` = /root/reference/PAPER.md line n (with its
section / equation label), ``S:n`` = SPEC.md line n.

Modules
  formulas  Eq. (1) parameter count, Eq. (2) FLOP count + Appendix terms,
            communication volumes (Sec. 3.2, Sec. 4.1), Eq. (3) train time.
  schedule  stage map, GPipe / 1F1B / interleaved schedules, exact event
            simulator, bubble, in-flight, validator, channel orders, brute force.
  layer     plain fp64 transformer layer fwd/bwd, unpartitioned and t-way
            partitioned (Sec. 2.3, Megatron partitioning).
  model     embedding, head, cross-entropy, full model fwd/bwd, pipeline-
            executed model, Adam.
  philox    Philox-4x32-10 counter-based generator used for dropout masks.

Parity status of every function is pinned by ``tests/test_oracle_*.py``; no
function here is "parity unpinned" (see DESIGN.md Sec. Oracle pins).
"""
