"""Plain, slow, obviously-correct CPU oracle for the Inf-CL loss hot path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may
import anything under ``oracle/``.  The product path (``paper_2410_17243_b200``) never imports it and shares no
code with it.  Everything here is numpy float64 (or pure Python with ``math.fsum`` for tiny brute-force cases).

Citations: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n.
Readings of ambiguous passages are listed in DESIGN.md "Readings" (Q1..Q23 of SURVEY.md 8(c)).

Pinning (every function below is pinned by a ``-m "not gpu"`` test against something other than itself):
  brute-force Python loops (tests/brute.py, used by tests/test_oracle_pins.py), closed forms (identical features, one-hot classes,
  codebook inputs), central finite differences, gradient invariants, swap symmetry, and the SPEC's printed
  examples (tests/golden/spec_examples.txt).  No function is "parity unpinned".
"""
from .infonce import (  # noqa: F401
    NEG_INF,
    similarity,
    tile_lse,
    merge_lse,
    lse_rows,
    lse_cols,
    tiled_lse_rows,
    forward,
    backward,
    backward_abs,
    loss_and_grads,
    loss_only,
    streamed_forward,
    streamed_grad_scale,
    sampled_row_grads,
    streamed_row_lse,
    streamed_row_grads,
    ring_schedule,
    ring_forward,
    ring_backward,
    onehot_closed_form,
    codebook_closed_form,
    to_f64,
)
from . import ntxent  # noqa: F401  (SimCLR NT-Xent, the second workload: SURVEY 8(f) f4)
