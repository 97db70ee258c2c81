"""CPU float64 oracle for the NeuRLP-PDE batched solve (arXiv 2502.18377).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2502_18377_b200``) never imports it and it
never imports the product path; the two share no code.  The only module both
sides use is ``synth`` (seeded input generators, no method arithmetic).

Every function cites the PAPER.md passage it follows as ``P:<lines> (<section,
equation>)``.  Readings of silent/ambiguous passages are listed in DESIGN.md
("Readings of the paper") and in SURVEY.md §8(c) Q1-Q20.

Parity status per function:
  * assemble / counts ............ pinned (paper counts P:244-249, MMS, bubble)
  * lstsq_forward/backward ....... pinned (hand cases, finite differences)
  * solve_forward/backward ....... pinned (dense SVD vs LU vs CG, MMS, analytic)
  * field_gradients .............. pinned (central finite differences)
  * derivative-row scaling (Q5) and edge stencils (Q4): "parity unpinned" by the
    paper -- both sides implement the DESIGN.md definition; MMS and the bubble
    identity are convention-independent cross-checks.
"""
from .neurlp import (  # noqa: F401
    Problem, n_fields, field_index, boundary_mask, fd_stencil, assemble, counts,
    lstsq_forward, lstsq_backward, solve_normal, solve_forward, solve_backward,
    field_gradients, normal_apply, assemble_dh, step_gradient,
)
