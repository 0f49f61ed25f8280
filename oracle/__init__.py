"""CPU oracle for the divergence-uncertainty hot path -- TEST INFRASTRUCTURE ONLY.

This package is the *checker*, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
(``paper_2510_01190_b200``) never imports, calls or links anything here, and
fails loudly when its CUDA library is missing instead of falling back to it.

Contents
--------
``ref2d``  numpy restatement of the reference's 2D hot path
           (``/root/reference/pkg/src/divuq``: stencils.py, divergence.py,
           gaussian.py, lcp.py, mc.py).  Pinned bitwise against golden vectors
           produced by the reference itself (``tests/golden/make_golden.py``).
``ref3d``  3D restatement (no reference code exists): the same
           per-axis stencil rule applied to z.  Parity here is pinned only by
           the planar-reduction test against the 2D reference plus the
           identity / rotation / uniform-sigma / zero-sigma invariants.
``philox`` Philox4x32-10 + Box-Muller stream used by the GPU Monte Carlo
           kernel (the north star mandates it instead of the reference's
           splitmix64 + AS241), pinned by the Random123 known-answer vectors,
           and the MC estimator restated with the GPU's exact chunk/merge order.
``refstream`` the reference's own MC stream (splitmix64 + AS241, rng.py) and
           its estimator / single-vertex sampler / histogram (mc.py:94-156),
           pinned bitwise against vectors the reference produced
           (``tests/golden/make_golden_refstream.py``).
``divuq1`` the DIVUQ1 container reader / header formatter (io.py:38-93),
           pinned against files the reference's own writer produced.
"""

from . import ref2d, ref3d, philox, divuq1  # noqa: F401
