"""fp64 CPU oracle for the 4D spectral-convolution layer of arXiv 2204.01205.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import or run
anything under ``oracle/``.  The product path (``paper_2204_01205_b200``) never
imports it, and it never imports the product path: the two share no code.

Every function is a plain, slow, obviously-correct restatement of a definition
in PAPER.md (cited as ``P:<line>``) under the readings listed in DESIGN.md
("Readings" table, Q1-Q20, taken from SURVEY.md §8.c).  No FFT is used: every
transform is an explicit DFT-matrix product whose integer phase ``(k*x) mod n``
is reduced before the angle is formed.  ``numpy.fft`` appears only in the tests,
as an independent cross-check.

Parity status per function:
  spectral.forward_modes / inverse_modes / spectral_conv / layer_fwd /
  spectral_conv_adjoint / layer_bwd / gelu / gelu_prime ........ pinned
  decomp.* (partition algebra, decomposition simulator, repartition) pinned
  network.* (lift, projection, relative-L2 loss, network gradients, Adam)  pinned
      (tests/test_oracle_network.py)
  equality with the authors' own ``dfno`` code ........... parity unpinned
  (that code is not available; the pins fix our reading of the paper).
"""

from . import spectral, decomp, network  # noqa: F401
