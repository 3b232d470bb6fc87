"""Plain, slow, obviously-correct CPU oracle for Hilbert-guided local attention.

TEST INFRASTRUCTURE ONLY.  Nothing under ``oracle/`` is part of the product path:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it.  It shares no code with the CUDA path
(``paper_2511_05832_b200/``) and imports nothing from it; the only module both
sides use is the seeded input generator ``hla_synth`` (no method arithmetic).

Citation convention: ``P:L123`` = /root/reference/PAPER.md line 123 (the paper,
arXiv 2511.05832), ``S:L45`` = SPEC.md line 45.  Readings of garbled / silent
passages are listed in DESIGN.md section "Readings".

Modules
  hilbert    - grid orderings (row-major, Hilbert via gilbert2d recursion)
  patterns   - allowed(q,k) predicates of HWA/HSA/HNA/HSWA/WSA/SA/NA2D/DENSE
  blocks     - full/partial/empty tile classification, CSR, sparsity
  attention  - fp64 dense masked attention forward and backward

Pinning status (see tests/test_oracle_*.py): every function is pinned; none is
"parity unpinned".
"""

from . import hilbert, patterns, blocks, attention  # noqa: F401
