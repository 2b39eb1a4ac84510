"""Plain FP64 CPU oracle for the sketch-then-LUPP skeleton-selection path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import anything
from this package.  The product path (``paper_2104_05877_b200``) never imports
it and has no CPU fallback.

The oracle is written from the paper (Dong & Martinsson, arXiv 2104.05877,
``/root/reference/PAPER.md``; citations ``P:<line>``) and shares no code with the
CUDA path: no kernels, headers, helpers, tables or constants.  Each function
cites the passage it follows.  Where the paper is silent the reading taken is
the one listed in ``DESIGN.md`` §3 ("Readings"), quoted in the docstring.

Modules
-------
philox    Philox4x32-10 counter-based generator (Salmon et al. 2011), numpy.
omega     The embeddings Gamma (Gaussian, sparse sign).
sketch    X = Gamma A (Alg. 2 line 2).
lupp      column-wise / row-wise LUPP (eq:def_LUPP; Alg. 2 lines 3-4).
cpqr      column-pivoted QR on the sketch (eq:def_QRCP).
idcoef    ID coefficients Z and the Theorem 4.1 certificate eta.
residual  ||A - CC^+A||_F and its row-ID / CUR / ID-coefficient analogues
          (eq:def_column_id, eq:def_row_id, Remark 2.3 P:133-137).
dist      the column-sharded LUPP merge rule, emulated on one host.

Parity status of every function is listed in DESIGN.md §4 ("Pins"); none is
"parity unpinned".
"""
