"""CPU oracle for the IE forward solver of arXiv 2306.17537 — TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct numpy/scipy implementation of what the
paper defines (§2, Eqs. 3-10, 11-24, Algorithm 1, Appendices A and C). It exists
to check the CUDA path. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it. The product package
``paper_2306_17537_b200`` never imports it, and it never imports the product package.
It shares no code with the CUDA path; the only shared module is ``ie_workloads``
(seeded input generators, which contain none of the method's arithmetic).

All arithmetic is float64 / complex128.  Field layout: ``(3, nz, ny, nx)`` complex
(component-major, x fastest) -- the same layout the C-ABI uses, so fields can be compared
element by element.  Conductivity tensors: ``(nz, ny, nx, 3, 3)`` float64.

Parity status per function is listed in DESIGN.md §Oracle.  Every function below is pinned
by a ``-m "not gpu"`` test in ``tests/test_oracle_*.py`` except where its docstring says
"parity unpinned".
"""

from . import physics, operator, gmres, dd, receivers, layered, preconditioner  # noqa: F401
