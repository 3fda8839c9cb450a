"""CPU oracle for the CBIE fill -> ACA -> H-LU hot path.

TEST INFRASTRUCTURE ONLY.  This package is a plain numpy/scipy restatement of
the reference algorithm (``chebscat``, arXiv 2408.17116 reference package) for
the hot path named in BASELINE.json.  It exists to CHECK the CUDA product in
``paper_2408_17116_b200`` and to provide the CPU baseline arm of ``bench.py``.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import it.  The product never imports it.

Parity pin: every module here is checked against golden vectors produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.  Each function cites the reference file:line
(relative to ``/root/reference/pkg/src/chebscat/``) whose behaviour it restates.
"""

from . import spectral, surface, physics, nearfield, hcompress, hfactor, pipeline  # noqa: F401
