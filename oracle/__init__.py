"""CPU oracle for the rangekit hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the reference algorithms that the CUDA
library (`paper_2112_02779_b200`) replaces.  It is the *checker*: only
`tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference`
legs of `bench.py` may import it.  The product package never imports it and
fails loudly when its CUDA library is missing.

Every function cites the reference file:line it follows
(`/root/reference/pkg/src/rangekit/...`).  Parity is pinned by
`tests/golden/*.npz`, produced by `tests/golden/make_golden.py` which imports
the unmodified reference in the build container; `tests/test_oracle_golden.py`
checks this restatement against those vectors bit-for-bit.

Two arithmetic switches exist for the parity tests:

* ``math="numpy"`` evaluates float32 ``arctan2``/``arcsin`` with numpy (SVML on
  AVX-512 hosts), i.e. exactly what the reference does on the same host.
* ``math="cr"`` evaluates them as ``float32(f64 function(float64 args))``, a
  host-independent, (almost always) correctly-rounded result.  The CUDA kernels
  have the same switch, so CR-mode results are compared bit-for-bit.

``fma="blas"`` computes the ``(n,3) @ (3,3)`` float64 transforms with numpy's
BLAS (the reference's own call, fastest — used for CPU baselines), while
``fma="exact"`` evaluates the FMA chain the survey pinned for OpenBLAS 0.3.30
 with an exact software FMA, independent of the host BLAS.
"""


