"""CPU oracle for the rPIE hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy restatement of the reference algorithm
(``ptychokit``, /root/reference/pkg/src/ptychokit) for the path named by
BASELINE.json's north star: one rPIE sweep with mixed-state probe modes,
upsampled-DFT registration and Adam position refinement.  Every function cites
the reference file:line it restates.

Rules:
  * only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import this package;
  * it is the checker, never the thing measured on the GPU path and never a
    fallback of the product (``paper_2205_04295_b200`` does not import it);
  * it is pinned against golden vectors produced by running the reference
    itself (tests/golden/make_golden.py, checked by tests/test_oracle_golden.py).

The restatement is written for an arbitrary complex dtype so the same code
gives the fp64 reference trajectory and a complex64 shadow used to bound the
fp32 kernels' per-visit error.
"""

from . import rpie, registration, batched  # noqa: F401
