"""HAPI oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (NumPy, float64) of what the
storage-side hot path of HAPI (arXiv 2210.08650) computes: the eval-mode forward of a
frozen DNN prefix up to the split layer, plus the planner's exact integer arithmetic
(Alg. 1, section 4.3 memory estimate, Eq. 4 single-request batch).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the CUDA
path (``paper_2210_08650_b200``); the only module both sides use is the seeded input
generator ``hapi_inputs``.

Parity pins (tests/test_oracle_*.py): brute-force loops on tiny tensors, torch fp64
functional ops and torchvision fp64 models (library pins), paper anchors in
tests/golden/ (section 5.3, 5.6, Table 2), closed forms and invariants.  No function
here is "parity unpinned".
"""
from . import archs, ops, planner, prefix  # noqa: F401
from .planner import choose_split, layer_sizes  # noqa: F401
from .prefix import prefix_forward  # noqa: F401
