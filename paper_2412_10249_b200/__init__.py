"""B200-native hot path of ImaSk (arXiv 2412.10249).

Drop-in for the per-iteration path of the reference package `mrtomo`:
`ctmodel` (projector), `mrsketch` (sketch family), `proxlib` (ridge /
quadratic-conjugate prox), `linops` (operator boundary) and `solvers`
(sketched SAGA step and run loop), executed by hand-written sm_100a kernels
in `libimask_b200.so` (sources in `csrc/`, C-ABI in `include/imask_b200.h`).
"""

from . import errors  # noqa: F401

__version__ = "0.1.0"
