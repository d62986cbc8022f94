"""bt200: B200-native (sm_100a) hot path of arXiv 2105.01170's structure-
preserving approximations, a drop-in behind the reference package
``blockten``'s API (same names, arguments, outputs, factor layouts and
exception types; cf. blockten/__init__.py:12-89).  All arithmetic runs in
libbt200.so (hand-written CUDA, FP64 DMMA tensor cores); PyTorch only
provides device memory and streams.
"""

from __future__ import annotations

from .blocks import (BlockPattern, build_pattern, classify_placements, detect_pattern,
                     extract_blocks, kernel_level_pattern, mat_to_tensor, struct_assemble,
                     struct_expand, struct_scalars, tensor_to_mat)
from .decomp import (CpResult, KruskalRep, SketchConfig, TuckerRep, cholesky, cp_als, hooi,
                     hosvd, qr_thin, st_hosvd, svd_truncated, tucker_partial)
from .errors import (ContainerExtentError, ContainerFormatError, ConvergenceError,
                     NotPositiveDefiniteError, PatternMismatchError, ShapeError)
from .multilevel import (MlKronTerm, MultilevelPattern, MultilevelTuckerRep,
                         ml_kron_sum_from_kruskal, ml_kron_sum_from_tucker, ml_matvec,
                         psf_weighted_tensor)
from .psd import (SpdRep, SpsdRep, check_transpose_closed, spd_compress, spsd_compress,
                  spsd_compress_blocks)
from .reconstruct import (BlockLowRankRep, FlopCounter, KronSumRep, TuckerBlockRep,
                          blr_from_kruskal, blr_from_tucker, densify, error_fro,
                          kron_sum_from_kruskal, kron_sum_from_tucker, matvec)
from .tensor import fold, fro_norm, mode_multiply, squeeze, twist, unfold
from .container import container_kind, container_read, container_write
from .apps import (EraResult, LtiSystem, MarkovSequence, era_identify_compressed,
                   hankel_pattern_from_markov, markov_from_lti)
from .dropin import install, installed, uninstall
from . import apps, container, decomp, dropin, multilevel, parallel, psd, reconstruct  # noqa: F401

__version__ = "0.1.0"
