"""B200-native FlatQuant online hot path (arXiv 2410.09426).

Per-token Kronecker transform P1^T X P2 + clip + INT4 quantize/pack (fq_transform_quant)
feeding a W4A4 GEMM with dequant epilogue (fq_w4a4_linear), hand-written for sm_100a and
exposed through the C ABI in include/flatquant.h.  See DESIGN.md.
"""
from .api import *  # noqa: F401,F403
from .api import __all__ as _api_all
from ._lib import FQ_BF16, FQ_F16, FQ_SYM, FQ_ASYM, FQ_ESINGULAR, FlatQuantError, LIB_PATH, load  # noqa: F401

__all__ = list(_api_all) + ["FQ_BF16", "FQ_F16", "FQ_SYM", "FQ_ASYM", "FQ_ESINGULAR", "FlatQuantError", "LIB_PATH", "load"]
