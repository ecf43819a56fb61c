"""Float64 CPU oracle for the FlatQuant online hot path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  See flatquant_oracle.py.
"""
from .flatquant_oracle import *  # noqa: F401,F403
from .flatquant_oracle import (choose_decomposition, kron_transform, kron_matrix, quantize_rows,
                               dequantize_rows, pack_int4, unpack_int4, transform_quant,
                               transform_weight, prepare_weight, int_gemm, int_gemm_bruteforce,
                               dequant, w4a4_linear, flatquant_linear, near_tie_mask,
                               quantize_rows_asym, dequantize_rows_asym, transform_quant_asym,
                               w4a4_linear_asym, kv_quant)
