// fq_weight_prep.cu -- GPU weight preparation: the inverse-transpose
// factors of Eq. 3's weight side, W'_o = P1^{-1} W~_o P2^{-T} = (P1^{-T})^T W~_o (P2^{-T})
// (PAPER.md:238-243), so that the activation kernel applied with (P1^{-T}, P2^{-T}, alpha_w)
// produces the per-channel quantized weights.
//
// inverse_t_kernel: Gauss-Jordan elimination with partial pivoting in float64 on one CTA of 1024
// threads over the augmented matrix [P | I] (n x 2n doubles in the caller's workspace, L2
// resident: n <= 256 -> <= 1 MiB).  Offline preparation: runs once per layer, so a single CTA is
// enough; it writes P^{-T} rounded to the weights' dtype and a status word (0 ok, 1 singular
// pivot, 2 inverse not representable in the dtype).
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"

namespace fq {
namespace prep {

constexpr int THREADS = 1024;

template <bool BF16>
FQ_DEVICE double load_elem(const uint16_t* p, int i) {
  if constexpr (BF16) return double(__bfloat162float(__ushort_as_bfloat16(p[i])));
  else return double(__half2float(__ushort_as_half(p[i])));
}

template <bool BF16>
FQ_DEVICE uint16_t store_elem(double v) {
  // double -> float is exact-to-nearest; float -> half/bf16 rounds to nearest even.  The double
  // rounding only matters at exact float-midpoints of the 16-bit grid (measure zero).
  if constexpr (BF16) return __bfloat16_as_ushort(__float2bfloat16_rn(float(v)));
  else return __half_as_ushort(__float2half_rn(float(v)));
}

template <bool BF16>
__global__ void __launch_bounds__(THREADS, 1)
inverse_t_kernel(const uint16_t* __restrict__ p, int n, double* __restrict__ aug, uint16_t* __restrict__ out,
                 int* __restrict__ status) {
  __shared__ double fac[256];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_piv;
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int w2 = 2 * n;
  for (int idx = tid; idx < n * w2; idx += THREADS) {
    const int r = idx / w2, c = idx - r * w2;
    aug[idx] = c < n ? load_elem<BF16>(p, r * n + c) : (c - n == r ? 1.0 : 0.0);
  }
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int c = 0; c < n; ++c) {
    // 1. pivot: row of max |aug[r][c]|, r >= c
    double bv = -1.0;
    int bi = c;
    for (int r = c + tid; r < n; r += THREADS) {
      const double v = fabs(aug[size_t(r) * w2 + c]);
      if (v > bv) { bv = v; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      bv = red_v[lane];
      bi = red_i[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) {
        s_piv = bi;
        if (!(bv > 0.0) || !isfinite(bv)) s_bad = 1;
      }
    }
    __syncthreads();
    if (s_bad) break;
    // 2. swap rows c and piv (columns c.. ; the left part before c is already zero below the diagonal)
    const int pr = s_piv;
    if (pr != c)
      for (int j = c + tid; j < w2; j += THREADS) {
        const double t = aug[size_t(c) * w2 + j];
        aug[size_t(c) * w2 + j] = aug[size_t(pr) * w2 + j];
        aug[size_t(pr) * w2 + j] = t;
      }
    __syncthreads();
    // 3. normalise the pivot row; save the elimination factors of every other row
    const double inv = 1.0 / aug[size_t(c) * w2 + c];
    for (int r = tid; r < n; r += THREADS) fac[r] = r == c ? 0.0 : aug[size_t(r) * w2 + c];
    __syncthreads();
    for (int j = c + tid; j < w2; j += THREADS) aug[size_t(c) * w2 + j] *= inv;
    __syncthreads();
    // 4. eliminate column c from every other row
    const int wc = w2 - c;
    for (int idx = tid; idx < n * wc; idx += THREADS) {
      const int r = idx / wc, j = c + (idx - r * wc);
      if (r != c) aug[size_t(r) * w2 + j] -= fac[r] * aug[size_t(c) * w2 + j];
    }
    __syncthreads();
  }
  // 5. out = (P^{-1})^T in the weights' dtype: out[i][j] = P^{-1}[j][i] = aug[j][n + i]
  if (!s_bad) {
    const double lim = BF16 ? 3.3895313892515355e38 : 65504.0;
    for (int idx = tid; idx < n * n; idx += THREADS) {
      const int i = idx / n, j = idx - i * n;
      const double v = aug[size_t(j) * w2 + n + i];
      if (!(fabs(v) <= lim)) s_bad = 2;        // benign race: any writer stores 2
      out[idx] = store_elem<BF16>(v);
    }
  }
  __syncthreads();
  if (tid == 0) *status = s_bad;
}

}  // namespace prep

size_t weight_prep_workspace(int n1, int n2) {
  const size_t nm = size_t(n1 > n2 ? n1 : n2);
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  return up(nm * 2 * nm * sizeof(double)) + up(size_t(n1) * n1 * 2) + up(size_t(n2) * n2 * 2) + 256;
}

cudaError_t inverse_t_launch(const void* p, int n, bool bf16, void* aug, void* out, int* status,
                             cudaStream_t stream) {
  if (bf16)
    prep::inverse_t_kernel<true><<<1, prep::THREADS, 0, stream>>>(static_cast<const uint16_t*>(p), n,
                                                                  static_cast<double*>(aug),
                                                                  static_cast<uint16_t*>(out), status);
  else
    prep::inverse_t_kernel<false><<<1, prep::THREADS, 0, stream>>>(static_cast<const uint16_t*>(p), n,
                                                                   static_cast<double*>(aug),
                                                                   static_cast<uint16_t*>(out), status);
  count_launch();
  return cudaGetLastError();
}

}  // namespace fq
