// fq_gemm_mma.cu -- W4A4 GEMM + dequant epilogue on the legacy warp-level IMMA path
// (mma.sync m16n8k32 s8).  This is the cross-check kernel: it is selected only through
// fq_set_gemm_impl(1) and exists so that the tcgen05 kernel can be validated against a
// second, independent GPU implementation.  PAPER.md:315 (INT4 GEMM).
//
//   acc[t,o] = sum_k qa[t,k] qw[o,k]  (int4 widened to int8 in shared memory)
//   y[t,o]   = cvt_rn(float(acc) * sa[t] * sw[o])   or acc itself (int32 export)
#include <cstdint>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"

namespace fq {

namespace {
constexpr int BM = 128, BN = 128, BK = 64;       // BK in int8 elements (32 packed bytes)
constexpr int PITCH = BK + 16;                    // bytes per smem row (conflict-free frags)
constexpr int THREADS = 256;
}  // namespace

template <bool OUT_I32, bool BF16>
__global__ void __launch_bounds__(THREADS)
gemm_mma_kernel(const uint8_t* __restrict__ qa, const float* __restrict__ sa, int64_t T, int K,
                const uint8_t* __restrict__ qw, const float* __restrict__ sw, int N,
                void* __restrict__ yv) {
  __shared__ __align__(16) uint8_t sA[BM * PITCH];
  __shared__ __align__(16) uint8_t sB[BN * PITCH];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, qd = lane & 3;
  const int wm = warp >> 2;        // 0..1 -> 64 rows each
  const int wn = warp & 3;         // 0..3 -> 32 cols each
  const int64_t m0 = int64_t(blockIdx.y) * BM;
  const int n0 = blockIdx.x * BN;
  const int KB = K / 2;            // packed bytes per row

  // loader mapping: row = tid/2, 16-byte chunk = tid%2 (32 nibbles)
  const int lrow = tid >> 1, lchunk = tid & 1;
  const bool a_ok = (m0 + lrow) < T;
  const bool b_ok = (n0 + lrow) < N;
  const uint8_t* a_src = qa + (a_ok ? (m0 + lrow) : 0) * int64_t(KB) + lchunk * 16;
  const uint8_t* b_src = qw + (b_ok ? (n0 + lrow) : 0) * int64_t(KB) + lchunk * 16;

  int acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0;

  auto gload = [&](int kb, uint4& ra, uint4& rb) {
    const int kbyte = kb * (BK / 2) + lchunk * 16;
    const bool kin = kbyte < KB;
    ra = (a_ok && kin) ? *reinterpret_cast<const uint4*>(a_src + kb * (BK / 2)) : make_uint4(0, 0, 0, 0);
    rb = (b_ok && kin) ? *reinterpret_cast<const uint4*>(b_src + kb * (BK / 2)) : make_uint4(0, 0, 0, 0);
  };
  auto sstore = [&](uint8_t* s, const uint4& r) {
    uint32_t w[8];
    widen_int4x8(r.x, w[0], w[1]);
    widen_int4x8(r.y, w[2], w[3]);
    widen_int4x8(r.z, w[4], w[5]);
    widen_int4x8(r.w, w[6], w[7]);
    uint8_t* dst = s + lrow * PITCH + lchunk * 32;
    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4*>(dst + 16) = make_uint4(w[4], w[5], w[6], w[7]);
  };

  const int nkb = (K + BK - 1) / BK;
  uint4 ra, rb;
  gload(0, ra, rb);
  for (int kb = 0; kb < nkb; ++kb) {
    __syncthreads();
    sstore(sA, ra);
    sstore(sB, rb);
    __syncthreads();
    if (kb + 1 < nkb) gload(kb + 1, ra, rb);
#pragma unroll
    for (int ks = 0; ks < BK; ks += 32) {
      uint32_t af[4][4], bf[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint8_t* base = sA + (wm * 64 + i * 16 + g) * PITCH + ks + 4 * qd;
        af[i][0] = *reinterpret_cast<const uint32_t*>(base);
        af[i][1] = *reinterpret_cast<const uint32_t*>(base + 8 * PITCH);
        af[i][2] = *reinterpret_cast<const uint32_t*>(base + 16);
        af[i][3] = *reinterpret_cast<const uint32_t*>(base + 8 * PITCH + 16);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint8_t* base = sB + (wn * 32 + j * 8 + g) * PITCH + ks + 4 * qd;
        bf[j][0] = *reinterpret_cast<const uint32_t*>(base);
        bf[j][1] = *reinterpret_cast<const uint32_t*>(base + 16);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) mma_s8_16832(acc[i][j], af[i], bf[j][0], bf[j][1]);
    }
  }

  // ---- epilogue: per-token x per-channel dequant (or raw int32) ----
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t row = m0 + wm * 64 + i * 16 + g + h * 8;
      if (row >= T) continue;
      const float s_a = OUT_I32 ? 0.f : sa[row];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = n0 + wn * 32 + j * 8 + 2 * qd;
        if (col >= N) continue;
        const int v0 = acc[i][j][2 * h], v1 = acc[i][j][2 * h + 1];
        if constexpr (OUT_I32) {
          *reinterpret_cast<int2*>(static_cast<int32_t*>(yv) + row * N + col) = make_int2(v0, v1);
        } else {
          const float f0 = float(v0) * s_a * sw[col];
          const float f1 = float(v1) * s_a * sw[col + 1];
          if constexpr (BF16) {
            __nv_bfloat162 o = __floats2bfloat162_rn(f0, f1);
            *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(yv) + row * N + col) = o;
          } else {
            __half2 o = __floats2half2_rn(f0, f1);
            *reinterpret_cast<__half2*>(static_cast<__half*>(yv) + row * N + col) = o;
          }
        }
      }
    }
  }
}

cudaError_t gemm_mma_launch(const GemmArgs& a) {
  dim3 grid(unsigned((a.N + BN - 1) / BN), unsigned((a.T + BM - 1) / BM));
  if (a.out_i32)
    gemm_mma_kernel<true, false><<<grid, THREADS, 0, a.stream>>>(a.qa, a.sa, a.T, a.K, a.qw, a.sw, a.N, a.y);
  else if (a.y_bf16)
    gemm_mma_kernel<false, true><<<grid, THREADS, 0, a.stream>>>(a.qa, a.sa, a.T, a.K, a.qw, a.sw, a.N, a.y);
  else
    gemm_mma_kernel<false, false><<<grid, THREADS, 0, a.stream>>>(a.qa, a.sa, a.T, a.K, a.qw, a.sw, a.N, a.y);
  count_launch();
  return cudaGetLastError();
}

}  // namespace fq
