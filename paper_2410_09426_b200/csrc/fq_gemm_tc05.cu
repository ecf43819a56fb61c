// fq_gemm_tc05.cu -- W4A4 GEMM + dequant epilogue on 5th-gen tensor cores (tcgen05 kind::i8).
//
//   acc[t,o] = sum_k qa[t,k] qw[o,k]               (Eq.3 outer product)
//   y[t,o]   = cvt_rn(float(acc) * sa[t] * sw[o])  (per-token x per-channel)
//
// Blackwell has no INT4 MMA, so INT4 is widened to INT8 on chip and fed to
// tcgen05.mma.kind::i8 with int32 accumulators in TMEM.  Widening trick: a nibble moved to the
// HIGH half of a byte whose low half is zero IS 16*q as a signed int8 (q in [-8,7] -> 16q in
// [-128,112]); one AND (odd elements) or SHL+AND (even elements) per 4 bytes.  Both operands are
// widened that way, so the tensor core accumulates 256*acc exactly (|256 acc| <= 256*64*K < 2^31
// for K < 131072) and the epilogue divides by 256 exactly.  Inside each 32-element group the
// int8 K order is a fixed permutation of the packed order, identical for A and B, so every dot
// product is unchanged.
//
// Data movement (per CTA, persistent, one CTA per SM, tile 128 tokens x 128 features):
//   A (activations): converter warps load packed rows with 16-byte LDGs (two K-blocks of
//       prefetch in registers), widen, and tcgen05.st them straight into TMEM -- the A
//       operand never touches shared memory (tcgen05.mma with A from TMEM).
//   B (weights):     converter warps load packed rows, widen, and store them into the
//       SWIZZLE_128B K-major shared-memory operand layout (fence.proxy.async, mbarrier).
//   MMA:             one thread issues tcgen05.mma kind::i8 M=128 N=128 K=32, double-buffered
//       TMEM accumulators, tcgen05.commit -> mbarriers.
//   Epilogue:        4 warps, TMEM -> registers -> dequant -> 16-byte global stores.
#include <cstdint>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"
#include "fq_tc05.cuh"

namespace fq {
namespace g2 {

constexpr int BM = 128;                   // tokens per tile (UMMA M)
constexpr int BN = 128;                   // output features per tile (UMMA N)
constexpr int BK = 128;                   // int8 K per stage (one 128-byte swizzle row)
constexpr int UK = 32;                    // K per tcgen05.mma kind::i8
constexpr int STAGES = 4;
constexpr int B_BYTES = BN * BK;          // 16 KB per stage
constexpr int A_COLS = BK / 4;            // TMEM columns per A stage (4 int8 per column)
constexpr int ACC_COLS = BN;
constexpr int TMEM_ACC0 = 0;              // two accumulators: [0, 2*BN)
constexpr int TMEM_A0 = 2 * ACC_COLS;     // A stages: [2*BN, 2*BN + STAGES*A_COLS)
constexpr int TMEM_COLS = 512;
constexpr int NUM_EPI_WARPS = 4;          // warps 0..3
constexpr int MMA_WARP = 4;
constexpr int A_WARP0 = 5, NUM_A_WARPS = 4;   // warps 5..8 (TMEM lane quarter = warp % 4)
constexpr int B_WARP0 = 9, NUM_B_WARPS = 4;   // warps 9..12 (one B row per thread)
constexpr int THREADS = (B_WARP0 + NUM_B_WARPS) * 32;
constexpr size_t SMEM_BYTES = size_t(STAGES) * B_BYTES + 1024 + 256;
constexpr int MAX_K = 131040;   // largest K % 32 == 0 with 256 * 64 * K < 2^31
constexpr uint32_t IDESC = tc::idesc_i8(BM, BN);

static_assert(TMEM_A0 + STAGES * A_COLS <= TMEM_COLS, "TMEM budget");

// 16 packed bytes (32 nibbles) -> 32 int8 values (2 x uint4), each 16x its code.
FQ_DEVICE void widen16x(const uint4& p, uint4& o0, uint4& o1) {
  o0.x = (p.x << 4) & 0xF0F0F0F0u;
  o0.y = p.x & 0xF0F0F0F0u;
  o0.z = (p.y << 4) & 0xF0F0F0F0u;
  o0.w = p.y & 0xF0F0F0F0u;
  o1.x = (p.z << 4) & 0xF0F0F0F0u;
  o1.y = p.z & 0xF0F0F0F0u;
  o1.z = (p.w << 4) & 0xF0F0F0F0u;
  o1.w = p.w & 0xF0F0F0F0u;
}

struct Sched {
  int num_m, num_n, num_tiles, num_kb;
  FQ_DEVICE void tile(int id, int& mb, int& nb) const {
    mb = id % num_m;   // consecutive CTAs share the weight tile
    nb = id / num_m;
  }
  // job j of this CTA: (tile, kb); returns false past the end
  FQ_DEVICE bool job(int j, int& mb, int& nb, int& kb) const {
    const int t = blockIdx.x + (j / num_kb) * gridDim.x;
    if (t >= num_tiles) return false;
    kb = j % num_kb;
    tile(t, mb, nb);
    return true;
  }
};

// One converter row-load: 64 packed bytes (128 K values) of row `row` at K-block kb.
FQ_DEVICE void load_row(uint4 (&r)[4], const uint8_t* base, int rows, int row, int KB, int kb, bool valid) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int kbyte = kb * (BK / 2) + c * 16;
    r[c] = (valid && row < rows && kbyte < KB)
               ? __ldg(reinterpret_cast<const uint4*>(base + size_t(row) * KB + kbyte))
               : make_uint4(0, 0, 0, 0);
  }
}

template <bool OUT_I32, bool BF16>
__global__ void __launch_bounds__(THREADS, 1)
gemm_tc05_kernel(const uint8_t* __restrict__ qa, const float* __restrict__ sa, int T, int K,
                 const uint8_t* __restrict__ qw, const float* __restrict__ sw, int N,
                 void* __restrict__ yv) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(STAGES) * B_BYTES);
  uint64_t* full = bars;                 // [STAGES]  converters -> MMA
  uint64_t* empty = bars + STAGES;       // [STAGES]  MMA -> converters
  uint64_t* tfull = bars + 2 * STAGES;   // [2]       MMA -> epilogue
  uint64_t* tempty = tfull + 2;          // [2]       epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Sched sc;
  sc.num_m = (T + BM - 1) / BM;
  sc.num_n = (N + BN - 1) / BN;
  sc.num_tiles = sc.num_m * sc.num_n;
  sc.num_kb = (K + BK - 1) / BK;
  const int KB = K / 2;  // packed bytes per row

  if (warp == MMA_WARP) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        tc::mbar_init(&full[s], (NUM_A_WARPS + NUM_B_WARPS) * 32);
        tc::mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        tc::mbar_init(&tfull[b], 1);
        tc::mbar_init(&tempty[b], NUM_EPI_WARPS * 32);
      }
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc(tmem_slot, TMEM_COLS);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp >= A_WARP0) {
    // ================================ converters ================================
    const bool is_a = warp < B_WARP0;
    const int quarter = warp & 3;                       // TMEM lane quarter of this warp
    const int r_local = is_a ? (quarter * 32 + lane)    // A row == TMEM lane
                             : ((warp - B_WARP0) * 32 + lane);
    const uint8_t* src = is_a ? qa : qw;
    const int rows = is_a ? T : N;
    uint4 buf0[4], buf1[4];
    int mb, nb, kb;
    bool v0 = sc.job(0, mb, nb, kb);
    load_row(buf0, src, rows, (is_a ? mb * BM : nb * BN) + r_local, KB, kb, v0);
    bool v1 = sc.job(1, mb, nb, kb);
    load_row(buf1, src, rows, (is_a ? mb * BM : nb * BN) + r_local, KB, kb, v1);
    int stage = 0;
    uint32_t phase = 0;
    for (int j = 0; v0; ++j) {
      uint4 buf2[4];
      const bool v2 = sc.job(j + 2, mb, nb, kb);
      load_row(buf2, src, rows, (is_a ? mb * BM : nb * BN) + r_local, KB, kb, v2);   // 2 blocks ahead
      tc::mbar_wait(&empty[stage], phase ^ 1);
      if (is_a) {
        uint32_t w[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint4 o0, o1;
          widen16x(buf0[c], o0, o1);
          w[8 * c + 0] = o0.x; w[8 * c + 1] = o0.y; w[8 * c + 2] = o0.z; w[8 * c + 3] = o0.w;
          w[8 * c + 4] = o1.x; w[8 * c + 5] = o1.y; w[8 * c + 6] = o1.z; w[8 * c + 7] = o1.w;
        }
        const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(TMEM_A0 + stage * A_COLS);
        tc::tmem_st32(taddr, w);
        tc::tmem_st_wait();
        tc::fence_before();
      } else {
        uint8_t* rowp = smem + size_t(stage) * B_BYTES + r_local * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint4 o0, o1;
          widen16x(buf0[c], o0, o1);
          *reinterpret_cast<uint4*>(rowp + (((2 * c) ^ (r_local & 7)) << 4)) = o0;
          *reinterpret_cast<uint4*>(rowp + (((2 * c + 1) ^ (r_local & 7)) << 4)) = o1;
        }
        tc::fence_proxy_async_smem();
      }
      tc::mbar_arrive(&full[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        buf0[c] = buf1[c];
        buf1[c] = buf2[c];
      }
      v0 = v1;
      v1 = v2;
    }
  } else if (warp == MMA_WARP) {
    // ================================ MMA issuer ================================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < sc.num_tiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        tc::mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t tmem_d = tmem_base + uint32_t(TMEM_ACC0 + buf * ACC_COLS);
        for (int kb = 0; kb < sc.num_kb; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
          const uint32_t a_t = tmem_base + uint32_t(TMEM_A0 + stage * A_COLS);
          const uint32_t b0 = smem_u32(smem + size_t(stage) * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            tc::mma_ts<true>(tmem_d, a_t + k * (UK / 4), tc::sdesc_sw128(b0 + k * UK, 16, 1024), IDESC,
                             (kb | k) != 0);
          tc::mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc::mma_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else {
    // ================================ epilogue ================================
    const int r_local = warp * 32 + lane;   // TMEM lane == tile row
    int it = 0;
    for (int tile = blockIdx.x; tile < sc.num_tiles; tile += gridDim.x, ++it) {
      int mb, nb;
      sc.tile(tile, mb, nb);
      const int buf = it & 1;
      tc::mbar_wait(&tfull[buf], (it >> 1) & 1);
      tc::fence_after();
      const int row = mb * BM + r_local;
      const bool row_ok = row < T;
      const float s_a = (!OUT_I32 && row_ok) ? sa[row] * (1.0f / 256.0f) : 0.f;
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        uint32_t v[32];
        tc::tmem_ld32(tmem_base + (uint32_t(warp * 32) << 16) + uint32_t(TMEM_ACC0 + buf * ACC_COLS + cc * 32), v);
        tc::tmem_ld_wait();
        const int col0 = nb * BN + cc * 32;
        if (row_ok) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            const int col = col0 + j;
            if (col >= N) break;
            if constexpr (OUT_I32) {
              int32_t* dst = static_cast<int32_t*>(yv) + size_t(row) * N + col;
              reinterpret_cast<int4*>(dst)[0] =
                  make_int4(int(v[j]) >> 8, int(v[j + 1]) >> 8, int(v[j + 2]) >> 8, int(v[j + 3]) >> 8);
              reinterpret_cast<int4*>(dst)[1] =
                  make_int4(int(v[j + 4]) >> 8, int(v[j + 5]) >> 8, int(v[j + 6]) >> 8, int(v[j + 7]) >> 8);
            } else {
              const float4 w0 = __ldg(reinterpret_cast<const float4*>(sw + col));
              const float4 w1 = __ldg(reinterpret_cast<const float4*>(sw + col + 4));
              const float f0 = float(int(v[j + 0])) * s_a * w0.x, f1 = float(int(v[j + 1])) * s_a * w0.y;
              const float f2 = float(int(v[j + 2])) * s_a * w0.z, f3 = float(int(v[j + 3])) * s_a * w0.w;
              const float f4 = float(int(v[j + 4])) * s_a * w1.x, f5 = float(int(v[j + 5])) * s_a * w1.y;
              const float f6 = float(int(v[j + 6])) * s_a * w1.z, f7 = float(int(v[j + 7])) * s_a * w1.w;
              uint4 o;
              if constexpr (BF16) {
                __nv_bfloat162 h0 = __floats2bfloat162_rn(f0, f1), h1 = __floats2bfloat162_rn(f2, f3);
                __nv_bfloat162 h2 = __floats2bfloat162_rn(f4, f5), h3 = __floats2bfloat162_rn(f6, f7);
                o = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                               *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
                *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(yv) + size_t(row) * N + col) = o;
              } else {
                o = make_uint4(pack_half2(f0, f1), pack_half2(f2, f3), pack_half2(f4, f5), pack_half2(f6, f7));
                *reinterpret_cast<uint4*>(static_cast<__half*>(yv) + size_t(row) * N + col) = o;
              }
            }
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&tempty[buf]);
    }
  }

  __syncthreads();
  if (warp == MMA_WARP) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace g2

bool gemm_tc05_supported(const GemmArgs& a) {
  return a.K % 32 == 0 && a.K <= g2::MAX_K && a.N % 8 == 0 && a.T <= int64_t(1) << 30;
}

cudaError_t gemm_tc05_launch(const GemmArgs& a) {
  using namespace g2;
  auto kern = a.out_i32 ? gemm_tc05_kernel<true, false>
                        : (a.y_bf16 ? gemm_tc05_kernel<false, true> : gemm_tc05_kernel<false, false>);
  static std::atomic<uint64_t> attr_done[3];   // per kernel variant: devices configured
  const int which = a.out_i32 ? 0 : (a.y_bf16 ? 1 : 2);
  if (cudaError_t e = ensure_smem_attr(kern, int(SMEM_BYTES), attr_done[which]); e != cudaSuccess) return e;
  const int num_tiles = int((a.T + BM - 1) / BM) * ((a.N + BN - 1) / BN);
  const int grid = std::min(num_tiles, num_sms());
  kern<<<grid, THREADS, SMEM_BYTES, a.stream>>>(a.qa, a.sa, int(a.T), a.K, a.qw, a.sw, a.N, a.y);
  count_launch();
  return cudaGetLastError();
}

}  // namespace fq
