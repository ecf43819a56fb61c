// fq_gemm_tc05.cu -- W4A4 GEMM + dequant epilogue on 5th-gen tensor cores (tcgen05 kind::i8).
//
//   acc[t,o] = sum_k qa[t,k] qw[o,k]            (Eq.3 outer product)
//   y[t,o]   = cvt_rn(float(acc) * sa[t] * sw[o])  (per-token x per-channel)
//
// Blackwell has no INT4 MMA, so INT4 is widened to INT8 in shared memory and fed to
// tcgen05.mma.kind::i8 with int32 accumulators in TMEM.  The widening uses a one/two-op
// trick: a nibble moved to the HIGH half of a byte with the low half zero IS 16*q as a
// signed int8 (q in [-8, 7] -> 16q in [-128, 112]).  Both operands are widened that way,
// so the tensor core accumulates 256 * acc exactly (|256 acc| <= 256*64*K < 2^31 for
// K <= 131072); the epilogue divides by 256 exactly.  Within a 32-element group the int8
// K order is a fixed permutation of the packed order, identical for A and B, so the dot
// product is unchanged.
//
// Structure (persistent, one CTA per SM, 1-CTA MMA M=128 x N=256 x K=32 per instruction):
//   warps 0-3  : epilogue (TMEM lanes 32w..32w+31 -> registers -> dequant -> global)
//   warp  4    : TMEM allocator + single-thread MMA issuer
//   warps 5-12 : converters (LDG packed int4 -> widen -> STS into the SWIZZLE_128B K-major
//                operand layout -> fence.proxy.async -> mbarrier arrive)
// Pipelines: smem stages full/empty (converters <-> MMA), TMEM double buffer
// tmem_full/tmem_empty (MMA <-> epilogue).
#include <cstdint>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"

namespace fq {
namespace tc05 {

constexpr int BM = 128;                    // tokens per tile (UMMA M)
constexpr int BN = 256;                    // output features per tile (UMMA N)
constexpr int BK = 128;                    // int8 K per stage (= one 128-byte swizzle row)
constexpr int UK = 32;                     // K per tcgen05.mma kind::i8
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;           // 16 KB
constexpr int B_BYTES = BN * BK;           // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_EPI_WARPS = 4;
constexpr int MMA_WARP = 4;
constexpr int NUM_CONV_WARPS = 8;
constexpr int CONV_THREADS = NUM_CONV_WARPS * 32;
constexpr int THREADS = (NUM_EPI_WARPS + 1 + NUM_CONV_WARPS) * 32;
constexpr int TMEM_COLS = 2 * BN;          // double-buffered int32 accumulator
constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int MAX_K = 131072;              // 256 * 64 * K < 2^31

// ---------------------------------------------------------------- PTX wrappers
FQ_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
FQ_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
FQ_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
FQ_DEVICE void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
FQ_DEVICE void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
FQ_DEVICE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
FQ_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

FQ_DEVICE void tmem_alloc(uint32_t* dst_smem, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
}
FQ_DEVICE void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(cols));
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row atoms of 1024 B.
FQ_DEVICE uint64_t make_sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);          // start address
  d |= uint64_t(1) << 16;                         // leading byte offset (unused for SW128 K-major)
  d |= uint64_t(1024 >> 4) << 32;                 // stride byte offset: 8 rows x 128 B
  d |= uint64_t(1) << 46;                         // descriptor version (sm_100)
  d |= uint64_t(2) << 61;                         // layout: SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::i8, D = s32, A = B = s8, both K-major, M = BM, N = BN.
constexpr uint32_t IDESC = (2u << 4)                    // c_format = S32
                           | (1u << 7)                   // a_format = signed 8-bit
                           | (1u << 10)                  // b_format = signed 8-bit
                           | (uint32_t(BN >> 3) << 17)   // N >> 3
                           | (uint32_t(BM >> 4) << 24);  // M >> 4

FQ_DEVICE void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
FQ_DEVICE void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}

FQ_DEVICE void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// 16 packed bytes (32 nibbles) -> 32 int8 values, each 16x the code (see file header).
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
    mb = id % num_m;   // consecutive CTAs share the weight tile; activations come from L2
    nb = id / num_m;
  }
};

template <bool OUT_I32, bool BF16>
__global__ void __launch_bounds__(THREADS, 1)
gemm_tc05_kernel(const uint8_t* __restrict__ qa, const float* __restrict__ sa, int T, int K,
                 const uint8_t* __restrict__ qw, const float* __restrict__ sw, int N,
                 void* __restrict__ yv) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(STAGES) * STAGE_BYTES);
  uint64_t* full = bars;                 // [STAGES]
  uint64_t* empty = bars + STAGES;       // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;   // [2]
  uint64_t* tempty = tfull + 2;          // [2]
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
        mbar_init(&full[s], CONV_THREADS);
        mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&tfull[b], 1);
        mbar_init(&tempty[b], NUM_EPI_WARPS * 32);
      }
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(tmem_slot, TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp >= NUM_EPI_WARPS + 1) {
    // ================================ converters ================================
    const int ct = threadIdx.x - (NUM_EPI_WARPS + 1) * 32;   // 0..255
    // task mapping inside a stage: row = task / 4, packed 16-byte chunk = task % 4
    constexpr int A_TASKS = BM * 4 / CONV_THREADS;   // 2
    constexpr int B_TASKS = BN * 4 / CONV_THREADS;   // 4
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < sc.num_tiles; tile += gridDim.x) {
      int mb, nb;
      sc.tile(tile, mb, nb);
      for (int kb = 0; kb < sc.num_kb; ++kb) {
        uint4 pa[A_TASKS], pb[B_TASKS];
#pragma unroll
        for (int i = 0; i < A_TASKS; ++i) {
          const int task = ct + i * CONV_THREADS, r = task >> 2, c = task & 3;
          const int row = mb * BM + r, kbyte = kb * (BK / 2) + c * 16;
          pa[i] = (row < T && kbyte < KB)
                      ? __ldg(reinterpret_cast<const uint4*>(qa + size_t(row) * KB + kbyte))
                      : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < B_TASKS; ++i) {
          const int task = ct + i * CONV_THREADS, r = task >> 2, c = task & 3;
          const int row = nb * BN + r, kbyte = kb * (BK / 2) + c * 16;
          pb[i] = (row < N && kbyte < KB)
                      ? __ldg(reinterpret_cast<const uint4*>(qw + size_t(row) * KB + kbyte))
                      : make_uint4(0, 0, 0, 0);
        }
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sA = smem + size_t(stage) * STAGE_BYTES;
        uint8_t* sB = sA + A_BYTES;
#pragma unroll
        for (int i = 0; i < A_TASKS; ++i) {
          const int task = ct + i * CONV_THREADS, r = task >> 2, c = task & 3;
          uint4 o0, o1;
          widen16x(pa[i], o0, o1);
          uint8_t* rowp = sA + r * 128;
          *reinterpret_cast<uint4*>(rowp + (((2 * c) ^ (r & 7)) << 4)) = o0;
          *reinterpret_cast<uint4*>(rowp + (((2 * c + 1) ^ (r & 7)) << 4)) = o1;
        }
#pragma unroll
        for (int i = 0; i < B_TASKS; ++i) {
          const int task = ct + i * CONV_THREADS, r = task >> 2, c = task & 3;
          uint4 o0, o1;
          widen16x(pb[i], o0, o1);
          uint8_t* rowp = sB + r * 128;
          *reinterpret_cast<uint4*>(rowp + (((2 * c) ^ (r & 7)) << 4)) = o0;
          *reinterpret_cast<uint4*>(rowp + (((2 * c + 1) ^ (r & 7)) << 4)) = o1;
        }
        fence_proxy_async_smem();
        mbar_arrive(&full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ================================ MMA issuer ================================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < sc.num_tiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        const uint32_t tphase = (it >> 1) & 1;
        mbar_wait(&tempty[buf], tphase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + uint32_t(buf * BN);
        for (int kb = 0; kb < sc.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + size_t(stage) * STAGE_BYTES);
          const uint32_t b0 = a0 + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {
            mma_i8(tmem_d, make_sdesc(a0 + k * UK), make_sdesc(b0 + k * UK), (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[buf]);
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
      const uint32_t tphase = (it >> 1) & 1;
      mbar_wait(&tfull[buf], tphase);
      tc_fence_after();
      const int row = mb * BM + r_local;
      const bool row_ok = row < T;
      const float s_a = (!OUT_I32 && row_ok) ? sa[row] * (1.0f / 256.0f) : 0.f;
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        uint32_t v[32];
        const uint32_t taddr = tmem_base + (uint32_t(warp * 32) << 16) + uint32_t(buf * BN + cc * 32);
        tmem_ld32(taddr, v);
        const int col0 = nb * BN + cc * 32;
        if (row_ok) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            const int col = col0 + j;
            if (col >= N) break;
            if constexpr (OUT_I32) {
              int32_t* dst = static_cast<int32_t*>(yv) + size_t(row) * N + col;
              int4 w0 = make_int4(int(v[j]) >> 8, int(v[j + 1]) >> 8, int(v[j + 2]) >> 8, int(v[j + 3]) >> 8);
              int4 w1 = make_int4(int(v[j + 4]) >> 8, int(v[j + 5]) >> 8, int(v[j + 6]) >> 8, int(v[j + 7]) >> 8);
              reinterpret_cast<int4*>(dst)[0] = w0;
              reinterpret_cast<int4*>(dst)[1] = w1;
            } else {
              const float4 w0 = __ldg(reinterpret_cast<const float4*>(sw + col));
              const float4 w1 = __ldg(reinterpret_cast<const float4*>(sw + col + 4));
              float f[8];
              f[0] = float(int(v[j + 0])) * s_a * w0.x;
              f[1] = float(int(v[j + 1])) * s_a * w0.y;
              f[2] = float(int(v[j + 2])) * s_a * w0.z;
              f[3] = float(int(v[j + 3])) * s_a * w0.w;
              f[4] = float(int(v[j + 4])) * s_a * w1.x;
              f[5] = float(int(v[j + 5])) * s_a * w1.y;
              f[6] = float(int(v[j + 6])) * s_a * w1.z;
              f[7] = float(int(v[j + 7])) * s_a * w1.w;
              uint4 o;
              if constexpr (BF16) {
                __nv_bfloat162 h0 = __floats2bfloat162_rn(f[0], f[1]), h1 = __floats2bfloat162_rn(f[2], f[3]);
                __nv_bfloat162 h2 = __floats2bfloat162_rn(f[4], f[5]), h3 = __floats2bfloat162_rn(f[6], f[7]);
                o = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                               *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
                *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(yv) + size_t(row) * N + col) = o;
              } else {
                o = make_uint4(pack_half2(f[0], f[1]), pack_half2(f[2], f[3]), pack_half2(f[4], f[5]),
                               pack_half2(f[6], f[7]));
                *reinterpret_cast<uint4*>(static_cast<__half*>(yv) + size_t(row) * N + col) = o;
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[buf]);
    }
  }

  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace tc05

bool gemm_tc05_supported(const GemmArgs& a) {
  return a.K % 32 == 0 && a.K <= tc05::MAX_K && a.N % 8 == 0 && a.T <= int64_t(1) << 30;
}

cudaError_t gemm_tc05_launch(const GemmArgs& a) {
  using namespace tc05;
  auto pick = [&]() {
    if (a.out_i32) return gemm_tc05_kernel<true, false>;
    return a.y_bf16 ? gemm_tc05_kernel<false, true> : gemm_tc05_kernel<false, false>;
  };
  auto kern = pick();
  static bool attr_done[3] = {false, false, false};
  const int which = a.out_i32 ? 0 : (a.y_bf16 ? 1 : 2);
  if (!attr_done[which]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
    if (e != cudaSuccess) return e;
    attr_done[which] = true;
  }
  const int num_tiles = int((a.T + BM - 1) / BM) * ((a.N + BN - 1) / BN);
  const int grid = std::min(num_tiles, num_sms());
  kern<<<grid, THREADS, SMEM_BYTES, a.stream>>>(a.qa, a.sa, int(a.T), a.K, a.qw, a.sw, a.N, a.y);
  count_launch();
  return cudaGetLastError();
}

}  // namespace fq
