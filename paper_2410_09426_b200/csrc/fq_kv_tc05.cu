// fq_kv_tc05.cu -- KV-cache path: per-head online transform + group-wise
// asymmetric INT4 quantization of keys / values.
//
//   y_r = x_r . P_h            (x_r one head vector, D = head_dim; P_h the per-head transform of
//                               keys after RoPE, §3.2; identity for values, whose
//                               P_v is merged into the weights)
//   group = the D values of one head vector (D = 128: "group-wise asymmetric quantization with the
//   size of 128", App. "KV Cache Quantization" PAPER.md:1101-1104)
//   asymmetric INT4 per group exactly as fq_transform_quant's FQ_ASYM (reading R19):
//   s = alpha (hi - lo) / 15, z = rint(-lo / s), q = clamp(rint(y / s) + z, 0, 15), nibble q - 8.
//
// One tcgen05.mma.kind::f16 per 16-wide K step, M = 128 head vectors per tile, N = K = D:
//   A = X tile [128 rows][D]  K-major SWIZZLE_128B (TMA, one box per 64-element K atom)
//   B = P_h    [K = D][N = D] MN-major SWIZZLE_128B (TMA, one box per 64-wide N atom)
// TMEM lane r holds y_r entirely, so the group statistics need no cross-thread reduction: each
// epilogue thread quantizes its own head vector and stores D/2 packed bytes.
// Warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4-7 epilogue; persistent over tiles,
// TMEM double-buffered, X ring of STAGES tiles, programmatic dependent launch.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"
#include "fq_tc05.cuh"

namespace fq {
namespace kv5 {

constexpr int THREADS = 8 * 32;
constexpr float MAGIC = 12582912.0f;   // 1.5 * 2^23

template <int D>
struct Cfg {
  static_assert(D == 64 || D == 128, "head_dim 64 or 128");
  static constexpr int KA = D / 64;                    // 64-element K atoms of a row
  static constexpr int X_BYTES = 128 * D * 2;          // one tile of 128 head vectors
  static constexpr int P_BYTES = D * D * 2;
  static constexpr int STAGES = D == 64 ? 8 : 5;
  static constexpr int TMEM_COLS = D == 64 ? 128 : 256; // two accumulators
  static constexpr size_t SMEM = size_t(P_BYTES) + size_t(STAGES) * X_BYTES + 1024 + 256;
};

FQ_DEVICE float fma_sat(float a, float b, float c) {
  float r;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
FQ_DEVICE uint32_t pack8(const float (&v)[8]) {       // low nibbles of 8 MAGIC-form values
  const uint32_t e = __byte_perm(__byte_perm(__float_as_uint(v[0]), __float_as_uint(v[2]), 0x0040),
                                 __byte_perm(__float_as_uint(v[4]), __float_as_uint(v[6]), 0x0040), 0x5410);
  const uint32_t o = __byte_perm(__byte_perm(__float_as_uint(v[1]), __float_as_uint(v[3]), 0x0040),
                                 __byte_perm(__float_as_uint(v[5]), __float_as_uint(v[7]), 0x0040), 0x5410);
  return (e & 0x0F0F0F0Fu) | ((o << 4) & 0xF0F0F0F0u);
}

template <int D, bool BF16>
__global__ void __launch_bounds__(THREADS, 1)
kv_quant_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmP, int64_t R,
                float alpha, uint8_t* __restrict__ q, float* __restrict__ scale, int8_t* __restrict__ zero) {
  using C = Cfg<D>;
  constexpr int S = C::STAGES;
  constexpr uint32_t IDESC = tc::idesc_f16(128, D, BF16 ? 1 : 0, 0 /*A K-major*/, 1 /*B MN-major*/);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sP = smem;
  uint8_t* sX = sP + C::P_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + size_t(S) * C::X_BYTES);
  uint64_t* xfull = bars;             // [S]
  uint64_t* xempty = bars + S;        // [S]
  uint64_t* pfull = bars + 2 * S;
  uint64_t* dfull = pfull + 1;        // [2] MMA commit -> epilogue
  uint64_t* dempty = dfull + 2;       // [2] epilogue (4 warps) -> MMA
  __shared__ uint32_t tmem_slot[1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = int((R + 127) / 128);
  const int my_tiles = num_tiles > int(blockIdx.x) ? (num_tiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;

  auto issue_x = [&](int k) {
    const int s = k % S;
    tc::mbar_wait(&xempty[s], ((k / S) & 1) ^ 1);
    tc::mbar_expect_tx(&xfull[s], C::X_BYTES);
    const int r0 = (int(blockIdx.x) + k * int(gridDim.x)) * 128;
#pragma unroll
    for (int a = 0; a < C::KA; ++a)
      tc::tma_load_2d(sX + size_t(s) * C::X_BYTES + a * 128 * 128, &tmX, &xfull[s], a * 64, r0);
  };
  const int prefill = my_tiles < S ? my_tiles : S;
  if (threadIdx.x == 0) {
    tc::tma_prefetch_desc(&tmX);
    tc::tma_prefetch_desc(&tmP);
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&xfull[s], 1);
      tc::mbar_init(&xempty[s], 1);
    }
    tc::mbar_init(pfull, 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&dfull[b], 1);
      tc::mbar_init(&dempty[b], 4);
    }
    tc::fence_barrier_init();
    tc::griddep_wait();
    tc::griddep_launch();              // dependents launch only after the wait (fq_internal.h)
    tc::mbar_expect_tx(pfull, C::P_BYTES);
#pragma unroll
    for (int a = 0; a < C::KA; ++a) tc::tma_load_2d(sP + a * D * 128, &tmP, pfull, a * 64, 0);
    for (int k = 0; k < prefill; ++k) issue_x(k);
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0)
      for (int k = prefill; k < my_tiles; ++k) issue_x(k);
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      tc::mbar_wait(pfull, 0);
      const uint32_t pa = smem_u32(sP);
      for (int k = 0; k < my_tiles; ++k) {
        const int s = k % S, buf = k & 1;
        tc::mbar_wait(&dempty[buf], ((k >> 1) & 1) ^ 1);
        tc::mbar_wait(&xfull[s], (k / S) & 1);
        tc::fence_after();
        const uint32_t xa = smem_u32(sX + size_t(s) * C::X_BYTES);
        const uint32_t d = tmem + uint32_t(buf * D);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          // A: K-major, K atom kk/4 (16 KB apart), 32 bytes per 16-element step inside the atom
          const uint64_t ad = tc::sdesc_sw128(xa + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
          // B: MN-major, 16 K rows = 2 KB per step, N atoms D rows x 128 B apart
          const uint64_t bd = tc::sdesc_sw128(pa + kk * 2048, D * 128, 1024);
          tc::mma_ss<false>(d, ad, bd, IDESC, kk > 0);
        }
        tc::mma_commit(&xempty[s]);
        tc::mma_commit(&dfull[buf]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int qd = warp & 3, L = qd * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t(qd * 32) << 16);
    for (int k = 0; k < my_tiles; ++k) {
      const int buf = k & 1;
      tc::mbar_wait(&dfull[buf], (k >> 1) & 1);
      tc::fence_after();
      const int64_t r = (int64_t(blockIdx.x) + int64_t(k) * gridDim.x) * 128 + L;
      // pass 1: group statistics of this head vector (in-thread)
      float hi = 0.f, lo = 0.f;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t v[32];
        tc::tmem_ld32(lane_base + uint32_t(buf * D + c), v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          hi = fmaxf(hi, __uint_as_float(v[e]));
          lo = fmaxf(lo, -__uint_as_float(v[e]));
        }
      }
      const float range = alpha * (hi + lo);
      const float sp = range * (1.0f / 15.0f);
      const float zq = sp > 0.f ? rintf(__fdiv_rn(alpha * lo, sp)) : 0.f;
      const float c15 = sp > 0.f ? __frcp_rn(range) : 0.f;
      const float b15 = zq * (1.0f / 15.0f);
      // pass 2: quantize + pack + store (D/2 bytes per head vector)
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t v[32];
        tc::tmem_ld32(lane_base + uint32_t(buf * D + c), v);
        tc::tmem_ld_wait();
        uint32_t w[4];
#pragma unroll
        for (int c8 = 0; c8 < 4; ++c8) {
          float z[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            z[e] = fmaf(fma_sat(__uint_as_float(v[8 * c8 + e]), c15, b15), 15.0f, MAGIC - 8.0f);
          w[c8] = pack8(z);
        }
        if (r < R) *reinterpret_cast<uint4*>(q + r * (D / 2) + c / 2) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      if (r < R) {
        scale[r] = sp > 0.f ? sp : 1.0f;
        zero[r] = int8_t(int(zq) - 8);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dempty[buf]);
    }
  }

  tc::fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int D, bool BF16>
static cudaError_t launch(const KVArgs& a) {
  using C = Cfg<D>;
  auto kern = kv_quant_kernel<D, BF16>;
  static std::atomic<uint64_t> attr_done{0};   // devices configured for this kernel
  if (cudaError_t e = ensure_smem_attr(kern, int(C::SMEM), attr_done); e != cudaSuccess) return e;
  CUtensorMap mx, mp;
  {
    const uint64_t dims[2] = {uint64_t(D), uint64_t(a.R)};
    const uint64_t strides[1] = {uint64_t(a.ldx) * 2};
    const uint32_t box[2] = {64, 128};
    if (!tmap_encode(&mx, a.x, 2, 2, dims, strides, box, TMAP_SW128)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {uint64_t(D), uint64_t(D)};
    const uint64_t strides[1] = {uint64_t(D) * 2};
    const uint32_t box[2] = {64, uint32_t(D)};
    if (!tmap_encode(&mp, a.p, 2, 2, dims, strides, box, TMAP_SW128)) return cudaErrorInvalidValue;
  }
  const int64_t tiles = (a.R + 127) / 128;
  const int grid = int(std::min<int64_t>(tiles, num_sms()));
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(THREADS), C::SMEM, a.stream, 1, mx, mp, a.R, a.alpha, a.q,
                             a.scale, a.zero);
  count_launch();
  return e;
}

}  // namespace kv5

bool kv_quant_supported(const KVArgs& a) {
  const bool al = ((reinterpret_cast<uintptr_t>(a.x) | reinterpret_cast<uintptr_t>(a.p) |
                    reinterpret_cast<uintptr_t>(a.q)) & 15u) == 0 &&
                  (a.ldx * 2) % 16 == 0 && a.R < (int64_t(1) << 31);
  return (a.D == 64 || a.D == 128) && al && tmap_available();
}

cudaError_t kv_quant_launch(const KVArgs& a) {
  using namespace kv5;
  if (a.D == 64) return a.bf16 ? launch<64, true>(a) : launch<64, false>(a);
  return a.bf16 ? launch<128, true>(a) : launch<128, false>(a);
}

}  // namespace fq
