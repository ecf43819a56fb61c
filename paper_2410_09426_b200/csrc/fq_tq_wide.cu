// fq_tq_wide.cu -- fused Kronecker transform + clip + per-token INT4 quantize + pack for WIDE
// decompositions, n1 = 128 and 128 < n2 <= 256 (LLaMA-3-70B down_proj: 28672 = 128 x 224, SURVEY
// 8(a) config C5), on tcgen05 with the stage-2 operand held in TMEM.
//
// Per token t (Eq.3; clip PAPER.md:258-259; per-token INT4 PAPER.md:367):
//   V_t = reshape(x_t, 128, n2)   W_t = P1^T V_t   Y_t = W_t P2
//   s_t = alpha max|Y_t| / 7       q = clamp(rint(Y_t / s_t), -8, 7), packed
//
// The general tcgen05 kernel (fq_tq_tc05.cu) keeps P1, P2, the X ring AND the fp16 intermediate
// in shared memory; at 128 x 224 that is 264 KB, over the 227 KB limit.  This kernel removes the
// intermediate from shared memory by choosing the operand roles so that stage 1 leaves W_t in
// TMEM in exactly the layout stage 2 reads its A operand from:
//   stage 1  D[i][j] = sum_i' P1[i'][i] V[i'][j]       A = P1 (smem, MN-major: A[m=i][k=i'])
//                                                     B = V  (smem, MN-major: B[k=i'][n=j])
//            -> TMEM lane i holds row i of W_t (fp32, n2 columns)
//   epilogue per-token power-of-two prescale (exact, overflow-safe; DESIGN reading R9), fp16,
//            written back IN PLACE as the A operand (lane i, K = j' two fp16 per column)
//   stage 2  D2[i][j] = sum_j' W[i][j'] P2[j'][j]     A = W  (TMEM)
//                                                     B = P2 (smem, MN-major: B[k=j'][n=j])
//            -> TMEM lane i holds row i of Y_t: quantized and stored as one contiguous run
// Shared memory: P1 32 KB + P2 (n2/64 atoms x n2 rows x 128 B) + X stages (n2/64 atoms x 16 KB).
// TMEM: region R1 [0, 256) holds D1 then (in place) the fp16 A operand; region R2 [256, 512)
// holds D2, so the stage-2 epilogue of token k overlaps stage 1 + its epilogue of token k+1.
//   warp 0   TMA producer (P1, P2 once, then X tokens into the ring)
//   warp 1   MMA issuer (one thread): stage 1 of token k, then stage 2 of token k
//   warp 2   TMEM allocator
//   warps 4-7 epilogue (TMEM lane quarter = warp % 4; lane i = row i of the token)
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"
#include "fq_tc05.cuh"

namespace fq {
namespace tqw {

constexpr int N1 = 128;
constexpr int SMEM_LIMIT = 232448;
constexpr int SMEM_OVERHEAD = 1024 + 512;
constexpr int THREADS = 12 * 32;                 // round 2c: two epilogue groups (stage 1 / stage 2)
constexpr int R2 = 256;                          // TMEM column of region R2 (D2)
constexpr float MAGIC = 12582912.0f;             // 1.5 * 2^23: fma(y, c, MAGIC) rounds half-to-even

template <int N2>
struct Cfg {
  static_assert(N2 % 32 == 0 && N2 > 128 && N2 <= 256, "n2 in (128, 256], multiple of 32");
  static constexpr int JB = (N2 + 63) / 64;            // 64-element j atoms
  static constexpr int P1_BYTES = 2 * N1 * 128;        // 2 i-atoms x 128 i' rows
  static constexpr int P2_BYTES = JB * N2 * 128;       // JB j-atoms x n2 j' rows
  static constexpr int X_BYTES = JB * N1 * 128;        // JB j-atoms x 128 i' rows
  static constexpr int FIXED = P1_BYTES + P2_BYTES;
  static constexpr int STAGES_FIT = (SMEM_LIMIT - SMEM_OVERHEAD - FIXED) / X_BYTES;
  static constexpr int STAGES = STAGES_FIT > 4 ? 4 : STAGES_FIT;
  static constexpr size_t SMEM = size_t(FIXED) + size_t(STAGES) * X_BYTES + SMEM_OVERHEAD;
  static_assert(STAGES >= 1, "shared-memory budget");
};

FQ_DEVICE int prescale_exp(float m) {            // m 2^e in [2^14, 2^15): fp16-safe, exact
  const int be = int(__float_as_uint(m) >> 23);
  if (be == 0) return 126;
  const int e = 14 - (be - 127);
  return e < -126 ? -126 : (e > 126 ? 126 : e);
}
FQ_DEVICE float exp2i(int e) { return __int_as_float((127 + e) << 23); }
FQ_DEVICE float max3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
FQ_DEVICE float fma_sat(float a, float b, float c) {
  float r;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
FQ_DEVICE uint32_t pack8(const float (&v)[8]) {  // MAGIC-form codes -> 8 nibbles, element 2m low
  const uint32_t e = __byte_perm(__byte_perm(__float_as_uint(v[0]), __float_as_uint(v[2]), 0x0040),
                                 __byte_perm(__float_as_uint(v[4]), __float_as_uint(v[6]), 0x0040), 0x5410);
  const uint32_t o = __byte_perm(__byte_perm(__float_as_uint(v[1]), __float_as_uint(v[3]), 0x0040),
                                 __byte_perm(__float_as_uint(v[5]), __float_as_uint(v[7]), 0x0040), 0x5410);
  return (e & 0x0F0F0F0Fu) | ((o << 4) & 0xF0F0F0F0u);
}
FQ_DEVICE void tmem_ld32c(uint32_t taddr, uint32_t (&v)[32]) {
  tc::tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
  tc::tmem_ld16(taddr + 16u, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
  tc::tmem_ld_wait();
}
FQ_DEVICE void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

template <int N2, bool BF16, bool WRITE_Y, bool ASYM>
__global__ void __launch_bounds__(THREADS, 1)
tq_wide_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmP1,
               const __grid_constant__ CUtensorMap tmP2, int64_t T, float alpha, uint8_t* __restrict__ q,
               float* __restrict__ scale, float* __restrict__ y_out, int8_t* __restrict__ zero, int pdl) {
  using C = Cfg<N2>;
  constexpr int S = C::STAGES;
  constexpr uint32_t IDESC1 = tc::idesc_f16(128, N2, BF16 ? 1 : 0, 1, 1);
  constexpr uint32_t IDESC2 = tc::idesc_f16(128, N2, 0, 0, 1);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sP1 = smem;
  uint8_t* sP2 = sP1 + C::P1_BYTES;
  uint8_t* sX = sP2 + C::P2_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + size_t(S) * C::X_BYTES);
  uint64_t* xfull = bars;            // [S] TMA -> MMA
  uint64_t* xempty = bars + S;       // [S] stage-1 MMA commit -> TMA
  uint64_t* pfull = bars + 2 * S;    // P1, P2 landed
  uint64_t* d1full = pfull + 1;      // stage-1 commit -> epilogue
  uint64_t* a2full = d1full + 1;     // epilogue (4 warps) -> stage-2 MMA
  uint64_t* d2full = a2full + 1;     // stage-2 commit -> epilogue
  uint64_t* d2empty = d2full + 1;    // epilogue (4 warps) -> next stage-2 MMA
  uint64_t* peready = d2empty + 1;   // [2] stage-1 group -> stage-2 group: token's prescale exponent
  __shared__ float red[16];          // [group][2 parities][4 warps]
  __shared__ int pe_buf[2];          // prescale exponent of token k, slot k % 2
  __shared__ uint32_t tmem_slot[1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int my_tiles = T > int64_t(blockIdx.x) ? int((T - 1 - int64_t(blockIdx.x)) / gridDim.x) + 1 : 0;
  auto issue_x = [&](int k) {
    const int s = k % S;
    tc::mbar_wait(&xempty[s], ((k / S) & 1) ^ 1);
    tc::mbar_expect_tx(&xfull[s], C::X_BYTES);
    const int t = int(blockIdx.x) + k * int(gridDim.x);
    uint8_t* dst = sX + size_t(s) * C::X_BYTES;
#pragma unroll
    for (int b = 0; b < C::JB; ++b) tc::tma_load_3d(dst + b * N1 * 128, &tmX, &xfull[s], b * 64, 0, t);
  };
  const int prefill = my_tiles < S ? my_tiles : S;
  if (threadIdx.x == 0) {
    tc::tma_prefetch_desc(&tmX);
    tc::tma_prefetch_desc(&tmP1);
    tc::tma_prefetch_desc(&tmP2);
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&xfull[s], 1);
      tc::mbar_init(&xempty[s], 1);
    }
    tc::mbar_init(pfull, 1);
    tc::mbar_init(d1full, 1);
    tc::mbar_init(a2full, 4);
    tc::mbar_init(d2full, 1);
    tc::mbar_init(d2empty, 4);
    tc::mbar_init(&peready[0], 4);
    tc::mbar_init(&peready[1], 4);
    tc::fence_barrier_init();
    auto load_p = [&] {                // PDL (fq_internal.h): before the wait unless the predecessor writes them
      tc::mbar_expect_tx(pfull, C::P1_BYTES + C::P2_BYTES);
      for (int a = 0; a < 2; ++a) tc::tma_load_2d(sP1 + a * N1 * 128, &tmP1, pfull, a * 64, 0);
      for (int b = 0; b < C::JB; ++b) tc::tma_load_2d(sP2 + b * N2 * 128, &tmP2, pfull, b * 64, 0);
    };
    if (pdl & PDL_P) load_p();
    if ((pdl & (PDL_P | PDL_X)) != (PDL_P | PDL_X)) tc::griddep_wait();
    if (!(pdl & PDL_P)) load_p();
    for (int k = 0; k < prefill; ++k) issue_x(k);
  }
  if (warp == 2) {
    tc::tmem_alloc(tmem_slot, 512);
    if (lane == 0) {
      tc::griddep_wait();              // dependents launch only after this kernel's wait returned
      tc::griddep_launch();
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  tc::mbar_wait(pfull, 0);
  // stage 2 runs in fp16 (R9): a bf16 P2 becomes fp16 P2 * 2^e2 in place (no overflow); the
  // statistics divide 2^e2 out exactly
  float inv_p2 = 1.0f;
  if constexpr (BF16) {
    __shared__ uint32_t p2max;
    inv_p2 = exp2i(-bf16_to_f16_pow2(sP2, C::P2_BYTES / 2, &p2max));
  }
  __syncthreads();

  if (warp == 0) {
    // ================================ TMA producer ================================
    if (lane == 0)
      for (int k = prefill; k < my_tiles; ++k) issue_x(k);
    __syncwarp();
  } else if (warp == 1) {
    // ================================ MMA issuer ================================
    // Stage 1 of token k overwrites region R1, the A operand of stage 2 of token k-1: it is
    // issued only after that stage-2 MMA has completed (its commit), not merely been issued.
    if (lane == 0) {
      const uint32_t p1a = smem_u32(sP1), p2a = smem_u32(sP2);
      for (int k = 0; k < my_tiles; ++k) {
        const int s = k % S;
        if (k > 0) tc::mbar_wait(d2full, (k - 1) & 1);
        tc::mbar_wait(&xfull[s], (k / S) & 1);
        tc::fence_after();
        const uint32_t xs = smem_u32(sX + size_t(s) * C::X_BYTES);
#pragma unroll
        for (int kk = 0; kk < N1 / 16; ++kk)
          tc::mma_ss<false>(tmem, tc::sdesc_sw128(p1a + kk * 2048, N1 * 128, 1024),
                            tc::sdesc_sw128(xs + kk * 2048, N1 * 128, 1024), IDESC1, kk > 0);
        tc::mma_commit(&xempty[s]);
        tc::mma_commit(d1full);
        tc::mbar_wait(a2full, k & 1);                   // fp16 W_t written in place
        if (k > 0) tc::mbar_wait(d2empty, (k - 1) & 1); // D2 of token k-1 read out
        tc::fence_after();
#pragma unroll
        for (int kk = 0; kk < N2 / 16; ++kk)
          tc::mma_ts<false>(tmem + uint32_t(R2), tmem + uint32_t(kk * 8),
                            tc::sdesc_sw128(p2a + kk * 2048, N2 * 128, 1024), IDESC2, kk > 0);
        tc::mma_commit(d2full);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ================================ epilogues ================================
    // Round 2c: warps 4-7 run the stage-1 epilogue of every token, warps 8-11 the stage-2
    // epilogue, so the stage-1 epilogue of token k+1 overlaps the stage-2 epilogue of token k
    // (one group doing both serialised them: ~4.4 us per token and SM at 128 x 224).
    const int grp = (warp - 4) >> 2;                     // 0: stage 1, 1: stage 2
    const int qd = warp & 3, i = qd * 32 + lane;        // TMEM lane == row i of the token
    const uint32_t lane_base = tmem + (uint32_t(qd * 32) << 16);
    float* redg = red + grp * 8;
    int rp = 0;
    auto exchange = [&](float m) {                       // max over the token's 128 rows (m >= 0)
      m = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(m)));
      if (lane == 0) redg[rp * 4 + qd] = m;
      named_bar_sync(1 + grp, 128);
      const float r = fmaxf(fmaxf(redg[rp * 4 + 0], redg[rp * 4 + 1]), fmaxf(redg[rp * 4 + 2], redg[rp * 4 + 3]));
      rp ^= 1;
      return r;
    };
    constexpr int QROW = N2 / 2, QTOK = N1 * N2 / 2;
    bool waited = (pdl & PDL_OUT) != 0;                  // outputs before the wait only if allowed
    for (int k = 0; k < my_tiles; ++k) {
      const int64_t t = int64_t(blockIdx.x) + int64_t(k) * gridDim.x;
      const uint32_t ph = k & 1;
      if (grp == 0) {
        // -------- stage-1 epilogue: D1 (fp32) -> prescaled fp16 A operand, in place --------
        tc::mbar_wait(d1full, ph);
        tc::fence_after();
        float m1 = 0.f;
#pragma unroll 1
        for (int c = 0; c < N2; c += 32) {
          uint32_t v[32];
          tmem_ld32c(lane_base + uint32_t(c), v);
#pragma unroll
          for (int e = 0; e < 32; e += 2) m1 = max3f(m1, fabsf(__uint_as_float(v[e])), fabsf(__uint_as_float(v[e + 1])));
        }
        const int pe = prescale_exp(exchange(m1));
        const float pre = exp2i(pe);
        // chunk c (columns [c, c+32)) becomes A columns [c/2, c/2 + 16): only columns already read
#pragma unroll 1
        for (int c = 0; c < N2; c += 32) {
          uint32_t v[32], h[16];
          tmem_ld32c(lane_base + uint32_t(c), v);
#pragma unroll
          for (int e = 0; e < 16; ++e)
            h[e] = pack_half2(__uint_as_float(v[2 * e]) * pre, __uint_as_float(v[2 * e + 1]) * pre);
          tmem_st16(lane_base + uint32_t(c / 2), h);
        }
        tc::tmem_st_wait();
        tc::fence_before();
        if (i == 0) pe_buf[k & 1] = pe;                  // for the stage-2 group (peready below)
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(a2full);
          tc::mbar_arrive(&peready[k & 1]);              // two slots: this group is < 2 tokens ahead
        }
        continue;
      }
      // -------- stage-2 epilogue: absmax, clip, quantize, pack, store --------
      tc::mbar_wait(d2full, ph);
      tc::mbar_wait(&peready[k & 1], (k >> 1) & 1);
      tc::fence_after();
      const int pe = *static_cast<volatile int*>(&pe_buf[k & 1]);
      const uint32_t d2 = lane_base + uint32_t(R2);
      float m2 = 0.f, hi2 = 0.f, lo2 = 0.f;
#pragma unroll 1
      for (int c = 0; c < N2; c += 32) {
        uint32_t v[32];
        tmem_ld32c(d2 + uint32_t(c), v);
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float a0 = __uint_as_float(v[e]), a1 = __uint_as_float(v[e + 1]);
          if constexpr (ASYM) {
            hi2 = max3f(hi2, a0, a1);
            lo2 = max3f(lo2, -a0, -a1);
          } else {
            m2 = max3f(m2, fabsf(a0), fabsf(a1));
          }
        }
      }
      float mp, lop = 0.f;
      if constexpr (ASYM) {
        const float hip = exchange(hi2);
        lop = exchange(lo2);
        mp = hip + lop;
      } else {
        mp = exchange(m2);
      }
      const float inv_pre = exp2i(-pe);
      // same FFMA.SAT quantizer as the general kernel (fq_tq_tc05.cu): clamp on the FMA pipe,
      // round-half-even by the magic-number add, nibble = low mantissa bits
      float c15, B15, zq = 0.f;
      if constexpr (ASYM) {
        const float sp = alpha * mp * (1.0f / 15.0f);
        zq = sp > 0.f ? rintf(__fdiv_rn(alpha * lop, sp)) : 0.f;
        c15 = sp > 0.f ? __frcp_rn(alpha * mp) : 0.f;
        B15 = zq * (1.0f / 15.0f);
      } else {
        c15 = mp > 0.f ? __fdividef(7.0f / 15.0f, alpha * mp) : 0.f;
        B15 = 8.0f / 15.0f;
      }
      uint8_t* qrow = q + t * QTOK + i * QROW;
      if (!waited) {
        tc::griddep_wait();
        waited = true;
      }
#pragma unroll 1
      for (int c = 0; c < N2; c += 32) {
        uint32_t v[32];
        tmem_ld32c(d2 + uint32_t(c), v);
        uint32_t w[4];
#pragma unroll
        for (int c8 = 0; c8 < 4; ++c8) {
          float z[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            z[e] = fmaf(fma_sat(__uint_as_float(v[8 * c8 + e]), c15, B15), 15.0f, MAGIC - 8.0f);
          w[c8] = pack8(z);
        }
        *reinterpret_cast<uint4*>(qrow + c / 2) = make_uint4(w[0], w[1], w[2], w[3]);
        if constexpr (WRITE_Y) {
          float2* yd = reinterpret_cast<float2*>(y_out + t * (N1 * N2) + i * N2 + c);
#pragma unroll
          for (int e = 0; e < 16; ++e)
            yd[e] = make_float2(__uint_as_float(v[2 * e]) * inv_pre * inv_p2,
                                __uint_as_float(v[2 * e + 1]) * inv_pre * inv_p2);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(d2empty);
      if (i == 0) {
        if constexpr (ASYM) {
          scale[t] = mp > 0.f ? alpha * (mp * inv_pre * inv_p2) / 15.0f : 1.0f;
          zero[t] = int8_t(int(zq) - 8);
        } else {
          scale[t] = mp > 0.f ? alpha * (mp * inv_pre * inv_p2) / 7.0f : 1.0f;
        }
      }
    }
  }

  tc::fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

template <int N2, bool BF16, bool WRITE_Y, bool ASYM>
static cudaError_t launch(const TQArgs& a) {
  using C = Cfg<N2>;
  auto kern = tq_wide_kernel<N2, BF16, WRITE_Y, ASYM>;
  static std::atomic<uint64_t> attr_done{0};   // devices configured for this kernel
  if (cudaError_t e = ensure_smem_attr(kern, int(C::SMEM), attr_done); e != cudaSuccess) return e;
  CUtensorMap mx, m1, m2;
  {
    const uint64_t dims[3] = {uint64_t(N2), uint64_t(N1), uint64_t(a.T)};
    const uint64_t strides[2] = {uint64_t(N2) * 2, uint64_t(a.ldx) * 2};
    const uint32_t box[3] = {64, uint32_t(N1), 1};
    if (!tmap_encode(&mx, a.x, 2, 3, dims, strides, box, TMAP_SW128)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {uint64_t(N1), uint64_t(N1)};
    const uint64_t strides[1] = {uint64_t(N1) * 2};
    const uint32_t box[2] = {64, uint32_t(N1)};
    if (!tmap_encode(&m1, a.p1, 2, 2, dims, strides, box, TMAP_SW128)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {uint64_t(N2), uint64_t(N2)};
    const uint64_t strides[1] = {uint64_t(N2) * 2};
    const uint32_t box[2] = {64, uint32_t(N2)};
    if (!tmap_encode(&m2, a.p2, 2, 2, dims, strides, box, TMAP_SW128)) return cudaErrorInvalidValue;
  }
  const int grid = int(std::min<int64_t>(a.T, num_sms()));
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(THREADS), C::SMEM, a.stream, 1, mx, m1, m2, a.T, a.alpha, a.q,
                             a.scale, a.y, a.zero, a.pdl);
  count_launch();
  return e;
}

template <int N2>
static cudaError_t dispatch(const TQArgs& a) {
  if (a.zero) return a.bf16 ? launch<N2, true, false, true>(a) : launch<N2, false, false, true>(a);
  if (a.bf16) return a.y ? launch<N2, true, true, false>(a) : launch<N2, true, false, false>(a);
  return a.y ? launch<N2, false, true, false>(a) : launch<N2, false, false, false>(a);
}

}  // namespace tqw

bool tq_wide_supported(const TQArgs& a) {
  const bool shape = a.n1 == 128 && (a.n2 == 160 || a.n2 == 192 || a.n2 == 224 || a.n2 == 256);
  const bool al = ((reinterpret_cast<uintptr_t>(a.x) | reinterpret_cast<uintptr_t>(a.p1) |
                    reinterpret_cast<uintptr_t>(a.p2) | reinterpret_cast<uintptr_t>(a.q)) & 15u) == 0 &&
                  (a.ldx * 2) % 16 == 0 && a.T < (int64_t(1) << 31);
  return shape && al && tmap_available();
}

cudaError_t tq_wide_launch(const TQArgs& a) {
  switch (a.n2) {
    case 160: return tqw::dispatch<160>(a);
    case 192: return tqw::dispatch<192>(a);
    case 224: return tqw::dispatch<224>(a);
    case 256: return tqw::dispatch<256>(a);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fq
