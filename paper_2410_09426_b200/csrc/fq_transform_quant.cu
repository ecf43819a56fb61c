// fq_transform_quant.cu -- fused Kronecker transform + clip + per-token INT4 quantize + pack.
//
// Computes, per token t (Eq.3 activation factor):
//   V_t = reshape(x_t, n1, n2) (row-major)      W_t = P1^T V_t      Y_t = W_t P2
//   s_t = alpha max|Y_t| / 7 (1 if Y_t == 0)     q = clamp(rint(Y_t / s_t), -8, 7), packed
//
// Tensor-core kernel (n1 % 16 == 0, n2 % 16 == 0): one "team" of n1/16 warps per token;
// warp w owns rows [16w, 16w+16) of the token tile.  Stage 1 (W = P1^T V) is a warp MMA
// with P1^T as the A operand held in registers for the kernel's lifetime and V read from
// shared memory (cp.async double buffer, rows padded by 16 B so ldmatrix is conflict-free).
// Its fp32 accumulator fragment is re-used in registers as the A operand of stage 2
// (Y = W P2) -- the intermediate never touches shared or global memory.  Before that re-use
// each warp multiplies its strip by an exact power of two so the fp16 operand can neither
// overflow nor underflow (codes are per-row scale invariant; the factor is divided out of Y
// exactly).  The order P1^T first matches the paper's kernel (App. B.3).
//
// CUDA-core kernel: any n1, n2 (the tiny-shape path of the north_star), fp32 throughout.
#include <cstdint>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"

namespace fq {

// ============================================================================================
// Tensor-core (mma.sync) kernel
// ============================================================================================
template <int N1, int N2, bool BF16, bool WRITE_Y, int TEAMS, int NBUF>
struct TQCfg {
  static constexpr int WARPS = N1 / 16;          // warps per token team
  static constexpr int TEAM_THREADS = WARPS * 32;
  static constexpr int THREADS = TEAM_THREADS * TEAMS;
  static constexpr int XPITCH = N2 + 8;          // halves per smem row (16 B pad)
  static constexpr int X_ELEMS = N1 * XPITCH;    // one token tile
  static constexpr int P2_ELEMS = N2 * XPITCH;
  static constexpr int QBYTES = N1 * N2 / 2;     // packed codes per token
  // smem: P2 | per team: X[NBUF] | staging codes | strip maxima (each team 128-B aligned)
  static constexpr size_t P2_BYTES = (size_t(P2_ELEMS) * 2 + 127) / 128 * 128;
  static constexpr size_t QOFF = size_t(NBUF * X_ELEMS) * 2;
  static constexpr size_t MAXOFF = QOFF + (QBYTES + 15) / 16 * 16;
  static constexpr size_t TEAM_BYTES = (MAXOFF + WARPS * 4 + 127) / 128 * 128;
  static constexpr size_t SMEM = P2_BYTES + size_t(TEAMS) * TEAM_BYTES;
};

// IDENT2: P2 = I (the online o_proj transform P_o (a x a) is applied across
// the heads of the attention output, identity inside each head), stage 2 is skipped and the fp32
// stage-1 accumulators are quantized directly (p2 is not read).
template <int N1, int N2, bool BF16, bool WRITE_Y, int TEAMS, int NBUF, bool IDENT2 = false>
__global__ void __launch_bounds__(TQCfg<N1, N2, BF16, WRITE_Y, TEAMS, NBUF>::THREADS, 1)
tq_mma_kernel(const uint16_t* __restrict__ x, int64_t T, int64_t ldx,
              const uint16_t* __restrict__ p1, const uint16_t* __restrict__ p2, float alpha,
              uint8_t* __restrict__ q, float* __restrict__ scale, float* __restrict__ y_out) {
  using C = TQCfg<N1, N2, BF16, WRITE_Y, TEAMS, NBUF>;
  constexpr int WARPS = C::WARPS;
  constexpr int KT1 = N1 / 16;   // k-tiles of stage 1 (reduction over i1)
  constexpr int NT = N2 / 8;     // n-tiles (columns j2)
  constexpr int KT2 = N2 / 16;   // k-tiles of stage 2 (reduction over j2)
  static_assert(N1 % 16 == 0 && N2 % 16 == 0, "tensor-core path needs multiples of 16");

  extern __shared__ __align__(128) uint8_t smem[];
  uint16_t* sP2 = reinterpret_cast<uint16_t*>(smem);
  const int team = threadIdx.x / C::TEAM_THREADS;
  const int tt = threadIdx.x % C::TEAM_THREADS;       // thread within team
  const int warp = tt / 32;
  const int lane = threadIdx.x % 32;
  const int g = lane >> 2, qd = lane & 3;
  uint8_t* team_base = smem + C::P2_BYTES + size_t(team) * C::TEAM_BYTES;
  uint16_t* sX = reinterpret_cast<uint16_t*>(team_base);
  uint8_t* sQ = team_base + C::QOFF;
  float* sMax = reinterpret_cast<float*>(team_base + C::MAXOFF);

  // ---- P2 -> smem (whole CTA), padded rows, always as fp16: stage 2 runs in fp16 so the
  //      re-fed intermediate keeps an 11-bit mantissa (a bf16 intermediate fails the code
  //      parity bar).  bf16 -> fp16 is exact for normal-range entries. ----
  //      A bf16 P2 is scaled by 2^e2 into fp16 range first (no entry overflows; 2^-e2 is
  //      applied to the result exactly). ----
  float p2_sc = 1.f, p2_inv = 1.f;
  if constexpr (BF16 && !IDENT2) {
    __shared__ uint32_t p2max;
    if (threadIdx.x == 0) p2max = 0u;
    __syncthreads();
    uint32_t m = 0;
    for (int i = threadIdx.x; i < N2 * N2; i += C::THREADS) m = max(m, (uint32_t(p2[i]) << 16) & 0x7FFFFFFFu);
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) atomicMax(&p2max, m);
    __syncthreads();
    const int e2 = p2_scale_exp(p2max);
    p2_sc = __int_as_float((127 + e2) << 23);
    p2_inv = __int_as_float((127 - e2) << 23);
  }
  for (int i = threadIdx.x; i < (IDENT2 ? 0 : N2 * N2); i += C::THREADS) {
    const int r = i / N2, c = i % N2;
    uint16_t v = p2[i];
    if constexpr (BF16) {
      __half h = __float2half_rn(__uint_as_float(uint32_t(v) << 16) * p2_sc);
      v = *reinterpret_cast<uint16_t*>(&h);
    }
    sP2[r * C::XPITCH + c] = v;
  }
  // ---- P1^T strip -> registers: A[r][c] = P1^T[16w + r][16kt + c] = P1[16kt + c][16w + r] ----
  uint32_t a1[KT1][4];
#pragma unroll
  for (int kt = 0; kt < KT1; ++kt) {
    const int r0 = 16 * warp + g, c0 = 16 * kt + 2 * qd;
    auto at = [&](int r, int c) -> uint32_t { return p1[size_t(c) * N1 + r]; };
    a1[kt][0] = at(r0, c0) | (at(r0, c0 + 1) << 16);
    a1[kt][1] = at(r0 + 8, c0) | (at(r0 + 8, c0 + 1) << 16);
    a1[kt][2] = at(r0, c0 + 8) | (at(r0, c0 + 9) << 16);
    a1[kt][3] = at(r0 + 8, c0 + 8) | (at(r0 + 8, c0 + 9) << 16);
  }

  const int64_t team_stride = int64_t(gridDim.x) * TEAMS;
  int64_t t = int64_t(blockIdx.x) * TEAMS + team;
  const int bar_id = 1 + team;

  auto load_x = [&](int64_t tok, int buf) {
    uint16_t* dst = sX + buf * C::X_ELEMS;
    const bool ok = tok < T;
    const uint16_t* src = x + (ok ? tok : 0) * ldx;
    constexpr int CHUNKS = N1 * N2 / 8;  // 16-byte chunks
    for (int i = tt; i < CHUNKS; i += C::TEAM_THREADS) {
      const int r = i / (N2 / 8), c = (i % (N2 / 8)) * 8;
      cp_async16(dst + r * C::XPITCH + c, src + r * N2 + c, ok);
    }
    cp_async_commit();
  };

  if constexpr (NBUF == 2) load_x(t, 0);
  __syncthreads();  // P2 visible
  int buf = 0;
  for (; t < T; t += team_stride) {
    if constexpr (NBUF == 2) {
      load_x(t + team_stride, buf ^ 1);   // prefetch next token (zero-filled past T)
      cp_async_wait<1>();
    } else {
      load_x(t, 0);
      cp_async_wait<0>();
    }
    named_bar_sync(bar_id, C::TEAM_THREADS);
    const uint16_t* cX = sX + buf * C::X_ELEMS;

    // ---------------- stage 1: W = P1^T V (rows of this warp's strip) ----------------
    float acc[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
#pragma unroll
    for (int kt = 0; kt < KT1; ++kt) {
#pragma unroll
      for (int n = 0; n < NT; n += 2) {
        const int row = 16 * kt + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = 8 * n + (lane >> 4) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_trans(b0, b1, b2, b3, smem_u32(cX + row * C::XPITCH + col));
        mma_16816<BF16>(acc[n], a1[kt], b0, b1);
        mma_16816<BF16>(acc[n + 1], a1[kt], b2, b3);
      }
    }
    float m = 0.f, inv_pre = 1.f;
    if constexpr (!IDENT2) {
    // ---------------- exact power-of-two prescale of the strip ----------------
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) m = fmaxf(m, fabsf(acc[n][e]));
    m = warp_max(m);
    // choose 2^k with m * 2^k in [2^14, 2^15): safe for fp16 (max 65504) and far from
    // its subnormals.
    float pre = 1.f;
    if (m > 0.f) {
      const int e = 14 - ilogbf(m);
      pre = ldexpf(1.f, e);
      inv_pre = ldexpf(1.f, -e);
    }
    uint32_t a2[KT2][4];   // fp16 A fragments of the prescaled intermediate
#pragma unroll
    for (int kt = 0; kt < KT2; ++kt) {
      const float* c0 = acc[2 * kt];
      const float* c1 = acc[2 * kt + 1];
      a2[kt][0] = pack_half2(c0[0] * pre, c0[1] * pre);
      a2[kt][1] = pack_half2(c0[2] * pre, c0[3] * pre);
      a2[kt][2] = pack_half2(c1[0] * pre, c1[1] * pre);
      a2[kt][3] = pack_half2(c1[2] * pre, c1[3] * pre);
    }
    // ---------------- stage 2: Y = W P2 ----------------
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
#pragma unroll
    for (int kt = 0; kt < KT2; ++kt) {
#pragma unroll
      for (int n = 0; n < NT; n += 2) {
        const int row = 16 * kt + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = 8 * n + (lane >> 4) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_trans(b0, b1, b2, b3, smem_u32(sP2 + row * C::XPITCH + col));
        mma_16816<false>(acc[n], a2[kt], b0, b1);
        mma_16816<false>(acc[n + 1], a2[kt], b2, b3);
      }
    }
    }  // !IDENT2
    // ---------------- per-token absmax (clip applied after the transform) ----------------
    m = 0.f;
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[n][e] = acc[n][e] * inv_pre * p2_inv;
        m = fmaxf(m, fabsf(acc[n][e]));
      }
    m = warp_max(m);
    if (lane == 0) sMax[warp] = m;
    named_bar_sync(bar_id, C::TEAM_THREADS);
    m = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) m = fmaxf(m, sMax[w]);
    const float s = (m > 0.f) ? alpha * m / 7.0f : 1.0f;
    const float inv_s = (m > 0.f) ? 7.0f / (alpha * m) : 0.0f;
    if constexpr (WRITE_Y) {
      if (t < T) {
        float* yt = y_out + t * int64_t(N1) * N2;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int r = 16 * warp + g, c = 8 * n + 2 * qd;
          *reinterpret_cast<float2*>(yt + r * N2 + c) = make_float2(acc[n][0], acc[n][1]);
          *reinterpret_cast<float2*>(yt + (r + 8) * N2 + c) = make_float2(acc[n][2], acc[n][3]);
        }
      }
    }
    // ---------------- quantize + pack into the staging buffer ----------------
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      int c[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        int v = __float2int_rn(acc[n][e] * inv_s);   // round half to even
        c[e] = min(7, max(-8, v));
      }
      const int r = 16 * warp + g;
      const int byte = 4 * n + qd;  // column pair (8n + 2qd, +1) -> byte 4n + qd of the row
      sQ[r * (N2 / 2) + byte] = uint8_t((c[0] & 15) | ((c[1] & 15) << 4));
      sQ[(r + 8) * (N2 / 2) + byte] = uint8_t((c[2] & 15) | ((c[3] & 15) << 4));
    }
    named_bar_sync(bar_id, C::TEAM_THREADS);
    if (t < T) {
      uint8_t* qt = q + t * int64_t(C::QBYTES);
      for (int i = tt; i < C::QBYTES / 16; i += C::TEAM_THREADS)
        *reinterpret_cast<uint4*>(qt + 16 * i) = *reinterpret_cast<const uint4*>(sQ + 16 * i);
      if (tt == 0) scale[t] = s;
    }
    if constexpr (NBUF == 2) buf ^= 1;
  }
  cp_async_wait<0>();
}

// ============================================================================================
// CUDA-core kernel (any n1, n2): one CTA per token, fp32 throughout.
// ============================================================================================
template <typename TIn, bool WRITE_Y>
__global__ void __launch_bounds__(256)
tq_simt_kernel(const TIn* __restrict__ x, int64_t T, int64_t ldx, int n1, int n2,
               const TIn* __restrict__ p1, const TIn* __restrict__ p2, float alpha,
               uint8_t* __restrict__ q, float* __restrict__ scale, float* __restrict__ y_out,
               int8_t* __restrict__ zero) {
  extern __shared__ __align__(16) float fsm[];
  const int n = n1 * n2;
  float* v = fsm;        // [n1][n2]
  float* z = fsm + n;    // [n1][n2]  (z = V P2)
  __shared__ float red[32];
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const TIn* xt = x + t * ldx;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = to_f32(xt[i]);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int r = i / n2, c = i % n2;
      float a = 0.f;
      for (int k = 0; k < n2; ++k) a = fmaf(v[r * n2 + k], to_f32(p2[k * n2 + c]), a);
      z[i] = a;
    }
    __syncthreads();
    // sym: m = max |y|;  asym (zero != nullptr): hi = max(max y, 0), lo = max(-min y, 0)
    float m = 0.f, hi = 0.f, lo = 0.f;
    // y[r][c] = sum_k P1[k][r] z[k][c]; each thread owns elements i = tid + j*blockDim
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int r = i / n2, c = i % n2;
      float a = 0.f;
      for (int k = 0; k < n1; ++k) a = fmaf(to_f32(p1[k * n1 + r]), z[k * n2 + c], a);
      v[i] = a;  // V no longer needed: reuse for Y
      m = fmaxf(m, fabsf(a));
      hi = fmaxf(hi, a);
      lo = fmaxf(lo, -a);
    }
    auto block_max = [&](float x) {
      x = warp_max(x);
      __syncthreads();
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
      __syncthreads();
      if (threadIdx.x < 32) {
        float mm = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.f;
        mm = warp_max(mm);
        if (threadIdx.x == 0) red[0] = mm;
      }
      __syncthreads();
      return red[0];
    };
    if (WRITE_Y)
      for (int i = threadIdx.x; i < n; i += blockDim.x) y_out[t * n + i] = v[i];
    if (zero == nullptr) {
      m = block_max(m);
      const float s = (m > 0.f) ? alpha * m / 7.0f : 1.0f;
      const float inv_s = (m > 0.f) ? 7.0f / (alpha * m) : 0.0f;
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        const int c0 = min(7, max(-8, __float2int_rn(v[2 * i] * inv_s)));
        const int c1 = min(7, max(-8, __float2int_rn(v[2 * i + 1] * inv_s)));
        q[t * (n / 2) + i] = uint8_t((c0 & 15) | ((c1 & 15) << 4));
      }
      if (threadIdx.x == 0) scale[t] = s;
    } else {                                           // asymmetric (reading R19)
      hi = block_max(hi);
      lo = block_max(lo);
      const float range = alpha * (hi + lo);           // (max(alpha max y, 0) - min(alpha min y, 0))
      const float s = range > 0.f ? range / 15.0f : 1.0f;
      const int zq = range > 0.f ? __float2int_rn(alpha * lo / s) : 0;
      const float inv_s = range > 0.f ? 1.0f / s : 0.0f;
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        const int c0 = min(15, max(0, __float2int_rn(v[2 * i] * inv_s) + zq)) - 8;
        const int c1 = min(15, max(0, __float2int_rn(v[2 * i + 1] * inv_s) + zq)) - 8;
        q[t * (n / 2) + i] = uint8_t((c0 & 15) | ((c1 & 15) << 4));
      }
      if (threadIdx.x == 0) {
        scale[t] = s;
        zero[t] = int8_t(zq - 8);
      }
    }
    __syncthreads();
  }
}

// ============================================================================================
// Launchers
// ============================================================================================
template <int N1, int N2, bool BF16, bool WRITE_Y, int TEAMS, int NBUF, bool IDENT2 = false>
static cudaError_t launch_mma(const TQArgs& a) {
  using C = TQCfg<N1, N2, BF16, WRITE_Y, TEAMS, NBUF>;
  auto kern = tq_mma_kernel<N1, N2, BF16, WRITE_Y, TEAMS, NBUF, IDENT2>;
  static std::atomic<uint64_t> attr_done{0};   // devices configured for this kernel
  if (cudaError_t e = ensure_smem_attr(kern, int(C::SMEM), attr_done); e != cudaSuccess) return e;
  const int64_t teams_needed = (a.T + TEAMS - 1) / TEAMS;
  int blocks_per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, C::THREADS, C::SMEM);
  if (blocks_per_sm < 1) blocks_per_sm = 1;
  const int64_t grid = std::min<int64_t>(teams_needed, int64_t(num_sms()) * blocks_per_sm);
  kern<<<dim3(unsigned(grid)), C::THREADS, C::SMEM, a.stream>>>(
      static_cast<const uint16_t*>(a.x), a.T, a.ldx, static_cast<const uint16_t*>(a.p1),
      static_cast<const uint16_t*>(a.p2), a.alpha, a.q, a.scale, a.y);
  count_launch();
  return cudaGetLastError();
}

template <int N1, int N2, int TEAMS, int NBUF>
static cudaError_t dispatch_mma(const TQArgs& a) {
  if (a.bf16)
    return a.y ? launch_mma<N1, N2, true, true, TEAMS, NBUF>(a) : launch_mma<N1, N2, true, false, TEAMS, NBUF>(a);
  return a.y ? launch_mma<N1, N2, false, true, TEAMS, NBUF>(a) : launch_mma<N1, N2, false, false, TEAMS, NBUF>(a);
}

template <int N1, int N2, int TEAMS, int NBUF>
static cudaError_t dispatch_mma_ident(const TQArgs& a) {
  if (a.bf16)
    return a.y ? launch_mma<N1, N2, true, true, TEAMS, NBUF, true>(a) : launch_mma<N1, N2, true, false, TEAMS, NBUF, true>(a);
  return a.y ? launch_mma<N1, N2, false, true, TEAMS, NBUF, true>(a) : launch_mma<N1, N2, false, false, TEAMS, NBUF, true>(a);
}

bool tq_ident2_supported(int n1, int n2) { return n2 == 128 && (n1 == 32 || n1 == 64); }

// P2 = I (p2 == nullptr): the paper's online o_proj transform P_o (a x a) (x) I_{d_head}
// (PAPER.md:297, 726), a heads of d_head = 128 (LLaMA-2-7B / LLaMA-3-8B: 32, LLaMA-3-70B: 64).
cudaError_t tq_ident2_launch(const TQArgs& a) {
  if (a.n1 == 32 && a.n2 == 128) return dispatch_mma_ident<32, 128, 4, 2>(a);
  if (a.n1 == 64 && a.n2 == 128) return dispatch_mma_ident<64, 128, 2, 2>(a);
  return cudaErrorInvalidValue;
}

template <typename TIn>
static cudaError_t launch_simt(const TQArgs& a) {
  const int n = a.n1 * a.n2;
  const size_t smem = size_t(2) * n * sizeof(float);
  auto kern = a.y ? tq_simt_kernel<TIn, true> : tq_simt_kernel<TIn, false>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
  }
  const int64_t grid = std::min<int64_t>(a.T, int64_t(num_sms()) * 8);
  kern<<<dim3(unsigned(grid)), 256, smem, a.stream>>>(
      static_cast<const TIn*>(a.x), a.T, a.ldx, a.n1, a.n2, static_cast<const TIn*>(a.p1),
      static_cast<const TIn*>(a.p2), a.alpha, a.q, a.scale, a.y, a.zero);
  count_launch();
  return cudaGetLastError();
}

bool tq_simt_supported(int n1, int n2) {
  return size_t(2) * n1 * n2 * sizeof(float) <= 200 * 1024;
}

bool tq_mma_supported(int n1, int n2) {
  // the configs' shapes plus the decompositions of 4096 and 14336 that scripts/fig5_sweep.py
  // measures (Fig. 5), so every n1 x n2 with 16 | n1, n2 runs on tensor cores
  return (n1 == 16 && n2 == 32) || (n1 == 64 && n2 == 64) || (n1 == 64 && n2 == 128) ||
         (n1 == 112 && n2 == 128) || (n1 == 128 && n2 == 224) || (n1 == 16 && n2 == 256) ||
         (n1 == 32 && n2 == 128) || (n1 == 128 && n2 == 32) || (n1 == 256 && n2 == 16) ||
         (n1 == 64 && n2 == 224) || (n1 == 128 && n2 == 112) || (n1 == 224 && n2 == 64);
}

cudaError_t tq_mma_launch(const TQArgs& a) {
  if (a.n1 == 16 && a.n2 == 32) return dispatch_mma<16, 32, 8, 2>(a);
  if (a.n1 == 64 && a.n2 == 64) return dispatch_mma<64, 64, 2, 2>(a);
  if (a.n1 == 64 && a.n2 == 128) return dispatch_mma<64, 128, 2, 2>(a);
  if (a.n1 == 112 && a.n2 == 128) return dispatch_mma<112, 128, 1, 2>(a);
  if (a.n1 == 128 && a.n2 == 224) return dispatch_mma<128, 224, 1, 1>(a);
  if (a.n1 == 16 && a.n2 == 256) return dispatch_mma<16, 256, 4, 2>(a);
  if (a.n1 == 32 && a.n2 == 128) return dispatch_mma<32, 128, 4, 2>(a);
  if (a.n1 == 128 && a.n2 == 32) return dispatch_mma<128, 32, 2, 2>(a);
  if (a.n1 == 256 && a.n2 == 16) return dispatch_mma<256, 16, 2, 2>(a);
  if (a.n1 == 64 && a.n2 == 224) return dispatch_mma<64, 224, 2, 1>(a);
  if (a.n1 == 128 && a.n2 == 112) return dispatch_mma<128, 112, 2, 2>(a);
  if (a.n1 == 224 && a.n2 == 64) return dispatch_mma<224, 64, 1, 2>(a);
  return cudaErrorInvalidValue;
}

cudaError_t tq_simt_launch(const TQArgs& a) {
  return a.bf16 ? launch_simt<__nv_bfloat16>(a) : launch_simt<__half>(a);
}

// impl 0: tcgen05 kernel where supported; tiny tiles (n <= 4096, e.g. 16 x 32) on CUDA cores in
//         fp32 (the north_star's "warp-level FMAs where n1 and n2 are tiny": no fp16 intermediate,
//         so no tie flips); the mma.sync kernel for the remaining instantiated shapes (128 x 224).
// impl 1: mma.sync where instantiated, else CUDA cores;  impl 2: CUDA cores.
bool tq_asym_supported(const TQArgs& a) {
  return (tq_impl() == 0 && (tq_tc05_supported(a) || tq_wide_supported(a))) || tq_simt_supported(a.n1, a.n2);
}

// true when transform_quant_launch has a kernel for this call (else the ABI returns FQ_ENOTSUP
// instead of a launch that cannot fit its shared memory)
bool tq_kernel_available(const TQArgs& a) {
  const int impl = tq_impl();
  if (a.p2 == nullptr)                             // P2 = I: tcgen05 (sym/asym), else mma.sync (sym)
    return (impl == 0 && tq_tc05_supported(a)) || (!a.zero && tq_ident2_supported(a.n1, a.n2));
  if (impl == 0 && (tq_tc05_supported(a) || tq_wide_supported(a))) return true;
  if (impl == 0 && int64_t(a.n1) * a.n2 <= 1024 && tq_simt_supported(a.n1, a.n2)) return true;
  const bool tc_shape = (a.n1 % 16 == 0) && (a.n2 % 16 == 0);
  if (!a.zero && impl <= 1 && tc_shape && tq_mma_supported(a.n1, a.n2)) return true;
  return tq_simt_supported(a.n1, a.n2);
}

bool tq_is_pdl(const TQArgs& a) {
  return tq_impl() == 0 && (tq_tc05_supported(a) || (a.p2 != nullptr && tq_wide_supported(a)));
}

cudaError_t transform_quant_launch(const TQArgs& a) {
  const int impl = tq_impl();
  if (a.p2 == nullptr)                                  // P2 = I (validated by the ABI layer)
    return (impl == 0 && tq_tc05_supported(a)) ? tq_tc05_launch(a) : tq_ident2_launch(a);
  if (a.zero) {                          // asymmetric: tcgen05 kernel, else the CUDA-core kernel
    if (impl == 0 && tq_tc05_supported(a)) return tq_tc05_launch(a);
    if (impl == 0 && tq_wide_supported(a)) return tq_wide_launch(a);
    return tq_simt_launch(a);
  }
  const bool tc_shape = (a.n1 % 16 == 0) && (a.n2 % 16 == 0);
  if (impl == 0 && tq_tc05_supported(a)) return tq_tc05_launch(a);
  if (impl == 0 && tq_wide_supported(a)) return tq_wide_launch(a);
  if (impl == 0 && int64_t(a.n1) * a.n2 <= 1024 && tq_simt_supported(a.n1, a.n2)) return tq_simt_launch(a);
  if (impl <= 1 && tc_shape && tq_mma_supported(a.n1, a.n2)) return tq_mma_launch(a);
  return tq_simt_launch(a);
}

}  // namespace fq
