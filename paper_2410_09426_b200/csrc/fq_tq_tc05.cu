// fq_tq_tc05.cu -- fused Kronecker transform + clip + per-token INT4 quantize + pack on the
// 5th-generation tensor cores (tcgen05, TMEM, TMA).
//
// Per token t (Eq.3 activation factor; clip PAPER.md:258-259; per-token
// symmetric INT4 PAPER.md:367, Eq.1):
//   V_t = reshape(x_t, n1, n2) (row-major)   W_t = P1^T V_t   Y_t = W_t P2
//   s_t = alpha max|Y_t| / 7 (1 if Y_t == 0)  q = clamp(rint(Y_t / s_t), -8, 7), packed
//
// P1^T is applied first, as in the paper's kernel (App. B.3).  Both small
// matmuls run as tcgen05.mma kind::f16 with M = 128 and every operand in the MN-major
// SWIZZLE_128B shared-memory layout, so the token tiles, P1 and P2 are TMA-loaded exactly as they
// sit in HBM (no transposes):
//   stage 1  D1[(t,j)][i] = sum_i' X_t[i'][j] P1[i'][i]   (= W_t^T)  A = X tile  [K=i'][M=(t,j)]
//                                                                  B = P1      [K=i'][N=i]
//   stage 2  D2[(t,i)][j] = sum_j' W_t[i][j'] P2[j'][j]   (= Y_t)    A = W (smem) [K=j'][M=(t,i)]
//                                                                  B = P2      [K=j'][N=j]
// Between the stages an epilogue moves W from TMEM (fp32) to shared memory as fp16 after an
// exact per-token power-of-two prescale (reading R9: an fp16 intermediate, never bf16;
// the prescale makes it overflow/underflow-safe and is divided out of Y exactly).  D2 lane (t,i)
// holds row i of Y_t, so the quantized row is packed in registers and stored contiguously.
//
// Tile = TOK tokens (2 for n1 = 64, else 1), so that both MMAs have M = 128.  Warp roles
// (persistent, one CTA per SM, tiles strided by gridDim):
//   warp 0      TMA producer: P1, P2 once, then X tiles into a STAGES-deep ring
//   warp 1      MMA issuer (one thread): stage 1 of tile k+1 is issued before stage 2 of tile k
//   warp 2      TMEM allocator
//   warps 4-7   epilogue group 0 (even tiles), warps 8-11 group 1 (odd tiles): each group does
//               stage-1 epilogue (prescale, fp16, smem) and stage-2 epilogue (absmax, quantize,
//               pack, store) of its own tiles; TMEM/smem buffers are indexed by the group.
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"
#include "fq_tc05.cuh"
#include "fq_quant.cuh"

namespace fq {
namespace tq5 {

// Optional device-side timeline (build with -DFQ_TRACE, scripts/trace_tq.py): globaltimer stamps
// of the pipeline events of the first TRACE_CTAS CTAs.  Compiled out of the production library.
constexpr int TRACE_CTAS = 4, TRACE_EV = 256;
#ifdef FQ_TRACE
__device__ unsigned long long g_trace[TRACE_CTAS * TRACE_EV];
__device__ unsigned long long g_cta[1024 * 2];     // every CTA: start, end
__device__ unsigned long long g_stamp[8];
FQ_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}
__global__ void stamp_kernel(int slot) { g_stamp[slot] = gtimer(); }
FQ_DEVICE void cta_stamp(int which) {
  if (blockIdx.x < 1024) g_cta[blockIdx.x * 2 + which] = gtimer();
}
FQ_DEVICE void trace(int ev) {
  if (blockIdx.x < TRACE_CTAS && ev < TRACE_EV) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    g_trace[blockIdx.x * TRACE_EV + ev] = t;
  }
}
#else
FQ_DEVICE void trace(int) {}
FQ_DEVICE void cta_stamp(int) {}
#endif

constexpr int MAX_GROUPS = 4;
// per-launch {claims, departures} counter pairs of the dynamic tile schedule: a ring of slots in
// this module's device memory, handed out round-robin per device, reset by each launch's last CTA
constexpr int TQ_SLOTS = 1024;
__device__ unsigned g_tq_sync[2 * TQ_SLOTS];
constexpr int SMEM_LIMIT = 232448;       // max dynamic smem per block on sm_100
constexpr int SMEM_OVERHEAD = 1024 + 512;  // 1024-B alignment slack + barriers/scratch

// SMALL (decode-size launches, T <= 64, so every CTA has exactly one tile): one epilogue group,
// one X stage, and the stage-2 operand A2 written over P1 and the X tile once the stage-1 MMA
// that read them has completed -- 112 x 128 needs 88 KB of shared memory (120 KB without the
// aliasing) and 256 TMEM columns, 64 x 64 32 KB and 128 columns, so the CTA becomes resident
// beside a decode-GEMM CTA of the preceding kernel (PDL): its setup and loads overlap that tail.
// IDENT2: P2 = I (the paper's online o_proj transform P_o (a x a) (x) I_{d_head}, PAPER.md:297, 726;
// DESIGN.md reading R22): stage 1 only, its fp32 result quantized directly (no fp16 intermediate,
// no D2 in TMEM); the A2 buffer is the staging area that turns TMEM's column-per-lane layout into
// row-major packed codes.
// SMALL = 2 (MULTI, experiment): one epilogue group, two X stages, no aliasing, a few tiles per
// CTA and several CTAs per SM, so the hardware block scheduler hands the tiles to SMs as they
// free up (e.g. while the preceding GEMM's last wave drains).
template <int N1, int N2, int SMALL = 0, bool IDENT2 = false>
struct Cfg {
  static_assert(N2 == 64 || N2 == 128, "n2 in {64, 128}");
  static_assert(N1 % 16 == 0 && N1 >= 16 && N1 <= 128, "n1 multiple of 16, <= 128");
  static_assert(N1 == 64 || N2 == 128, "n1 != 64 needs n2 == 128 (stage-1 M = n2)");
  static constexpr int TOK = (N1 == 64) ? 2 : 1;       // tokens per tile
  static constexpr int JB = N2 / 64;                   // 64-element j blocks of a token row
  static constexpr int G1 = TOK * N2 / 128;            // stage-1 MMA groups (M = 128) per tile
  static constexpr int P1_ATOMS = (N1 + 63) / 64;
  static constexpr int P1_BYTES = P1_ATOMS * N1 * 128;
  static constexpr int P2_BYTES = JB * N2 * 128;
  static constexpr int X_BYTES = TOK * JB * N1 * 128;  // TOK * n * 2
  static constexpr int A2_BYTES = 2 * N2 * 128;        // 2 M-atoms x N2 K-rows x 128 B
  static constexpr int D1C = G1 * N1;                  // TMEM columns of one stage-1 result
  // epilogue groups = tiles in flight (each owns a D1, D2 and A2 slot), as many as TMEM allows
  static constexpr int D2C = IDENT2 ? 0 : N2;         // TMEM columns of one stage-2 result
  // ALIAS_D (round 2c, n2 = 128): a group's stage-2 result is written over its stage-1 result (the
  // stage-2 MMA runs after the stage-1 epilogue has read D1; the next stage-1 MMA of the group waits
  // until the stage-2 epilogue has read D2), so a group needs max(D1, D2) columns, not their sum:
  // three epilogue groups instead of two at 64 x 128 and 112 x 128
  static constexpr bool ALIAS_D = SMALL == 0 && !IDENT2 && N2 == 128;
  static constexpr int GW = ALIAS_D ? (D1C > N2 ? D1C : N2) : D1C + D2C;   // TMEM columns per group
  static constexpr int GROUPS_TMEM = (512 / GW) > MAX_GROUPS ? MAX_GROUPS : (512 / GW);
  static constexpr bool ALIAS_A2 = SMALL == 1 && !IDENT2;     // A2 over P1 + X (one tile per CTA)
  // and as many as leave shared memory for two X stages
  static constexpr int fixed_of(int g) { return P1_BYTES + (IDENT2 ? 0 : P2_BYTES) + (ALIAS_A2 ? 0 : g * A2_BYTES); }
  static constexpr int GROUPS_FIT =
      (GROUPS_TMEM > 1 && (SMEM_LIMIT - SMEM_OVERHEAD - fixed_of(GROUPS_TMEM)) / X_BYTES < 2)
          ? ((GROUPS_TMEM > 2 && (SMEM_LIMIT - SMEM_OVERHEAD - fixed_of(GROUPS_TMEM - 1)) / X_BYTES < 2)
                 ? GROUPS_TMEM - 2 : GROUPS_TMEM - 1)
          : GROUPS_TMEM;
  static constexpr int GROUPS = SMALL ? 1 : GROUPS_FIT;
  static constexpr int THREADS = (4 + 4 * GROUPS) * 32;
  static constexpr int TMEM_USED = GROUPS * GW;
  static constexpr int TMEM_COLS = TMEM_USED <= 128 ? 128 : (TMEM_USED <= 256 ? 256 : 512);
  static constexpr int D1_STRIDE = ALIAS_D ? GW : D1C;        // D1 of group par: par * D1_STRIDE
  static constexpr int D2_COL0 = ALIAS_D ? 0 : GROUPS * D1C;   // D2 of group par: D2_COL0 + par * D2_STRIDE
  static constexpr int D2_STRIDE = ALIAS_D ? GW : N2;
  static constexpr int FIXED = fixed_of(GROUPS);
  static constexpr int STAGES_FIT = (SMEM_LIMIT - SMEM_OVERHEAD - FIXED) / X_BYTES;
  static constexpr int STAGES = SMALL == 1 ? 1 : SMALL == 2 ? 2 : (STAGES_FIT > 8 ? 8 : STAGES_FIT);
  static constexpr size_t SMEM = size_t(FIXED) + size_t(STAGES) * X_BYTES + SMEM_OVERHEAD;
  static_assert(TMEM_USED <= 512, "TMEM budget");
  static_assert(SMALL || STAGES >= 2, "shared-memory budget");
  static_assert(!ALIAS_A2 || A2_BYTES <= P1_BYTES + X_BYTES, "A2 fits over P1 + X");
};

using namespace qz;   // MAGIC, prescale_exp, exp2i, max3f, fma_sat (fq_quant.cuh)

// max |v[i]| over N values: 8 independent accumulators fed two values per 3-input max
// (a running max would be a dependent chain of N operations)
template <int N>
FQ_DEVICE float absmax(const uint32_t* v) {
  static_assert(N % 16 == 0, "");
  float a[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) a[e] = fmaxf(fabsf(__uint_as_float(v[e])), fabsf(__uint_as_float(v[8 + e])));
#pragma unroll
  for (int i = 16; i < N; i += 16)
#pragma unroll
    for (int e = 0; e < 8; ++e)
      a[e] = max3f(a[e], fabsf(__uint_as_float(v[i + e])), fabsf(__uint_as_float(v[i + 8 + e])));
  return max3f(max3f(a[0], a[1], a[2]), max3f(a[3], a[4], a[5]), fmaxf(a[6], a[7]));
}

// Walk N TMEM columns of this warp's 32 lanes in chunks of 32 (and a 16-column tail): fn(v, n, col)
// gets n (32 or 16) fp32 values starting at column col.  Keeps at most 32 values live.
template <int N, typename F>
FQ_DEVICE void tmem_chunks(uint32_t taddr, F&& fn) {
#pragma unroll
  for (int c = 0; c + 32 <= N; c += 32) {
    uint32_t v[32];
    tc::tmem_ld16(taddr + uint32_t(c), *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
    tc::tmem_ld16(taddr + uint32_t(c + 16), *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
    tc::tmem_ld_wait();
    fn(v, 32, c);
  }
  if constexpr (N % 32 == 16) {
    uint32_t v[32];
    tc::tmem_ld16(taddr + uint32_t(N - 16), *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
    tc::tmem_ld_wait();
    fn(v, 16, N - 16);
  }
}

// Single-pass variant for rows of N <= 64 columns: the row is loaded from TMEM once into
// registers and both the statistics and the conversion read the registers (TMEM reads are the
// epilogues' throughput limit: one pass instead of two halves them).
template <int N>
FQ_DEVICE void tmem_ld_row(uint32_t taddr, uint32_t* v) {
  static_assert(N % 16 == 0 && N <= 64, "");
#pragma unroll
  for (int c = 0; c < N; c += 16) tc::tmem_ld16(taddr + uint32_t(c), *reinterpret_cast<uint32_t(*)[16]>(v + c));
  tc::tmem_ld_wait();
}
template <int N, bool SINGLE, typename F>
FQ_DEVICE void row_chunks(uint32_t taddr, const uint32_t* regs, F&& fn) {
  if constexpr (SINGLE) {
    static_assert(N % 32 == 0, "");
#pragma unroll
    for (int c = 0; c < N; c += 32) fn(regs + c, 32, c);
  } else {
    tmem_chunks<N>(taddr, fn);
  }
}

template <int N1, int N2, bool BF16, bool WRITE_Y, bool ASYM, int SMALL = 0, bool IDENT2 = false>
__global__ void __launch_bounds__(Cfg<N1, N2, SMALL, IDENT2>::THREADS, 1)
tq_tc05_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmP1,
               const __grid_constant__ CUtensorMap tmP2, int64_t T, float alpha, uint8_t* __restrict__ q,
               float* __restrict__ scale, float* __restrict__ y_out, int8_t* __restrict__ zero, int pdl,
               unsigned* __restrict__ tsync) {
  using C = Cfg<N1, N2, SMALL, IDENT2>;
  // Tile schedule.  DYN (the persistent configuration): every CTA starts with a static chunk of CH
  // tiles and then claims further chunks from a per-launch counter, so CTAs that become resident
  // early -- on the SMs the preceding GEMM's last wave leaves idle (PDL) -- take more of the work
  // than CTAs placed after that GEMM has drained.  Otherwise (SMALL, IDENT2) tiles are strided.
  // Either way the producer publishes each tile index with its X stage (tile_id, -1 = end), the
  // stage-1 MMA thread forwards it per sequence index (seq_tile + tready) to the epilogue groups and
  // the stage-2 MMA thread, which all stop at the first -1.
  constexpr bool DYN = !SMALL && !IDENT2;
  constexpr int CH = 2;                                   // tiles per claim
  constexpr int S = C::STAGES, TOK = C::TOK, G = C::GROUPS, THREADS = C::THREADS;
  constexpr uint32_t IDESC1 = tc::idesc_f16(128, N1, BF16 ? 1 : 0, 1, 1);
  constexpr uint32_t IDESC2 = tc::idesc_f16(128, N2, 0, 1, 1);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // layout P1 | P2 | A2 [G] | X [S]; SMALL: P2 | P1 | X with A2 over P1 + X (C::ALIAS_A2)
  uint8_t* sP1 = C::ALIAS_A2 ? smem + C::P2_BYTES : smem;
  uint8_t* sP2 = C::ALIAS_A2 ? smem : sP1 + C::P1_BYTES;
  uint8_t* sA2 = C::ALIAS_A2 ? sP1 : sP2 + (IDENT2 ? 0 : C::P2_BYTES);
  uint8_t* sX = C::ALIAS_A2 ? sP1 + C::P1_BYTES : sA2 + G * C::A2_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + size_t(S) * C::X_BYTES);
  uint64_t* xfull = bars;            // [S]  TMA -> MMA
  uint64_t* xempty = bars + S;       // [S]  MMA commit -> TMA
  uint64_t* pfull = bars + 2 * S;    // P1, P2 landed
  uint64_t* d1full = pfull + 1;      // [G]  MMA commit -> epilogue group
  uint64_t* a2full = d1full + G;     // [G]  epilogue group (4 warps) -> MMA
  uint64_t* d2full = a2full + G;     // [G]  MMA commit -> epilogue group
  uint64_t* tready = d2full + G;     // [G]  stage-1 MMA thread: tile index of the group's next tile
  uint64_t* d2free = tready + G;     // [G]  ALIAS_D: stage-2 epilogue read D2 -> next stage-1 MMA
  __shared__ float red[MAX_GROUPS * 8];                        // [groups][2 parities][4 warps]
  __shared__ uint32_t tmem_slot[1];
  __shared__ int tile_id[8];                                   // [S] tile of each X stage (-1: end)
  __shared__ int seq_tile[32];                                 // [k % 32] tile of sequence index k

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    trace(0);
    cta_stamp(0);
  }
  const int num_tiles = int((T + TOK - 1) / TOK);                 // T < 2^31 (host check)
  const int my_tiles = num_tiles > int(blockIdx.x) ? (num_tiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;

  // X tiles stream into the ring as early as possible (before the TMEM allocation completes)
  int kq = 0;                                            // producer's sequence index
  auto issue_tile = [&](int tile) {
    const int k = kq++, s = k % S;
    tc::mbar_wait(&xempty[s], ((k / S) & 1) ^ 1);
    tile_id[s] = tile;                                   // published by the arrive (release) below
    tc::mbar_expect_tx(&xfull[s], C::X_BYTES);
    uint8_t* dst = sX + size_t(s) * C::X_BYTES;
#pragma unroll
    for (int b = 0; b < C::JB; ++b) tc::tma_load_3d(dst + b * TOK * N1 * 128, &tmX, &xfull[s], b * 64, 0, tile * TOK);
    if (k < 16) trace(8 + k);
  };
  auto issue_end = [&] {
    const int k = kq, s = k % S;
    tc::mbar_wait(&xempty[s], ((k / S) & 1) ^ 1);
    tile_id[s] = -1;
    tc::mbar_arrive(&xfull[s]);
  };
  // DYN: static first chunk [CH b, CH b + CH); strided: tiles b, b + grid, ...
  const int first_n = DYN ? (CH < num_tiles - CH * int(blockIdx.x) ? CH : num_tiles - CH * int(blockIdx.x)) : my_tiles;
  auto static_tile = [&](int k) { return DYN ? CH * int(blockIdx.x) + k : int(blockIdx.x) + k * int(gridDim.x); };
  const int prefill = first_n < S ? first_n : S;
  unsigned nxt = 0;                                      // DYN: the claim in flight (producer thread)
  if (threadIdx.x == 0) {
    tc::tma_prefetch_desc(&tmX);
    tc::tma_prefetch_desc(&tmP1);
    if constexpr (!IDENT2) tc::tma_prefetch_desc(&tmP2);
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&xfull[s], 1);
      tc::mbar_init(&xempty[s], 1);
    }
    tc::mbar_init(pfull, 1);
    for (int b = 0; b < G; ++b) {
      tc::mbar_init(&d1full[b], 1);
      tc::mbar_init(&a2full[b], 4);
      tc::mbar_init(&d2full[b], 1);
      tc::mbar_init(&tready[b], 1);
      tc::mbar_init(&d2free[b], 4);
    }
    tc::fence_barrier_init();
    if constexpr (DYN) nxt = atomicAdd(tsync, 1u);      // first claim: its latency hides behind the loads
    // PDL (fq_internal.h): P1, P2 and X stream in while the preceding kernel finishes unless it
    // writes them (host-side hazard check, fq_abi.cu)
    auto load_p = [&] {
      tc::mbar_expect_tx(pfull, C::P1_BYTES + (IDENT2 ? 0 : C::P2_BYTES));
      for (int a = 0; a < C::P1_ATOMS; ++a) tc::tma_load_2d(sP1 + a * N1 * 128, &tmP1, pfull, a * 64, 0);
      if constexpr (!IDENT2)
        for (int b = 0; b < C::JB; ++b) tc::tma_load_2d(sP2 + b * N2 * 128, &tmP2, pfull, b * 64, 0);
    };
    if (pdl & PDL_P) load_p();
    trace(3);
    if ((pdl & (PDL_P | PDL_X)) != (PDL_P | PDL_X)) tc::griddep_wait();
    if (!(pdl & PDL_P)) load_p();
    trace(4);
    for (int k = 0; k < prefill; ++k) issue_tile(static_tile(k));
    trace(1);
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  tc::mbar_wait(pfull, 0);
  if (threadIdx.x == 0) trace(2);
  // stage 2 runs in fp16 (R9): a bf16 P2 becomes fp16 P2 * 2^e2 in place (power-of-two scaled
  // into fp16 range, so no entry overflows); 2^-e2 is applied to the statistics below, exactly
  float inv_p2 = 1.0f;
  if constexpr (BF16 && !IDENT2) {
    __shared__ uint32_t p2max;
    inv_p2 = exp2i(-bf16_to_f16_pow2(sP2, C::P2_BYTES / 2, &p2max));
  } else {
    __syncthreads();
  }
  // PDL protocol (fq_internal.h): dependents launch only after this kernel's griddepcontrol.wait
  // has returned.  One thread waits (round 2c: after the last CTA-wide barrier before the roles,
  // not in front of it) while the other warps already compute; outputs are written before the
  // wait only if the host allowed it (PDL_OUT), see `waited` below.
  if (warp == 2 && lane == 0) {
    tc::griddep_wait();
    tc::griddep_launch();
  }

  if (warp == 0) {
    // ================================ TMA producer ================================
    if (lane == 0) {
      for (int k = prefill; k < first_n; ++k) issue_tile(static_tile(k));
      if constexpr (DYN) {
        for (;;) {                                       // claim chunks until the tiles run out
          const int base = CH * (int(gridDim.x) + int(nxt));
          if (base >= num_tiles) break;
          nxt = atomicAdd(tsync, 1u);                    // the next claim travels while this chunk loads
          for (int i = 0; i < CH && base + i < num_tiles; ++i) issue_tile(base + i);
        }
        if (atomicAdd(tsync + 1, 1u) == gridDim.x - 1) {   // last CTA out: every claim is made, reset
          atomicExch(tsync, 0u);
          atomicExch(tsync + 1, 0u);
        }
      }
      issue_end();
    }
    __syncwarp();
  } else if (warp == 1 || warp == 3) {
    // ================================ MMA issuers ================================
    // warp 1 issues stage 1 of every tile, warp 3 stage 2: a stage-1 MMA waiting for its X tile
    // never holds up a stage-2 MMA that is ready (and vice versa).
    if (lane == 0) {
      const uint32_t p1a = smem_u32(sP1), p2a = smem_u32(sP2);
      auto mma1 = [&](int k) {
        const int s = k % S, par = k % G;
        if (k < 16) trace(24 + k);
        const uint32_t xs = smem_u32(sX + size_t(s) * C::X_BYTES);
#pragma unroll
        for (int g = 0; g < C::G1; ++g) {
          // M = 128 rows (t, j): n2 = 64 -> the TOK tokens' j-block 0; n2 = 128 -> token g's 2 j-blocks
          const uint32_t a0 = xs + uint32_t(N2 == 64 ? 0 : g * N1 * 128);
          const uint32_t lbo = uint32_t(N2 == 64 ? N1 * 128 : TOK * N1 * 128);
          const uint32_t d = tmem + uint32_t(par * C::D1_STRIDE + g * N1);
#pragma unroll
          for (int kk = 0; kk < N1 / 16; ++kk)
            tc::mma_ss<false>(d, tc::sdesc_sw128(a0 + kk * 2048, lbo, 1024),
                              tc::sdesc_sw128(p1a + kk * 2048, N1 * 128, 1024), IDESC1, kk > 0);
        }
        tc::mma_commit(&xempty[s]);
        tc::mma_commit(&d1full[par]);
      };
      auto mma2 = [&](int k) {
        const int par = k % G;
        if (k < 16) trace(40 + k);
        const uint32_t a0 = smem_u32(sA2 + par * C::A2_BYTES);
        const uint32_t d = tmem + uint32_t(C::D2_COL0 + par * C::D2_STRIDE);
#pragma unroll
        for (int kk = 0; kk < N2 / 16; ++kk)
          tc::mma_ss<false>(d, tc::sdesc_sw128(a0 + kk * 2048, N2 * 128, 1024),
                            tc::sdesc_sw128(p2a + kk * 2048, N2 * 128, 1024), IDESC2, kk > 0);
        tc::mma_commit(&d2full[par]);
      };
      if (warp == 1) {
        // D1 slot k % G is free once the group finished the stage-1 epilogue of tile k - G
        for (int k = 0;; ++k) {
          const int s = k % S;
          tc::mbar_wait(&xfull[s], (k / S) & 1);
          tc::fence_after();
          const int tile = *static_cast<volatile int*>(&tile_id[s]);
          if (tile < 0) {                                // end: tell each group (and warp 3) in turn
            for (int g = 0; g < G; ++g) {
              const int kk = k + g;
              if (kk >= G) tc::mbar_wait(&a2full[kk % G], ((kk - G) / G) & 1);
              seq_tile[kk % 32] = -1;
              tc::mbar_arrive(&tready[kk % G]);
            }
            break;
          }
          if (k >= G) {                                  // the group's TMEM slot is free
            if constexpr (C::ALIAS_D) tc::mbar_wait(&d2free[k % G], ((k - G) / G) & 1);
            else tc::mbar_wait(&a2full[k % G], ((k - G) / G) & 1);
          }
          seq_tile[k % 32] = tile;
          tc::mbar_arrive(&tready[k % G]);
          mma1(k);
        }
      } else if constexpr (!IDENT2) {
        for (int k = 0;; ++k) {
          tc::mbar_wait(&a2full[k % G], (k / G) & 1);    // the group's stage-1 epilogue (or its end)
          tc::fence_after();
          if (*static_cast<volatile int*>(&seq_tile[k % 32]) < 0) break;
          mma2(k);
        }
        trace(122);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ================================ epilogue groups ================================
    const int grp = (warp - 4) >> 2, qd = warp & 3;
    const int L = qd * 32 + lane;                        // TMEM lane of this thread
    const uint32_t lane_base = tmem + (uint32_t(qd * 32) << 16);
    float* redg = red + grp * 8;
    int rp = 0;
    auto exchange = [&](float m) {                       // per-warp max -> all 4 warps' maxima
      m = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(m)));   // m >= 0: uint order
      if (lane == 0) redg[rp * 4 + qd] = m;
      named_bar_sync(1 + grp, 128);
      float r[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) r[w] = redg[rp * 4 + w];
      rp ^= 1;
      return make_float4(r[0], r[1], r[2], r[3]);
    };
    constexpr int QROW = N2 / 2;                         // packed bytes per row i of a token
    constexpr int QTOK = N1 * N2 / 2;                    // packed bytes per token
    bool waited = (pdl & PDL_OUT) != 0;                  // outputs written before the wait only if allowed
    for (int k = grp;; k += G) {
      const int par = grp;                               // == k % G
      const uint32_t ph = (k / G) & 1;
      tc::mbar_wait(&tready[par], ph);
      const int tile = *static_cast<volatile int*>(&seq_tile[k % 32]);
      if (tile < 0) {                                    // end: release warp 3 (it reads the -1 too)
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&a2full[par]);
        break;
      }
      const int64_t t0 = int64_t(tile) * TOK;
      if constexpr (IDENT2) {
        // ---- P2 = I: D1 lane j, column i holds Y_t[i][j] (fp32, the whole token in 128 lanes) ----
        tc::mbar_wait(&d1full[par], ph);
        tc::fence_after();
        uint8_t* stg = sA2 + par * C::A2_BYTES;          // [N1][N2/2] packed bytes of one token
#pragma unroll 1
        for (int g = 0; g < C::G1; ++g) {
          const uint32_t d1 = lane_base + uint32_t(par * C::D1_STRIDE + g * N1);
          const int64_t t = t0 + g;
          float m1 = 0.f, hi1 = 0.f, lo1 = 0.f;
          tmem_chunks<N1>(d1, [&](const uint32_t* v, int n, int) {
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              if (e < n) {
                const float a0 = __uint_as_float(v[e]), a1 = __uint_as_float(v[e + 1]);
                if constexpr (ASYM) {
                  hi1 = max3f(hi1, a0, a1);
                  lo1 = max3f(lo1, -a0, -a1);
                } else {
                  m1 = max3f(m1, fabsf(a0), fabsf(a1));
                }
              }
            }
          });
          auto tok_max = [](float4 r) { return fmaxf(fmaxf(r.x, r.y), fmaxf(r.z, r.w)); };
          float mp, lop = 0.f;
          if constexpr (ASYM) {
            const float hip = tok_max(exchange(hi1));
            lop = tok_max(exchange(lo1));
            mp = hip + lop;
          } else {
            mp = tok_max(exchange(m1));
          }
          float c15, B15, zq = 0.f;                        // the quantizer of the two-stage path below
          if constexpr (ASYM) {
            const float sp = alpha * mp * (1.0f / 15.0f);
            zq = sp > 0.f ? rintf(__fdiv_rn(alpha * lop, sp)) : 0.f;
            c15 = sp > 0.f ? __frcp_rn(alpha * mp) : 0.f;
            B15 = zq * (1.0f / 15.0f);
          } else {
            c15 = mp > 0.f ? __fdividef(7.0f / 15.0f, alpha * mp) : 0.f;
            B15 = 8.0f / 15.0f;
          }
          // codes of column j (this lane) for every row i, 8 nibbles per word (nibble e = row 8w + e)
          uint32_t cw[N1 / 8];
          tmem_chunks<N1>(d1, [&](const uint32_t* v, int n, int col) {
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              if (e < n) {
                uint32_t wv = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  const float z = fmaf(fma_sat(__uint_as_float(v[e + u]), c15, B15), 15.0f, MAGIC - 8.0f);
                  wv |= (__float_as_uint(z) & 0xFu) << (4 * u);
                }
                cw[(col + e) / 8] = wv;
              }
            }
          });
          if constexpr (WRITE_Y) {
            if (t < T)
              tmem_chunks<N1>(d1, [&](const uint32_t* v, int n, int col) {
#pragma unroll
                for (int e = 0; e < 32; ++e)
                  if (e < n) y_out[t * (N1 * N2) + int64_t(col + e) * N2 + L] = __uint_as_float(v[e]);
              });
          }
          if (g == C::G1 - 1) {                            // D1 slot read completely: MMA1 may reuse it
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&a2full[par]);
          }
          // column pair (j, j+1) -> one byte per row i (low nibble = even j): the even lane of the
          // pair writes rows [0, N1/2), the odd lane rows [N1/2, N1)
          uint32_t ow[N1 / 8];
#pragma unroll
          for (int w = 0; w < N1 / 8; ++w) ow[w] = __shfl_xor_sync(0xffffffffu, cw[w], 1);
          const bool odd = L & 1;
#pragma unroll
          for (int w = 0; w < N1 / 16; ++w) {
            const uint32_t lo = odd ? ow[w + N1 / 16] : cw[w];    // codes of column j & ~1
            const uint32_t hi = odd ? cw[w + N1 / 16] : ow[w];    // codes of column j | 1
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int i = (odd ? N1 / 2 : 0) + 8 * w + u;
              stg[i * (N2 / 2) + (L >> 1)] = uint8_t(((lo >> (4 * u)) & 0xFu) | (((hi >> (4 * u)) & 0xFu) << 4));
            }
          }
          named_bar_sync(1 + grp, 128);                    // the token's packed bytes are staged
          if (!waited) {
            tc::griddep_wait();
            waited = true;
          }
          if (t < T) {
            constexpr int CH = N1 * N2 / 2 / 16;           // 16-byte chunks of one token
#pragma unroll
            for (int c = L; c < CH; c += 128)
              *reinterpret_cast<uint4*>(q + t * (N1 * N2 / 2) + c * 16) = *reinterpret_cast<const uint4*>(stg + c * 16);
            if (L == 0) {
              if constexpr (ASYM) {
                scale[t] = mp > 0.f ? alpha * mp / 15.0f : 1.0f;
                zero[t] = int8_t(int(zq) - 8);
              } else {
                scale[t] = mp > 0.f ? alpha * mp / 7.0f : 1.0f;
              }
            }
          }
        }
        continue;
      }
      // -------- stage-1 epilogue: D1 (fp32) -> prescaled fp16 A operand of stage 2 --------
      int pe[TOK];                                       // per-token prescale exponents
      tc::mbar_wait(&d1full[par], ph);
      tc::fence_after();
      if (L == 0 && k < 16) trace(56 + k);
#define FQ_SUB(sub) \
  if (L == 0 && k < 8) trace(128 + k * 16 + (sub))
      constexpr bool SINGLE1 = (N1 == 64);               // row of 64: one TMEM pass (registers)
      constexpr bool SINGLE2 = (N2 == 64);
#pragma unroll
      for (int g = 0; g < C::G1; ++g) {
        const uint32_t d1 = lane_base + uint32_t(par * C::D1_STRIDE + g * N1);
        uint32_t rv1[SINGLE1 ? N1 : 1];
        if constexpr (SINGLE1) tmem_ld_row<N1>(d1, rv1);
        // pass 1: max |W| over this lane's row (rows > 64 columns: two passes over TMEM keep
        // <= 32 values in registers)
        float m1 = 0.f;
        row_chunks<N1, SINGLE1>(d1, rv1, [&](const uint32_t* v, int n, int) {
#pragma unroll
          for (int e = 0; e < 32; e += 2)
            if (e < n) m1 = max3f(m1, fabsf(__uint_as_float(v[e])), fabsf(__uint_as_float(v[e + 1])));
        });
        FQ_SUB(1);
        const float4 r = exchange(m1);
        FQ_SUB(2);
        int tt;
        if constexpr (N2 == 64) {                        // tokens = lane halves (quadrants 0-1, 2-3)
          pe[0] = prescale_exp(fmaxf(r.x, r.y));
          if constexpr (TOK > 1) pe[1] = prescale_exp(fmaxf(r.z, r.w));
          tt = L >> 6;
        } else {                                         // token g spans all 128 lanes
          pe[g] = prescale_exp(fmaxf(fmaxf(r.x, r.y), fmaxf(r.z, r.w)));
          tt = g;
        }
        const float pre = exp2i((TOK > 1 && tt) ? pe[TOK - 1] : pe[0]);
        const int j = (N2 == 64) ? (L & 63) : L;         // K row (j') of the stage-2 A operand
        const uint32_t row = smem_u32(sA2) + uint32_t(par * C::A2_BYTES + j * 128);
        // pass 2: prescale, fp16, swizzled MN-major row j of A2
        row_chunks<N1, SINGLE1>(d1, rv1, [&](const uint32_t* v, int n, int col) {
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            if (e < n) {
              const int c8 = (col + e) >> 3;
              const int atom = (N1 == 64) ? tt : (c8 >> 3), ch = c8 & 7;
              tc::sts128(row + uint32_t(atom * (N2 * 128) + ((ch ^ (j & 7)) << 4)),
                         pack_half2(__uint_as_float(v[e + 0]) * pre, __uint_as_float(v[e + 1]) * pre),
                         pack_half2(__uint_as_float(v[e + 2]) * pre, __uint_as_float(v[e + 3]) * pre),
                         pack_half2(__uint_as_float(v[e + 4]) * pre, __uint_as_float(v[e + 5]) * pre),
                         pack_half2(__uint_as_float(v[e + 6]) * pre, __uint_as_float(v[e + 7]) * pre));
            }
          }
        });
      }
      FQ_SUB(3);
      tc::fence_proxy_async_smem();
      FQ_SUB(4);
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&a2full[par]);
      if (L == 0 && k < 16) trace(72 + k);

      // -------- stage-2 epilogue: absmax, clip, quantize, pack, store --------
      tc::mbar_wait(&d2full[par], ph);
      tc::fence_after();
      if (L == 0 && k < 16) trace(88 + k);
      FQ_SUB(8);
      const uint32_t d2 = lane_base + uint32_t(C::D2_COL0 + par * C::D2_STRIDE);
      const int tt = (N1 == 64) ? (L >> 6) : 0;
      const int i = (N1 == 64) ? (L & 63) : L;
      const bool valid = (N1 == 64) || (L < N1);
      float m2 = 0.f, hi2 = 0.f, lo2 = 0.f;             // sym: max |y|; asym: max(max y, 0), -min(min y, 0)
      uint32_t rv2[SINGLE2 ? N2 : 1];
      if constexpr (SINGLE2) tmem_ld_row<N2>(d2, rv2);
      row_chunks<N2, SINGLE2>(d2, rv2, [&](const uint32_t* v, int, int) {
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
      });
      FQ_SUB(9);
      float mp, hip = 0.f, lop = 0.f;                    // token statistics (prescaled by 2^pe)
      {
        auto tok_max = [&](float4 r) {
          if constexpr (N1 == 64) return tt == 0 ? fmaxf(r.x, r.y) : fmaxf(r.z, r.w);
          else return fmaxf(fmaxf(r.x, r.y), fmaxf(r.z, r.w));
        };
        if constexpr (ASYM) {
          hip = tok_max(exchange(valid ? hi2 : 0.f));
          lop = tok_max(exchange(valid ? lo2 : 0.f));
          mp = hip + lop;                                // hi - lo, both >= 0 terms
        } else {
          mp = tok_max(exchange(valid ? m2 : 0.f));
        }
      }
      FQ_SUB(10);
      const int64_t t = t0 + tt;
      const bool store = valid && t < T;
      const float inv_pre = exp2i(-((TOK > 1 && tt) ? pe[TOK - 1] : pe[0]));
      // code = clamp(rint(y * cq), -8, 7) with cq = 7 / (alpha m) (on the prescaled values, exactly
      // (7 / (alpha m)) / 2^pe).  The clamp rides on the FMA pipe: u = sat((y cq + 8) / 15) in [0, 1],
      // then fma(u, 15, MAGIC - 8) rounds u*15 - 8 half-to-even into the low mantissa bits; the
      // extra rounding of u moves y*cq by < 1e-5 code units (well inside the near-tie window).
      // asymmetric (R19): s = alpha (hi - lo) / 15, z = rint(alpha lo' / s) with lo' = -min(min y, 0);
      // q = clamp(rint(y / s) + z, 0, 15), stored as q - 8: the same FFMA.SAT form with
      // c15 = 1 / (15 s) and offset z / 15 (z an integer, so rint(y/s + z) = rint(y/s) + z).
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
      uint8_t* qrow = q + (store ? t * QTOK + i * QROW : 0);
      if (!waited) {
        tc::griddep_wait();
        waited = true;
      }
      row_chunks<N2, SINGLE2>(d2, rv2, [&](const uint32_t* v, int, int col) {   // N2 % 32 == 0: full chunks
        uint32_t w[4];
#pragma unroll
        for (int c8 = 0; c8 < 4; ++c8) {
          float z[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            z[e] = fmaf(fma_sat(__uint_as_float(v[8 * c8 + e]), c15, B15), 15.0f, MAGIC - 8.0f);
          w[c8] = pack8(z);
        }
        if (store) *reinterpret_cast<uint4*>(qrow + col / 2) = make_uint4(w[0], w[1], w[2], w[3]);
        if constexpr (WRITE_Y) {
          if (store) {
            float2* yd = reinterpret_cast<float2*>(y_out + t * (N1 * N2) + i * N2 + col);   // 8-B aligned (ABI)
#pragma unroll
            for (int e = 0; e < 16; ++e)
              yd[e] = make_float2(__uint_as_float(v[2 * e]) * inv_pre * inv_p2,
                                  __uint_as_float(v[2 * e + 1]) * inv_pre * inv_p2);
          }
        }
      });
      tc::fence_before();
      if constexpr (C::ALIAS_D) {                        // D2 read out: the group's columns are free
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&d2free[par]);
      }
      if (store && i == 0) {
        if constexpr (ASYM) {
          scale[t] = mp > 0.f ? alpha * (mp * inv_pre * inv_p2) / 15.0f : 1.0f;
          zero[t] = int8_t(int(zq) - 8);
        } else {
          scale[t] = mp > 0.f ? alpha * (mp * inv_pre * inv_p2) / 7.0f : 1.0f;
        }
      }
      if (L == 0 && k < 16) trace(104 + k);
    }
  }

  tc::fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    trace(120);
    cta_stamp(1);
  }
  if (threadIdx.x == 4 * 32) trace(121);
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, C::TMEM_COLS);
    if (lane == 0) trace(123);
  }
}

// ------------------------------------------------------------------------------ host side
static unsigned* tq_sync_slot() {
  static unsigned* base[64] = {nullptr};
  static std::atomic<uint32_t> next[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!base[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_tq_sync) != cudaSuccess) return nullptr;
    base[dev] = static_cast<unsigned*>(p);
  }
  return base[dev] + 2 * (next[dev].fetch_add(1, std::memory_order_relaxed) % TQ_SLOTS);
}

static int multi_tpc() {                           // FQ_TQ_MULTI=<tiles per CTA>: experiment (MULTI)
  static const int v = [] {
    const char* e = std::getenv("FQ_TQ_MULTI");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  return v;
}

static bool small_enabled() {                      // FQ_TQ_SMALL=0: testing aid (large config)
  static const bool on = [] {
    const char* v = std::getenv("FQ_TQ_SMALL");
    return !(v && v[0] == '0');
  }();
  return on;
}

template <int N1, int N2, bool BF16, bool WRITE_Y, bool ASYM = false, int SMALL = 0, bool IDENT2 = false>
static cudaError_t launch(const TQArgs& a) {
  using C = Cfg<N1, N2, SMALL, IDENT2>;
  auto kern = tq_tc05_kernel<N1, N2, BF16, WRITE_Y, ASYM, SMALL, IDENT2>;
  static std::atomic<uint64_t> attr_done{0};   // devices configured for this kernel
  if (cudaError_t e = ensure_smem_attr(kern, int(C::SMEM), attr_done); e != cudaSuccess) return e;
  CUtensorMap mx, m1, m2;
  {
    const uint64_t dims[3] = {uint64_t(N2), uint64_t(N1), uint64_t(a.T)};
    const uint64_t strides[2] = {uint64_t(N2) * 2, uint64_t(a.ldx) * 2};
    const uint32_t box[3] = {64, uint32_t(N1), uint32_t(C::TOK)};
    if (!tmap_encode(&mx, a.x, 2, 3, dims, strides, box, TMAP_SW128)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {uint64_t(N1), uint64_t(N1)};
    const uint64_t strides[1] = {uint64_t(N1) * 2};
    const uint32_t box[2] = {64, uint32_t(N1)};
    if (!tmap_encode(&m1, a.p1, 2, 2, dims, strides, box, TMAP_SW128)) return cudaErrorInvalidValue;
  }
  if (IDENT2) {
    m2 = m1;                                       // unused
  } else {
    const uint64_t dims[2] = {uint64_t(N2), uint64_t(N2)};
    const uint64_t strides[1] = {uint64_t(N2) * 2};
    const uint32_t box[2] = {64, uint32_t(N2)};
    if (!tmap_encode(&m2, a.p2, 2, 2, dims, strides, box, TMAP_SW128)) return cudaErrorInvalidValue;
  }
  const int64_t tiles = (a.T + C::TOK - 1) / C::TOK;
  constexpr bool DYN = !SMALL && !IDENT2;
  unsigned* tsync = nullptr;
  int grid;
  if (DYN) {                                      // static first chunk of 2 tiles per CTA, then claims
    grid = int(std::min<int64_t>((tiles + 1) / 2, num_sms()));
    tsync = tq_sync_slot();
    if (!tsync) return cudaErrorInvalidValue;
  } else {
    grid = SMALL == 2 ? int((tiles + multi_tpc() - 1) / multi_tpc()) : int(std::min<int64_t>(tiles, num_sms()));
  }
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(C::THREADS), C::SMEM, a.stream, 1, mx, m1, m2, a.T, a.alpha,
                             a.q, a.scale, a.y, a.zero, a.pdl, tsync);
  count_launch();
  return e;
}

template <int N1>
static cudaError_t dispatch_ident2(const TQArgs& a) {     // P2 = I, n2 = 128
  if (a.zero) return a.bf16 ? launch<N1, 128, true, false, true, false, true>(a)
                            : launch<N1, 128, false, false, true, false, true>(a);
  if (a.bf16) return a.y ? launch<N1, 128, true, true, false, false, true>(a) : launch<N1, 128, true, false, false, false, true>(a);
  return a.y ? launch<N1, 128, false, true, false, false, true>(a) : launch<N1, 128, false, false, false, false, true>(a);
}

template <int N1, int N2>
static cudaError_t dispatch(const TQArgs& a) {
  if (a.zero) return a.bf16 ? launch<N1, N2, true, false, true>(a) : launch<N1, N2, false, false, true>(a);
  if (a.T <= 64 && !a.y && small_enabled())       // decode (C4) launches: one tile per CTA
    return a.bf16 ? launch<N1, N2, true, false, false, 1>(a) : launch<N1, N2, false, false, false, 1>(a);
  if (multi_tpc() > 0 && !a.y)                    // experiment: a few tiles per CTA, several CTAs per SM
    return a.bf16 ? launch<N1, N2, true, false, false, 2>(a) : launch<N1, N2, false, false, false, 2>(a);
  if (a.bf16) return a.y ? launch<N1, N2, true, true>(a) : launch<N1, N2, true, false>(a);
  return a.y ? launch<N1, N2, false, true>(a) : launch<N1, N2, false, false>(a);
}

}  // namespace tq5

#ifdef FQ_TRACE
extern "C" int fq_debug_trace_tq(unsigned long long* out, int n) {
  if (n > tq5::TRACE_CTAS * tq5::TRACE_EV) n = tq5::TRACE_CTAS * tq5::TRACE_EV;
  return int(cudaMemcpyFromSymbol(out, tq5::g_trace, sizeof(unsigned long long) * n));
}
extern "C" int fq_debug_cta_tq(unsigned long long* out) {   // [1024][start, end]
  return int(cudaMemcpyFromSymbol(out, tq5::g_cta, sizeof(unsigned long long) * 2048));
}
extern "C" int fq_debug_stamp(int slot, void* stream) {     // globaltimer into stamp slot (0..7)
  tq5::stamp_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(slot);
  return int(cudaGetLastError());
}
extern "C" int fq_debug_stamps(unsigned long long* out) {
  return int(cudaMemcpyFromSymbol(out, tq5::g_stamp, sizeof(unsigned long long) * 8));
}
#endif

bool tq_tc05_supported(const TQArgs& a) {
  const bool shape = a.p2 == nullptr ? (a.n2 == 128 && (a.n1 == 32 || a.n1 == 64))   // P2 = I
                                     : (a.n1 == 64 && (a.n2 == 64 || a.n2 == 128)) ||
                                           (a.n2 == 128 && (a.n1 == 80 || a.n1 == 96 || a.n1 == 112 || a.n1 == 128));
  const bool al = ((reinterpret_cast<uintptr_t>(a.x) | reinterpret_cast<uintptr_t>(a.p1) |
                    reinterpret_cast<uintptr_t>(a.p2) | reinterpret_cast<uintptr_t>(a.q)) & 15u) == 0 &&
                  (a.ldx * 2) % 16 == 0 && a.T < (int64_t(1) << 31);
  return shape && al && tmap_available();
}

cudaError_t tq_tc05_launch(const TQArgs& a) {
  using namespace tq5;
  if (a.p2 == nullptr) {
    if (a.n1 == 32 && a.n2 == 128) return dispatch_ident2<32>(a);
    if (a.n1 == 64 && a.n2 == 128) return dispatch_ident2<64>(a);
    return cudaErrorInvalidValue;
  }
  if (a.n1 == 64 && a.n2 == 64) return dispatch<64, 64>(a);
  if (a.n1 == 64 && a.n2 == 128) return dispatch<64, 128>(a);
  if (a.n1 == 80 && a.n2 == 128) return dispatch<80, 128>(a);
  if (a.n1 == 96 && a.n2 == 128) return dispatch<96, 128>(a);
  if (a.n1 == 112 && a.n2 == 128) return dispatch<112, 128>(a);
  if (a.n1 == 128 && a.n2 == 128) return dispatch<128, 128>(a);
  return cudaErrorInvalidValue;
}

}  // namespace fq
