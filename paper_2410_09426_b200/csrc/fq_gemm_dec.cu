// fq_gemm_dec.cu -- W4A4 GEMM + dequant for SMALL token counts (decode, T <= 64) on tcgen05.
//
//   acc[t,o] = sum_k qa[t,k] qw[o,k]               (Eq.3; PAPER.md:315 INT4 GEMM)
//   y[t,o]   = cvt_rn(float(acc) * sa[t] * sw[o])  (per-token x per-channel)
//
// At decode (64 tokens per step) the linear layer is bound by the weight
// bytes, not by the tensor pipe: a 256-token pair tile would waste 3/4 of every MMA and leave
// most SMs idle (48 qkv tiles of 128 features on 148 SMs).  This kernel therefore
//   * swaps the operands: the MMA's M side is 128 weight rows (output features), its N side the
//     T <= 64 tokens (N = T rounded up to 16), D[o][t] in TMEM;
//   * splits K across a thread-block CLUSTER of S CTAs (S <= 8) working on the same 128 features,
//     and reduces the S int32 partial tiles through distributed shared memory (exact: integer
//     addition, so the result is bit-identical for every S);
//   * sizes every CTA to two per SM (about 110 KB shared memory, 64 TMEM columns), so that the
//     whole grid (num_feature_blocks x S <= 2 x SMs) is resident at once and every CTA streams an
//     equal share of the weights -- no partial last wave;
//   * issues the TMA loads of its first weight stages BEFORE griddepcontrol.wait, so the weight
//     stream overlaps the tail of the transform kernel that produces the activation codes (PDL).
// Same INT4 -> INT8 widening contract as the other GEMMs (x16 per operand, the accumulator holds
// 256 acc exactly; the K permutation inside each 32-element group is identical for both operands).
//
//   warp 0      : TMA producer (packed weights + packed activations, PSTAGES-deep ring)
//   warp 1      : MMA issuer (one thread, tcgen05.mma.cta_group::1.kind::i8, both operands smem)
//   warp 2      : TMEM allocator
//   warps 4-7   : TMEM -> shared-memory partial tile (lane quarter = warp % 4)
//   warps 8-15  : converters: packed rows -> widened SWIZZLE_128B K-major operands
//   all warps   : cluster reduction of the partial tiles + dequant epilogue (coalesced stores)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"
#include "fq_tc05.cuh"
#include "fq_quant.cuh"

namespace fq {
namespace gd {

// Optional device timeline of 4 CTAs (build with -DFQ_TRACE; scripts/trace_dec.py): globaltimer
// stamps of [0] start, [1] setup done, [2] TMA issue of stage j (4+j), converters done (40+j),
// MMA issued (76+j), [112] tfull, [113] partial tile stored, [114] reduced, [115] end; FUSED: [116]
// phase-A X tile landed, [119] stage-1 epilogue done, [117] tile counted, [118] all tiles counted.
#ifdef FQ_TRACE
__device__ unsigned long long g_dtrace[4 * 128];
__device__ int g_dtrace_cta[4];
FQ_DEVICE void dtrace(int slot, int ev) {
  if (slot >= 0 && ev < 128) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    g_dtrace[slot * 128 + ev] = t;
  }
}
#else
FQ_DEVICE void dtrace(int, int) {}
#endif

constexpr int BM = 128;                       // output features per CTA (MMA M)
constexpr int TN_MAX = 64;                    // tokens (MMA N, multiple of 16)
#ifndef FQ_DEC_BK
#define FQ_DEC_BK 128
#endif
constexpr int BK = FQ_DEC_BK;                 // int8 K per stage (128: one 128-byte swizzle atom, 256: two)
constexpr int KA = BK / 128;                  // swizzle atoms per widened row
constexpr int CPR = BK / 32;                  // packed 16-byte chunks per row and stage
constexpr int UK = 32;                        // K per tcgen05.mma kind::i8
#ifndef FQ_DEC_STAGES
#define FQ_DEC_STAGES 2
#endif
#ifndef FQ_DEC_PSTAGES
#define FQ_DEC_PSTAGES 5
#endif
#ifndef FQ_DEC_MINB
#define FQ_DEC_MINB 2
#endif
#ifndef FQ_DEC_TMEMW
#define FQ_DEC_TMEMW 1
#endif
// FQ_DEC_TMEMW: the widened weights go to TMEM (the MMA's A operand straight from tensor memory,
// tcgen05.st by one converter thread per weight row), only the widened activations to shared
// memory -- 6 MMA stages in flight instead of 2 within the same shared-memory budget.
constexpr bool TMEMW = FQ_DEC_TMEMW != 0;
#ifndef FQ_DEC_TSTAGES
#define FQ_DEC_TSTAGES 6
#endif
constexpr int STAGES = TMEMW ? FQ_DEC_TSTAGES : FQ_DEC_STAGES;   // widened operand stages
constexpr int PSTAGES = FQ_DEC_PSTAGES;       // packed TMA ring
#ifndef FQ_DEC_BATCH
#define FQ_DEC_BATCH 2
#endif
constexpr int DB = FQ_DEC_BATCH;              // K-blocks converted per synchronisation (TMEMW path)
static_assert(DB >= 1 && DB < FQ_DEC_PSTAGES, "batch within the packed ring");
constexpr int WP_BYTES = BM * BK / 2;         // packed weights per stage (8 KB at BK = 128)
constexpr int AP_BYTES = TN_MAX * BK / 2;     // packed activations per stage (max)
constexpr int P_BYTES = WP_BYTES + AP_BYTES;  // ring stage (1 KB multiple)
constexpr int WW_BYTES = BM * BK;             // widened weights per stage (16 KB at BK = 128)
constexpr int AW_BYTES = TN_MAX * BK;         // widened activations per stage
constexpr int WW_ATOM = BM * 128, AW_ATOM = TN_MAX * 128;   // one 128-byte K atom of each
constexpr int W_BYTES = (TMEMW ? 0 : WW_BYTES) + AW_BYTES;   // shared-memory bytes per MMA stage
constexpr int W_COL0 = 64;                    // TMEM: accumulator [0, 64), weight stages after it
constexpr int WT_COLS = BK / 4;               // TMEM columns per weight stage (4 int8 per column)
constexpr int RED_BYTES = TN_MAX * BM * 4;    // 32 KB int32 partial tile [token][feature]
constexpr int TMA_WARP = 0, MMA_WARP = 1, ALLOC_WARP = 2;
constexpr int EPI_WARP0 = 4;                  // warps 4-7 (TMEM lane quarter = warp % 4)
constexpr int CONV_WARP0 = 8, NUM_CONV_WARPS = 8;
constexpr int THREADS = (CONV_WARP0 + NUM_CONV_WARPS) * 32;
constexpr int CONV_THREADS = NUM_CONV_WARPS * 32;
// TMEMW: warps 8-11 widen the weights into TMEM; the activations are widened by warps 12-15 AND
// the epilogue warps 4-7 (idle until the last MMA), one 16-byte chunk per thread at T = 64
#ifndef FQ_DEC_L2PF
#define FQ_DEC_L2PF 0
#endif
#ifndef FQ_DEC_L2PF_WIDE
#define FQ_DEC_L2PF_WIDE 0    // warp 3 prefetches the CTA's weight slice into L2: 1 TMA boxes, 2 LSU lines
#endif
#ifndef FQ_DEC_EPI_CONV
#define FQ_DEC_EPI_CONV 0     // round 2: the converter warps alone are as fast (C4 74.7 vs 77.9 us)
#endif
constexpr bool EPI_CONV = FQ_DEC_EPI_CONV != 0;            // epilogue warps help widen activations
constexpr int A_CONV_THREADS = EPI_CONV ? 256 : 128;
constexpr int NUM_ARRIVE = TMEMW ? (EPI_CONV ? 12 : 8) : NUM_CONV_WARPS;   // converter warps signalling per stage
constexpr int TMEM_COLS = TMEMW ? 256 : 64;
constexpr int MAX_SPLIT = 8;                  // portable cluster size
constexpr size_t SMEM_BYTES = size_t(STAGES) * W_BYTES + size_t(PSTAGES) * P_BYTES + 1024 + 256;
static_assert(RED_BYTES <= STAGES * W_BYTES, "the partial tile reuses the widened-operand stages");

// Two resident-CTA configurations, picked per shape at launch (round 2): CFG 0 -- two CTAs per SM,
// 6 MMA stages, a 5-deep packed ring (the shapes with more feature blocks than SMs: gate/up); CFG 1
// -- one CTA per SM, 4 MMA stages and a 14-deep packed ring (112 KB of weights in flight per CTA,
// prefetched before the PDL wait): the decode GEMM streams weights at the rate its bytes in flight
// allow (Little's law, ~1.3 us per round trip), and the shapes with few feature blocks cannot fill
// two CTAs per SM under cluster residency limits.
#ifndef FQ_DEC_S1
#define FQ_DEC_S1 4
#endif
#ifndef FQ_DEC_KP1
#define FQ_DEC_KP1 2
#endif
#ifndef FQ_DEC_P1
#define FQ_DEC_P1 (FQ_DEC_KP1 == 2 ? 7 : 14)
#endif
template <int CFG, int FUSED = 0>
struct DecCfg {
  // FUSED: the transform tile of phase A borrows the widened-operand stages (48 KB), so the
  // one-CTA-per-SM configuration keeps at least 6 of them
  static constexpr int STAGES = CFG == 0 ? gd::STAGES : ((FUSED && FQ_DEC_S1 < 6) ? 6 : FQ_DEC_S1);
  static constexpr int PSTAGES = CFG == 0 ? gd::PSTAGES : FQ_DEC_P1;
  // K-blocks per packed ring stage: 2 loads 128-byte rows (one TMA row request per 128 B instead
  // of per 64 B: the TMA unit's request rate, not HBM, paced the one-CTA-per-SM main loop)
  static constexpr int KP = (CFG == 0 || !TMEMW) ? 1 : FQ_DEC_KP1;
  static constexpr int PB = KP * P_BYTES;                     // packed ring stage bytes
  static constexpr int WPB = KP * WP_BYTES;                   // weight part of a ring stage
  static constexpr int MINB = CFG == 0 ? FQ_DEC_MINB : 1;
  // accumulator [0, 64) + one 32-column weight stage per MMA stage (a power of two >= 32)
  static constexpr int TMEM_COLS = !TMEMW ? 64 : (W_COL0 + STAGES * WT_COLS <= 256 ? 256 : 512);
  static constexpr size_t SMEM = size_t(STAGES) * W_BYTES + size_t(PSTAGES) * PB + 1024 + (FUSED ? 512 : 256);
  static_assert(RED_BYTES <= STAGES * W_BYTES, "partial tile in the operand stages");
  // phase A (the transform tile, fd_geo below): 64 x 64 in the widened-operand stages, 112 x 128 in
  // those stages plus the first packed ring stages (whose weights the ticket CTAs load afterwards)
#ifndef FQ_EXP_DEC_NOFUSED            // experiment builds that only time the plain decode GEMM
  static_assert(FUSED != 1 || STAGES * W_BYTES >= 48 * 1024, "64 x 64 phase A in the operand stages");
#endif
  static_assert(FUSED != 2 || STAGES * W_BYTES + PSTAGES * PB >= 88 * 1024, "112 x 128 phase A");
  static_assert(FUSED != 3 || STAGES * W_BYTES + PSTAGES * PB >= 72 * 1024, "64 x 128 phase A");
  static_assert(!TMEMW || W_COL0 + STAGES * WT_COLS <= TMEM_COLS, "TMEM budget");
  static_assert(MINB == 1 || TMEM_COLS <= 256, "two CTAs per SM share the 512 TMEM columns");
  static_assert(SMEM * MINB <= 232448, "shared memory per SM");
  static_assert(DB < PSTAGES * KP, "batch within the packed ring");
  static_assert(KP == 1 || DB == KP, "a conversion batch is one ring stage");
};
static_assert(P_BYTES % 1024 == 0 && W_BYTES % 1024 == 0 && WW_BYTES % 1024 == 0, "1 KB alignment");
static_assert(!TMEMW || (BK == 128 && W_COL0 + STAGES * WT_COLS <= TMEM_COLS), "TMEM budget");

FQ_DEVICE void widen8(uint32_t p, uint32_t& lo, uint32_t& hi) {   // 8 nibbles -> 8 x (16 q) int8
  lo = (p << 4) & 0xF0F0F0F0u;
  hi = p & 0xF0F0F0F0u;
}

FQ_DEVICE uint4 ld_cluster128(uint32_t local_addr, uint32_t cta) {
  uint4 v;
  asm volatile(
      "{\n.reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %4, %5;\n"
      "ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [ra];\n}\n"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "r"(local_addr), "r"(cta)
      : "memory");
  return v;
}

// One packed 16-byte chunk (32 codes) of row `row` -> 32 widened bytes at K positions 32c..32c+31
// of a SWIZZLE_128B K-major operand (K atom c / 4 at atom_bytes stride; 16-byte chunk ^= row % 8).
FQ_DEVICE void convert_chunk(uint32_t src, uint32_t dst_rows, int row, int c, int atom_bytes) {
  const uint4 pk = tc::lds128(src);
  uint32_t o[8];
  widen8(pk.x, o[0], o[1]);
  widen8(pk.y, o[2], o[3]);
  widen8(pk.z, o[4], o[5]);
  widen8(pk.w, o[6], o[7]);
  const uint32_t rowp = dst_rows + uint32_t((c >> 2) * atom_bytes + row * 128);
  const int cc = c & 3;
  tc::sts128(rowp + uint32_t(((2 * cc) ^ (row & 7)) << 4), o[0], o[1], o[2], o[3]);
  tc::sts128(rowp + uint32_t(((2 * cc + 1) ^ (row & 7)) << 4), o[4], o[5], o[6], o[7]);
}

// ---- fused decode linear (NEXT-4(i)): transform + quantize inside the GEMM launch ----
// The first `ntiles` CTAs of the grid ("ticket" CTAs) each transform one two-token tile
// (n1 = n2 = 64: Y_t = P1^T V_t P2, Eq.3) exactly as fq_tq_tc05.cu's kernel does
// (same tcgen05 MMAs, same fp16 intermediate with the power-of-two prescale, same quantizer from
// fq_quant.cuh), write the codes and scales to the caller's workspace (L2-resident at decode
// sizes), and count themselves into a per-launch counter; every CTA streams its weight slice from
// the start of the kernel and loads the activation codes once the count is complete.  The
// counter pair (arrivals, departures) lives in a ring of slots in this module's device memory
// and is reset by the last CTA to leave, so a slot is reusable by a later launch (and by a CUDA
// graph replay).  Ticket CTAs are the lowest block indices; the launcher runs the fused kernel
// only when the whole grid fits on the device at once (larger grids take the two-kernel path),
// so the tickets can always run whatever order the blocks are dispatched in.
constexpr int FD_SLOTS = 1024;
__device__ unsigned g_fd_sync[2 * FD_SLOTS];

struct alignas(64) FdParams {
  CUtensorMap tmX, tmP1, tmP2;   // x [T][n1][n2] (box 64 x n1 x TOK tokens), P1, P2 (SWIZZLE_128B)
  float alpha;
  uint8_t* q;                    // [T, n/2] packed codes (the caller's q_ws)
  float* s;                      // [T] scales (s_ws)
  unsigned* sync;                // {arrivals, departures} of this launch's slot
  int ntiles;                    // ticket CTAs = ceil(T / TOK)
  int bf16x;                     // x, P1, P2 are bf16 (stage 2 runs in fp16 with P2 scaled, as K1)
};
// Phase-A geometry (the same tiles as fq_tq_tc05.cu): F = 1 -> n1 = n2 = 64, two tokens per tile;
// F = 2 -> 112 x 128 (LLaMA-3-8B down_proj), one token; F = 3 -> 64 x 128 (n = 8192, e.g. the
// 70B models' attention and MLP inputs), two tokens as two M = 128 stage-1 groups.  Layout in shared
// memory from offset 0: F = 1: X | P1 | P2 | A2 (48 KB, the widened-operand stages); F = 2, 3:
// P2 | P1 | X with the stage-2 operand A2 written over P1 + X once the stage-1 MMA has read them
// (88 / 72 KB, into the first packed ring stages).
template <int F>
struct FdGeo {
  static constexpr int N1 = F == 2 ? 112 : 64, N2 = F == 1 ? 64 : 128;
  static constexpr int TOK = N1 == 64 ? 2 : 1;
  static constexpr int G1 = TOK * N2 / 128;                // stage-1 MMA groups (M = 128) per tile
  static constexpr int JB = N2 / 64, P1_ATOMS = (N1 + 63) / 64;
  static constexpr int X_BYTES = TOK * JB * N1 * 128, P1_BYTES = P1_ATOMS * N1 * 128, P2_BYTES = JB * N2 * 128;
  static constexpr int A2_BYTES = 2 * N2 * 128;
  static constexpr bool ALIAS = F != 1;
  static constexpr int OFF_P2 = ALIAS ? 0 : X_BYTES + P1_BYTES;
  static constexpr int OFF_P1 = ALIAS ? P2_BYTES : X_BYTES;
  static constexpr int OFF_X = ALIAS ? P2_BYTES + P1_BYTES : 0;
  static constexpr int OFF_A2 = ALIAS ? OFF_P1 : X_BYTES + P1_BYTES + P2_BYTES;
  static constexpr int BYTES = ALIAS ? P2_BYTES + P1_BYTES + X_BYTES : OFF_A2 + A2_BYTES;
  static constexpr int LOAD_BYTES = X_BYTES + P1_BYTES + P2_BYTES;
  static constexpr uint32_t IDESC1 = tc::idesc_f16(128, N1, 0, 1, 1);   // fp16 x fp16 -> fp32, MN-major
  static constexpr uint32_t IDESC1_BF16 = tc::idesc_f16(128, N1, 1, 1, 1);
  static constexpr uint32_t IDESC2 = tc::idesc_f16(128, N2, 0, 1, 1);
  static_assert(G1 == 1 || (N1 == 64 && N2 == 128), "two stage-1 groups only at 64 x 128");
  static_assert(!ALIAS || A2_BYTES <= P1_BYTES + X_BYTES, "A2 over P1 + X");
};

FQ_DEVICE unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FQ_DEVICE void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
FQ_DEVICE void red_release_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
FQ_DEVICE void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }

template <int CFG, bool OUT_I32, bool BF16, bool ASYM, int FUSED = 0>
__global__ void __launch_bounds__(THREADS, DecCfg<CFG, FUSED>::MINB)
gemm_dec_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA,
                const __grid_constant__ CUtensorMap tmWpf, const uint8_t* __restrict__ qwp,
                const float* __restrict__ sa, int T, int TN, int K, const float* __restrict__ sw, int N,
                void* __restrict__ yv, const int8_t* __restrict__ za, const int32_t* __restrict__ colsum,
                int S, int pdl, const __grid_constant__ FdParams fd) {
  constexpr int STAGES = DecCfg<CFG, FUSED>::STAGES, PSTAGES = DecCfg<CFG, FUSED>::PSTAGES;
  constexpr int KP = DecCfg<CFG, FUSED>::KP, PB = DecCfg<CFG, FUSED>::PB, WPB = DecCfg<CFG, FUSED>::WPB;
  constexpr int PROW = KP * (BK / 2);                        // packed bytes of one row in a ring stage
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;                                        // widened stages [W 16 KB | A 8 KB]
  uint8_t* sP = smem + size_t(STAGES) * W_BYTES;             // packed ring    [W 8 KB | A 4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + size_t(PSTAGES) * PB);
  uint64_t* full = bars;                   // [STAGES]  converters -> MMA
  uint64_t* empty = bars + STAGES;         // [STAGES]  MMA commit -> converters
  uint64_t* pfull = bars + 2 * STAGES;     // [PSTAGES] TMA (weights) -> converters
  uint64_t* pempty = pfull + PSTAGES;      // [PSTAGES] converter warps -> TMA
  uint64_t* afull = pempty + PSTAGES;      // [PSTAGES] TMA (activation codes) -> converters: the weights
                                           //           of a stage are widened as soon as they land,
                                           //           whether or not the codes exist yet (FUSED)
  uint64_t* tfull = afull + PSTAGES;       // [1]       last MMA commit -> partial-tile warps
  uint64_t* fdx = tfull + 1;               // FUSED: X tile + P1 + P2 landed (ticket CTAs)
  uint64_t* fd1 = fdx + 1;                 //        stage-1 MMA commit -> epilogue warps
  uint64_t* fda2 = fd1 + 1;                //        stage-1 epilogue (4 warps) -> stage-2 MMA
  uint64_t* fd2 = fda2 + 1;                //        stage-2 MMA commit -> epilogue warps
  uint64_t* actready = fd2 + 1;            //        all tickets counted: codes and scales visible
  uint64_t* fdone = actready + 1;          //        F = 2: phase-A buffers free (ring stages usable)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1 + (FUSED ? 6 : 0));
  using FG = FdGeo<FUSED == 0 ? 1 : FUSED>;
  // FUSED phase A borrows the widened-operand stages (and, F = 2, the first packed ring stages)
  uint8_t* fsX = smem + FG::OFF_X;
  uint8_t* fsP1 = smem + FG::OFF_P1;
  uint8_t* fsP2 = smem + FG::OFF_P2;
  uint8_t* fsA2 = smem + FG::OFF_A2;
  __shared__ float fd_red[8];                                // [2 parities][4 warps] token maxima
  const bool ticket = FUSED && int(blockIdx.x) < fd.ntiles;
  __shared__ float s_sa[TN_MAX];                             // sa[t] / 256 (0 past T)
  __shared__ int s_za[TN_MAX];                               // 256 (z_t - 8) (asymmetric)
  __shared__ __align__(16) float s_sw[BM];                  // sw of this feature block
  __shared__ __align__(16) int s_cs[BM];                     // colsum_w of this feature block

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tslot = blockIdx.x < 2 ? int(blockIdx.x) : (blockIdx.x + 2 >= gridDim.x ? int(blockIdx.x + 4 - gridDim.x) : -1);
  if (threadIdx.x == 0) dtrace(tslot, 0);
  const int rank = S > 1 ? int(tc::cluster_ctarank()) : 0;
  const int fb = blockIdx.x / S;                             // feature block of this cluster
  // units of KP K-blocks ("super-blocks", one packed ring stage each) are split across the cluster;
  // a super-block's K-blocks past K are zero-filled by TMA and contribute nothing
  const int NKB = (K + BK * KP - 1) / (BK * KP);
  const int kb0 = rank * NKB / S, kb1 = (rank + 1) * NKB / S, nsb = kb1 - kb0, nk = nsb * KP;
  // Every CTA reads the same few KB of activation codes per K-block; walking the K-blocks in the
  // same order would make all CTAs hit the same L2 lines at the same time.  Each CTA starts at a
  // different K-block instead (integer accumulation: the order does not change the result).
  const int krot = nsb > 0 ? int((unsigned(fb) * 5u + unsigned(rank) * 3u) % unsigned(nsb)) : 0;
  auto kb_of = [&](int u) { const int r = u + krot; return kb0 + (r >= nsb ? r - nsb : r); };   // super-block
  const uint32_t idesc = tc::idesc_i8(BM, TN);
#ifdef FQ_EXP_DEC_NOACT            // experiment builds only: activation codes not loaded (timing)
  const int ap_bytes = 0;
#else
  const int ap_bytes = TN * (BK / 2);
#endif

  if (warp == MMA_WARP && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], NUM_ARRIVE);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < PSTAGES; ++s) {
      tc::mbar_init(&pfull[s], 1);
      tc::mbar_init(&afull[s], 1);
      tc::mbar_init(&pempty[s], NUM_ARRIVE);
    }
    tc::mbar_init(tfull, 1);
    if constexpr (FUSED) {
      tc::mbar_init(fd1, 1);
      tc::mbar_init(fda2, 4);
      tc::mbar_init(fd2, 1);
      tc::mbar_init(actready, 1);
      tc::mbar_init(fdone, 4);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch_desc(&tmW);
    tc::tma_prefetch_desc(&tmA);
    if (ticket) {
      tc::tma_prefetch_desc(&fd.tmX);
      tc::tma_prefetch_desc(&fd.tmP1);
      tc::tma_prefetch_desc(&fd.tmP2);
    }
  }
  // FUSED, ticket CTAs: the phase-A loads leave first, before the setup barrier, when x, P1 and P2
  // may be read before the PDL wait (otherwise after the weights, in the producer loop below)
  const bool early_x = ticket && (pdl & (PDL_P | PDL_X)) == (PDL_P | PDL_X);
  auto fd_load = [&] {                       // this CTA's tile of x, P1 and P2 (fq_tq_tc05.cu boxes)
    tc::mbar_expect_tx(fdx, uint32_t(FG::LOAD_BYTES));
#pragma unroll
    for (int b = 0; b < FG::JB; ++b)
      tc::tma_load_3d(fsX + b * FG::TOK * FG::N1 * 128, &fd.tmX, fdx, b * 64, 0, FG::TOK * int(blockIdx.x));
#pragma unroll
    for (int a = 0; a < FG::P1_ATOMS; ++a) tc::tma_load_2d(fsP1 + a * FG::N1 * 128, &fd.tmP1, fdx, a * 64, 0);
#pragma unroll
    for (int b = 0; b < FG::JB; ++b) tc::tma_load_2d(fsP2 + b * FG::N2 * 128, &fd.tmP2, fdx, b * 64, 0);
  };
  if (FUSED && ticket && warp == TMA_WARP && lane == 0) {
    tc::mbar_init(fdx, 1);
    tc::fence_barrier_init();
    if (early_x) fd_load();
  }
  if (warp == ALLOC_WARP) tc::tmem_alloc(tmem_slot, DecCfg<CFG, FUSED>::TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) dtrace(tslot, 1);

  // activation rows (TN x 4 chunks) -> widened SWIZZLE_128B K-major stage, by 256 threads
  // (at = 0..255: epilogue warps 4-7 and converter warps 12-15)
  // Both converter paths work on DB K-blocks per iteration and synchronise once per batch (one
  // fence / tcgen05.wait::st for the DB stages), so DB K-blocks are in conversion at a time: a
  // single K-block's wait -> load -> widen -> store -> fence -> signal chain is latency-bound
  // (~0.27 us on the B200, scripts/trace_dec.py), far longer than its share of the weight stream.
  auto convert_a = [&](int at) {
    for (int j0 = 0; j0 < nk; j0 += DB) {
      const int nb = nk - j0 < DB ? nk - j0 : DB;
#pragma unroll
      for (int b = 0; b < DB; ++b) {
        if (b < nb) {
          const int j = j0 + b, u = j / KP, h = j % KP, sp = u % PSTAGES, st = j % STAGES;
          tc::mbar_wait(&empty[st], ((j / STAGES) & 1) ^ 1);
          tc::mbar_wait(&afull[sp], (u / PSTAGES) & 1);
          const uint32_t src = smem_u32(sP + size_t(sp) * PB + WPB);
          const uint32_t dst = smem_u32(sW + size_t(st) * W_BYTES);
#ifndef FQ_EXP_DEC_SKIPA          // (experiment build: activation conversion removed)
          for (int task = at; task < TN * CPR; task += A_CONV_THREADS) {
            const int row = task / CPR, c = task % CPR;
            // KP 1: dense 64-byte rows; KP 2: 128-byte SWIZZLE_128B rows, this K-block's half
            const uint32_t a = KP == 1 ? uint32_t(task * 16)
                                       : uint32_t(row * PROW + (((h * CPR + c) ^ (row & 7)) << 4));
            convert_chunk(src + a, dst, row, c, AW_ATOM);
          }
#endif
          __syncwarp();
          if (lane == 0 && h == KP - 1) tc::mbar_arrive(&pempty[sp]);
        }
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
#pragma unroll
      for (int b = 0; b < DB; ++b)
        if (b < nb && lane == 0) tc::mbar_arrive(&full[(j0 + b) % STAGES]);
    }
  };

  if (warp == TMA_WARP) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      if (FG::ALIAS && ticket) {
        // the 112 x 128 / 64 x 128 phase-A tile occupies the first packed ring stages: this CTA's weights
        // stream only once its transform tile is done (the other CTAs' from kernel start)
        if (!early_x) {
          tc::griddep_wait();
          fd_load();
        }
        tc::mbar_wait(fdone, 0);
      }
      // the weights are parameters: unless the preceding kernel of the stream writes them
      // (host-side hazard check, fq_abi.cu), start streaming them before the wait
      if (!(pdl & PDL_P)) tc::griddep_wait();
      const int pre = nsb < PSTAGES ? nsb : PSTAGES;          // ring stages (super-blocks)
#if FQ_DEC_L2PF
      // the rest of this CTA's weight slice into L2 now (one bulk tensor prefetch per K-block):
      // the ring's loads then hit L2 instead of waiting a full HBM round trip each
      for (int j = pre; j < nsb; ++j) tc::tma_prefetch_l2_2d(&tmW, kb_of(j) * PROW, fb * BM);
#endif
      for (int j = 0; j < pre; ++j) {
        if (j < 36) dtrace(tslot, 4 + j);
        tc::mbar_expect_tx(&pfull[j], uint32_t(WPB));
        tc::tma_load_2d(sP + size_t(j) * PB, &tmW, &pfull[j], kb_of(j) * PROW, fb * BM);
      }
      if (FUSED == 1 && ticket && !early_x) {     // phase-A loads that had to wait for the predecessor
        tc::griddep_wait();
        fd_load();
      }
      if constexpr (FUSED) {
        // every ticket CTA has stored its codes and scales (release/acquire at GPU scope); the
        // activation codes are then read through the async proxy (TMA)
        const unsigned need = unsigned(fd.ntiles);
        const long long t_start = clock64();
        // relaxed polling (an acquire load per poll invalidates L1 each time), one acquire fence
        while (ld_relaxed_gpu(fd.sync) < need) {
          if (clock64() - t_start > (1ll << 36)) __trap();    // never hang the GPU: ~35 s without progress
        }
        fence_acq_rel_gpu();
        fence_proxy_async_global();
        dtrace(tslot, 118);
        tc::mbar_arrive(actready);
        // last CTA out resets the slot for its next launch (all arrivals have been counted)
        if (atomicAdd(fd.sync + 1, 1u) == gridDim.x - 1) {
          atomicExch(fd.sync, 0u);
          atomicExch(fd.sync + 1, 0u);
        }
      } else if (!(pdl & PDL_X)) {
        tc::griddep_wait();                      // qa written by the transform kernel is visible
      }
      for (int j = 0; j < pre; ++j) {
        tc::mbar_expect_tx(&afull[j], uint32_t(KP * ap_bytes));
        if (ap_bytes) tc::tma_load_2d(sP + size_t(j) * PB + WPB, &tmA, &afull[j], kb_of(j) * PROW, 0);
      }
      for (int j = pre; j < nsb; ++j) {
        const int sp = j % PSTAGES;
        tc::mbar_wait(&pempty[sp], ((j / PSTAGES) & 1) ^ 1);
        if (j < 36) dtrace(tslot, 4 + j);
        uint8_t* dst = sP + size_t(sp) * PB;
        tc::mbar_expect_tx(&pfull[sp], uint32_t(WPB));
        tc::tma_load_2d(dst, &tmW, &pfull[sp], kb_of(j) * PROW, fb * BM);
        tc::mbar_expect_tx(&afull[sp], uint32_t(KP * ap_bytes));
        if (ap_bytes) tc::tma_load_2d(dst + WPB, &tmA, &afull[sp], kb_of(j) * PROW, 0);
      }
    }
    __syncwarp();
  } else if (warp >= CONV_WARP0) {
    // ======================= converters =======================
    // tasks per stage: BM weight rows x 4 chunks, then TN activation rows x 4 chunks; a warp's
    // 32 tasks cover 8 consecutive rows (conflict-free 16-byte loads and swizzled stores)
    const int ct = threadIdx.x - CONV_WARP0 * 32;
    const int ntask = (BM + TN) * CPR;
    if constexpr (TMEMW) {
      if (warp < CONV_WARP0 + 4) {
        // weight rows: one per thread (TMEM lane), packed row from the SWIZZLE_64B ring
        // (conflict-free) -> widened in registers -> tcgen05.st into this stage's TMEM columns
        const int q = warp & 3, r = q * 32 + lane;
        const uint32_t tl = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(W_COL0);
        for (int j0 = 0; j0 < nk; j0 += DB) {
          const int nb = nk - j0 < DB ? nk - j0 : DB;
#pragma unroll
          for (int b = 0; b < DB; ++b) {
            if (b < nb) {
              const int j = j0 + b, u = j / KP, h = j % KP, sp = u % PSTAGES, st = j % STAGES;
              tc::mbar_wait(&empty[st], ((j / STAGES) & 1) ^ 1);
              tc::mbar_wait(&pfull[sp], (u / PSTAGES) & 1);
              const uint32_t src = smem_u32(sP + size_t(sp) * PB) + uint32_t(r * PROW);
              uint32_t w[32];
#ifdef FQ_EXP_DEC_SKIPW           // experiment build only: weight conversion removed
              if (true) {
                __syncwarp();
                if (lane == 0 && h == KP - 1) tc::mbar_arrive(&pempty[sp]);
                continue;
              }
#endif
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                // KP 1: SWIZZLE_64B 64-byte rows; KP 2: SWIZZLE_128B 128-byte rows, this block's half
                const int pos = KP == 1 ? (c ^ ((r >> 1) & 3)) : ((h * 4 + c) ^ (r & 7));
                const uint4 pk = tc::lds128(src + uint32_t(pos << 4));
                widen8(pk.x, w[8 * c + 0], w[8 * c + 1]);
                widen8(pk.y, w[8 * c + 2], w[8 * c + 3]);
                widen8(pk.z, w[8 * c + 4], w[8 * c + 5]);
                widen8(pk.w, w[8 * c + 6], w[8 * c + 7]);
              }
              tc::tmem_st32(tl + uint32_t(st * WT_COLS), w);
              __syncwarp();
              if (lane == 0 && h == KP - 1) tc::mbar_arrive(&pempty[sp]);   // loads consumed by the st
            }
          }
          tc::tmem_st_wait();
          tc::fence_before();
          __syncwarp();
#pragma unroll
          for (int b = 0; b < DB; ++b)
            if (b < nb && lane == 0) tc::mbar_arrive(&full[(j0 + b) % STAGES]);
          if (threadIdx.x == CONV_WARP0 * 32 && j0 < 36) dtrace(tslot, 40 + j0);
        }
      } else {
        convert_a(threadIdx.x - (CONV_WARP0 + 4) * 32 + (EPI_CONV ? 128 : 0));
      }
    } else {
    for (int j = 0; j < nk; ++j) {
      const int sp = j % PSTAGES, st = j % STAGES;
      tc::mbar_wait(&empty[st], ((j / STAGES) & 1) ^ 1);
      tc::mbar_wait(&pfull[sp], (j / PSTAGES) & 1);
      tc::mbar_wait(&afull[sp], (j / PSTAGES) & 1);
      const uint32_t src = smem_u32(sP + size_t(sp) * PB);
      const uint32_t dst = smem_u32(sW + size_t(st) * W_BYTES);
      for (int task = ct; task < ntask; task += CONV_THREADS) {
        const int row = task / CPR, c = task % CPR;
        if (row < BM) convert_chunk(src + uint32_t(task * 16), dst, row, c, WW_ATOM);
        else convert_chunk(src + uint32_t(WP_BYTES + (task - CPR * BM) * 16), dst + WW_BYTES, row - BM, c, AW_ATOM);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&pempty[sp]);   // packed slot consumed (stored above)
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full[st]);
      if (threadIdx.x == CONV_WARP0 * 32 && j < 36) dtrace(tslot, 40 + j);
    }
    }
  } else if (warp == 3) {
#if FQ_DEC_L2PF_WIDE == 2
    // LSU variant: every lane prefetches 128-byte lines of its rows (no TMA-engine time)
    if (!(pdl & PDL_P)) tc::griddep_wait();
    {
      const int pre = nsb < PSTAGES ? nsb : PSTAGES;
      const size_t ld = size_t(K / 2);
      for (int u = pre; u < nsb; ++u) {
        const int kb = kb_of(u);
        const size_t off = size_t(kb) * PROW;
        if (PROW < 128 && (off & 127)) continue;              // this half-line came with the previous block
        for (int r = lane; r < BM; r += 32) {
          const uint8_t* pa = qwp + size_t(fb * BM + r) * ld + off;
          if (fb * BM + r < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(pa));
        }
      }
    }
#elif FQ_DEC_L2PF_WIDE
    // ======================= L2 prefetch of this CTA's weight slice =======================
    // The packed ring keeps only ~5 K-blocks per CTA in flight (Little's law at the HBM latency
    // under load: ~30 GB/s per CTA); bulk prefetches into L2 (no shared memory, 256-byte x 128-row
    // boxes, a few instructions per CTA) keep the rest of the slice in flight, so the ring's loads
    // hit L2.  Consumption order (the rotated K walk), from the first block the ring prefill misses.
    if (lane == 0) {
      if (!(pdl & PDL_P)) tc::griddep_wait();
      const int per = 256 / PROW;                           // super-blocks per prefetch box
      const int pre = nsb < PSTAGES ? nsb : PSTAGES;
      for (int u = pre; u < nsb;) {
        const int kb = kb_of(u);
        int run = 1;                                        // consecutive super-blocks (no wrap)
        while (run < per && u + run < nsb && kb_of(u + run) == kb + run) ++run;
        tc::tma_prefetch_l2_2d(&tmWpf, kb * PROW, fb * BM);
        u += run;
      }
    }
#endif
    __syncwarp();
  } else if (warp == MMA_WARP) {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      if (ticket) {
        // phase A (fq_tq_tc05.cu's MMAs, M = 128: two tokens at 64 x 64, one at 112 x 128): D =
        // (X^T P1) into TMEM columns [0, n1) -- the accumulator columns, unused until the first GEMM
        // MMA (which follows every ticket's epilogue); at 112 x 128 also the first two weight
        // stages, which this CTA fills only after phase A (fdone) -- then D = W P2 into columns
        // [0, n2) once the stage-1 epilogue has read D and written W (fp16) to shared memory
        tc::mbar_wait(fdx, 0);
        tc::fence_after();
        dtrace(tslot, 116);
        const uint32_t xs = smem_u32(fsX), p1a = smem_u32(fsP1), p2a = smem_u32(fsP2), a2 = smem_u32(fsA2);
        constexpr uint32_t XLBO = FG::N2 == 64 ? FG::N1 * 128 : FG::TOK * FG::N1 * 128;
#pragma unroll
        for (int g = 0; g < FG::G1; ++g) {               // 64 x 128: token g's M = 128 rows (j)
          const uint32_t a0 = xs + uint32_t(FG::N2 == 64 ? 0 : g * FG::N1 * 128);
#pragma unroll
          for (int kk = 0; kk < FG::N1 / 16; ++kk)
            tc::mma_ss<false>(tmem_base + uint32_t(g * FG::N1), tc::sdesc_sw128(a0 + kk * 2048, XLBO, 1024),
                              tc::sdesc_sw128(p1a + kk * 2048, FG::N1 * 128, 1024),
                              fd.bf16x ? FG::IDESC1_BF16 : FG::IDESC1, kk > 0);
        }
        tc::mma_commit(fd1);
        tc::mbar_wait(fda2, 0);
        tc::fence_after();
        dtrace(tslot, 119);
#pragma unroll
        for (int kk = 0; kk < FG::N2 / 16; ++kk)
          tc::mma_ss<false>(tmem_base, tc::sdesc_sw128(a2 + kk * 2048, FG::N2 * 128, 1024),
                            tc::sdesc_sw128(p2a + kk * 2048, FG::N2 * 128, 1024), FG::IDESC2, kk > 0);
        tc::mma_commit(fd2);
      }
      for (int j = 0; j < nk; ++j) {
        const int st = j % STAGES;
        tc::mbar_wait(&full[st], (j / STAGES) & 1);
        tc::fence_after();
        const uint32_t w0 = smem_u32(sW + size_t(st) * W_BYTES);
        if constexpr (TMEMW) {
          const uint32_t wt = tmem_base + uint32_t(W_COL0 + st * WT_COLS);
#ifndef FQ_EXP_DEC_NMMA
#define FQ_EXP_DEC_NMMA (BK / UK)      // experiment builds only: fewer MMAs per K-block (timing)
#endif
#pragma unroll
          for (int k = 0; k < FQ_EXP_DEC_NMMA; ++k)
            tc::mma_ts<true>(tmem_base, wt + uint32_t(k * (UK / 4)), tc::sdesc_sw128(w0 + k * UK, 16, 1024), idesc,
                             (j | k) != 0);
        } else {
#pragma unroll
        for (int k = 0; k < BK / UK; ++k)
          tc::mma_ss<true>(tmem_base, tc::sdesc_sw128(w0 + (k >> 2) * WW_ATOM + (k & 3) * UK, 16, 1024),
                           tc::sdesc_sw128(w0 + WW_BYTES + (k >> 2) * AW_ATOM + (k & 3) * UK, 16, 1024), idesc,
                           (j | k) != 0);
        }
        tc::mma_commit(&empty[st]);
        if (j < 36) dtrace(tslot, 76 + j);
      }
      tc::mma_commit(tfull);
    }
    __syncwarp();
  } else if (warp >= EPI_WARP0) {
    // ======================= TMEM -> shared-memory partial tile =======================
    if constexpr (FUSED) {
      if (ticket) {
        // ---- phase A epilogues (fq_tq_tc05.cu's, one group of 4 warps, 16-column TMEM chunks) ----
        const int qd = warp & 3, L = qd * 32 + lane;
        const uint32_t lb = tmem_base + (uint32_t(qd * 32) << 16);
        int rp = 0;
        auto exchange = [&](float m) {                     // per-warp max -> the 4 warps' maxima
          m = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(m)));   // m >= 0
          if (lane == 0) fd_red[rp * 4 + qd] = m;
          named_bar_sync(1, 128);
          const float4 r = make_float4(fd_red[rp * 4 + 0], fd_red[rp * 4 + 1], fd_red[rp * 4 + 2], fd_red[rp * 4 + 3]);
          rp ^= 1;
          return r;
        };
        auto ld16 = [&](int c, uint32_t(&v)[16]) {
          tc::tmem_ld16(lb + uint32_t(c), v);
          tc::tmem_ld_wait();
        };
        constexpr int N1 = FG::N1, N2 = FG::N2, TOK = FG::TOK;
        // bf16 x / P: stage 2 runs in fp16 (R9), so P2 becomes fp16 P2 2^e2 in place
        // (K1's power-of-two scaling into fp16 range) while the stage-1 MMA runs; 2^-e2 is
        // divided out of the statistics exactly.  The stage-2 MMA reads P2 only after fda2 below.
        float inv_p2 = 1.0f;
        if (fd.bf16x) {
          __shared__ uint32_t fd_p2max;
          tc::mbar_wait(fdx, 0);
          inv_p2 = qz::exp2i(-bf16_to_f16_pow2_group(fsP2, FG::P2_BYTES / 2, &fd_p2max, L, 128, 1));
        }
        // stage 1: D lane (t, j), column i = W_t[i][j] (64 x 64: token t = L / 64; 64 x 128: token g
        // of stage-1 group g spans all 128 lanes)
        tc::mbar_wait(fd1, 0);
        tc::fence_after();
        int pe0 = 0, pe1 = 0;
#pragma unroll
        for (int g = 0; g < FG::G1; ++g) {
          const uint32_t dg = uint32_t(g * N1);
          float m1 = 0.f;
#pragma unroll
          for (int c = 0; c < N1; c += 16) {
            uint32_t v[16];
            ld16(int(dg) + c, v);
#pragma unroll
            for (int e = 0; e < 16; e += 2)
              m1 = qz::max3f(m1, fabsf(__uint_as_float(v[e])), fabsf(__uint_as_float(v[e + 1])));
          }
          const float4 r1 = exchange(m1);
          const float all = fmaxf(fmaxf(r1.x, r1.y), fmaxf(r1.z, r1.w));
          if (N2 == 64) {                                  // two tokens in the lane halves
            pe0 = qz::prescale_exp(fmaxf(r1.x, r1.y));
            pe1 = qz::prescale_exp(fmaxf(r1.z, r1.w));
          } else if (g == 0) {
            pe0 = qz::prescale_exp(all);
            pe1 = pe0;
          } else {
            pe1 = qz::prescale_exp(all);
          }
          const int tg = N2 == 64 ? (L >> 6) : g;          // token of this thread's row in group g
          const float pre = qz::exp2i(tg ? pe1 : pe0);
          const int j = N2 == 64 ? (L & 63) : L;           // K row j' of the stage-2 A operand
          const uint32_t row = smem_u32(fsA2) + uint32_t(j * 128);
#pragma unroll
          for (int c = 0; c < N1; c += 16) {
            uint32_t v[16];
            ld16(int(dg) + c, v);
#pragma unroll
            for (int e = 0; e < 16; e += 8) {
              const int c8 = (c + e) >> 3, ch = c8 & 7;
              const int atom = N1 == 64 ? tg : (c8 >> 3);    // 64-element M atoms of A2
              tc::sts128(row + uint32_t(atom * (N2 * 128) + ((ch ^ (j & 7)) << 4)),
                         pack_half2(__uint_as_float(v[e + 0]) * pre, __uint_as_float(v[e + 1]) * pre),
                         pack_half2(__uint_as_float(v[e + 2]) * pre, __uint_as_float(v[e + 3]) * pre),
                         pack_half2(__uint_as_float(v[e + 4]) * pre, __uint_as_float(v[e + 5]) * pre),
                         pack_half2(__uint_as_float(v[e + 6]) * pre, __uint_as_float(v[e + 7]) * pre));
            }
          }
        }
        const int tt = TOK == 2 ? (L >> 6) : 0;            // stage 2: token of this thread's row
        tc::fence_proxy_async_smem();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(fda2);
        // stage 2: D lane (t, i), column j = Y_t[i][j] (prescaled by 2^pe); 112 x 128: lanes >= 112
        // hold no row (their A2 rows were never written) and are left out of the statistics
        tc::mbar_wait(fd2, 0);
        tc::fence_after();
        if (L == 0) dtrace(tslot, 120);
        const bool valid = N1 == 64 || L < N1;
        float m2 = 0.f;
#pragma unroll
        for (int c = 0; c < N2; c += 16) {
          uint32_t v[16];
          ld16(c, v);
#pragma unroll
          for (int e = 0; e < 16; e += 2)
            m2 = qz::max3f(m2, fabsf(__uint_as_float(v[e])), fabsf(__uint_as_float(v[e + 1])));
        }
        const float4 r2 = exchange(valid ? m2 : 0.f);
        const float mp = TOK == 2 ? (tt == 0 ? fmaxf(r2.x, r2.y) : fmaxf(r2.z, r2.w))
                                  : fmaxf(fmaxf(r2.x, r2.y), fmaxf(r2.z, r2.w));
        const int t = TOK * int(blockIdx.x) + tt, i = N1 == 64 ? (L & 63) : L;
        const bool store = valid && t < T;
        const float inv_pre = qz::exp2i(-(tt ? pe1 : pe0));
        const float c15 = qz::sym_c15(fd.alpha, mp);
        if (!(pdl & PDL_OUT)) tc::griddep_wait();          // the predecessor no longer reads q_ws / s_ws
        uint8_t* qrow = fd.q + (store ? size_t(t) * (N1 * N2 / 2) + size_t(i) * (N2 / 2) : 0);
#pragma unroll
        for (int c = 0; c < N2; c += 32) {
          uint32_t v[32];
          tc::tmem_ld16(lb + uint32_t(c), *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
          tc::tmem_ld16(lb + uint32_t(c + 16), *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
          tc::tmem_ld_wait();
          uint32_t w[4];
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            float z[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) z[e] = qz::sym_code(__uint_as_float(v[8 * c8 + e]), c15);
            w[c8] = qz::pack8(z);
          }
          if (store) *reinterpret_cast<uint4*>(qrow + c / 2) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if (store && i == 0) fd.s[t] = mp > 0.f ? fd.alpha * (mp * inv_pre * inv_p2) / 7.0f : 1.0f;
        if constexpr (FG::ALIAS) {                         // TMEM and the phase-A buffers are free
          tc::fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(fdone);
        }
        if (L == 0) dtrace(tslot, 121);
        fence_proxy_async_global();                        // (the consumers read the codes through TMA)
        tc::fence_before();
        named_bar_sync(1, 128);
        if (L == 0) {
          dtrace(tslot, 122);
          // the group's stores happen before this release through the barrier (bar.sync orders
          // them at CTA scope; the GPU-scope release is cumulative), as in CUTLASS's grid barrier
          red_release_gpu_add(fd.sync, 1u);                // this tile is done
          dtrace(tslot, 117);
        }
      }
    }
    // while the main loop runs: stage the epilogue's scales in shared memory
    tc::griddep_wait();
    if (threadIdx.x == EPI_WARP0 * 32) tc::griddep_launch();   // only after the wait (fq_internal.h)
    {
      const int e = threadIdx.x - EPI_WARP0 * 32;          // 0..127
      const int o = fb * BM + e;
      if constexpr (!OUT_I32) {
        s_sw[e] = o < N ? __ldg(sw + o) : 0.f;
        if constexpr (ASYM) s_cs[e] = o < N ? __ldg(colsum + o) : 0;
        if (e < TN_MAX) {
          if constexpr (FUSED) tc::mbar_wait(actready, 0);     // the scales come from the tickets
          s_sa[e] = e < T ? (FUSED ? __ldcg(sa + e) : sa[e]) * (ASYM ? 1.0f : 1.0f / 256.0f) : 0.f;
          if constexpr (ASYM) s_za[e] = e < T ? int(za[e]) : 0;
        }
      }
    }
    if constexpr (TMEMW && EPI_CONV) convert_a(threadIdx.x - EPI_WARP0 * 32);
    tc::mbar_wait(tfull, 0);
    tc::fence_after();
    if (threadIdx.x == EPI_WARP0 * 32) dtrace(tslot, 112);
    const int q = warp & 3, f = q * 32 + lane;
    int32_t* red = reinterpret_cast<int32_t*>(sW);           // [token][BM] (MMAs have finished)
    if constexpr (DecCfg<CFG>::MINB == 1) {
      // all of this lane's accumulator columns in one TMEM round trip, then the stores (the
      // one-CTA-per-SM configuration has the registers for it)
      uint32_t v[TN_MAX];
#pragma unroll
      for (int c = 0; c < TN_MAX / 16; ++c)
        if (c < TN / 16) tc::tmem_ld16(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(c * 16),
                                       *reinterpret_cast<uint32_t(*)[16]>(v + c * 16));
      tc::tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < TN_MAX / 16; ++c)
        if (c < TN / 16)
#pragma unroll
          for (int i = 0; i < 16; ++i) red[(c * 16 + i) * BM + f] = int32_t(v[c * 16 + i]);
    } else {
      for (int c = 0; c < TN / 16; ++c) {
        uint32_t v[16];
        tc::tmem_ld16(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(c * 16), v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) red[(c * 16 + i) * BM + f] = int32_t(v[i]);
      }
    }
  }

  // ======================= cluster reduction + dequant epilogue (all warps) =======================
  tc::griddep_wait();                          // sa / za of the previous kernel are visible to every thread
  tc::fence_before();
  __syncthreads();
  if (S > 1) tc::cluster_sync();               // every CTA's partial tile is in its shared memory
  if (threadIdx.x == 0) dtrace(tslot, 113);
  {
    const int groups = TN * (BM / 4);          // 4 consecutive features of one token per group
    const int g0 = rank * groups / S, g1 = (rank + 1) * groups / S;
    const uint32_t red0 = smem_u32(sW);
    for (int g = g0 + int(threadIdx.x); g < g1; g += THREADS) {
      const int t = g / (BM / 4), f0 = (g % (BM / 4)) * 4;
      const int o = fb * BM + f0;
      int4 acc = make_int4(0, 0, 0, 0);
      if (S == 1) {
        const uint4 p = tc::lds128(red0 + uint32_t(g * 16));
        acc = make_int4(int(p.x), int(p.y), int(p.z), int(p.w));
      } else {
        // all S remote loads in flight before the first add (integer sums: order-free, exact)
        uint4 p[MAX_SPLIT];
#pragma unroll
        for (int r = 0; r < MAX_SPLIT; ++r)
          if (r < S) p[r] = ld_cluster128(red0 + uint32_t(g * 16), uint32_t(r));
#pragma unroll
        for (int r = 0; r < MAX_SPLIT; ++r)
          if (r < S) {
            acc.x += int(p[r].x);
            acc.y += int(p[r].y);
            acc.z += int(p[r].z);
            acc.w += int(p[r].w);
          }
      }
      if (t >= T || o >= N) continue;          // N % 8 == 0: a group is all in or all out
      if constexpr (OUT_I32) {
        *reinterpret_cast<int4*>(static_cast<int32_t*>(yv) + size_t(t) * N + o) =
            make_int4(acc.x >> 8, acc.y >> 8, acc.z >> 8, acc.w >> 8);
      } else {
        if constexpr (ASYM) {                  // acc_true = acc - (z - 8) colsum_w after the exact >> 8
          const int zc = s_za[t];              // (TMEM held 256 acc), so no int32 wrap for K < 131072
          const int4 cs = *reinterpret_cast<const int4*>(s_cs + f0);
          acc.x = (acc.x >> 8) - zc * cs.x;
          acc.y = (acc.y >> 8) - zc * cs.y;
          acc.z = (acc.z >> 8) - zc * cs.z;
          acc.w = (acc.w >> 8) - zc * cs.w;
        }
        const float s_a = s_sa[t];
        const float4 w = *reinterpret_cast<const float4*>(s_sw + f0);
        const float f0v = float(acc.x) * s_a * w.x, f1v = float(acc.y) * s_a * w.y;
        const float f2v = float(acc.z) * s_a * w.z, f3v = float(acc.w) * s_a * w.w;
        uint2 out;
        if constexpr (BF16) {
          __nv_bfloat162 h0 = __floats2bfloat162_rn(f0v, f1v), h1 = __floats2bfloat162_rn(f2v, f3v);
          out = make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
          *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(yv) + size_t(t) * N + o) = out;
        } else {
          out = make_uint2(pack_half2(f0v, f1v), pack_half2(f2v, f3v));
          *reinterpret_cast<uint2*>(static_cast<__half*>(yv) + size_t(t) * N + o) = out;
        }
      }
    }
  }
  if (threadIdx.x == 0) dtrace(tslot, 114);
  if (S > 1) tc::cluster_sync();               // peers have finished reading this CTA's tile
  else __syncthreads();
  if (threadIdx.x == 0) dtrace(tslot, 115);
  if (warp == ALLOC_WARP) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_base, DecCfg<CFG, FUSED>::TMEM_COLS);
  }
}

}  // namespace gd

#ifdef FQ_TRACE
extern "C" int fq_debug_trace_dec(unsigned long long* out) {
  return int(cudaMemcpyFromSymbol(out, gd::g_dtrace, sizeof(unsigned long long) * 512));
}
#endif

bool gemm_dec_supported(const GemmArgs& a) {
  return a.T >= 1 && a.T <= gd::TN_MAX && a.K % 32 == 0 && a.K < 131072 && a.N % 8 == 0 && tmap_available();
}

static int dec_policy() {                         // FQ_DEC_POLICY: testing aid (0/1/2)
  static const int p = [] {
    const char* v = std::getenv("FQ_DEC_POLICY");
    return v ? std::atoi(v) : 2;
  }();
  return p;
}

// CTAs of a kernel resident on one SM at once, from its threads, registers, shared memory and
// TMEM columns.  (cudaOccupancyMaxActiveBlocksPerMultiprocessor reports 1 for every kernel that
// contains tcgen05.alloc, whatever its resources; scripts/probes/occ_tc05.cu measures 2-4 such
// CTAs running concurrently on one SM, so the limits are computed here.)
static int resident_ctas_per_sm(const void* kern, int threads, size_t dyn_smem, int tmem_cols) {
  cudaFuncAttributes fa{};
  int dev = 0, thr = 0, regs = 0, smem = 0, rsv = 0;
  if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&thr, cudaDevAttrMaxThreadsPerMultiProcessor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&regs, cudaDevAttrMaxRegistersPerMultiprocessor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  const int warps = (threads + 31) / 32;
  const int regs_per_warp = ((fa.numRegs * 32 + 255) / 256) * 256;   // 256-register allocation unit
  const size_t smem_per_cta = dyn_smem + fa.sharedSizeBytes + size_t(rsv);
  int n = std::min({thr / threads, regs / std::max(1, regs_per_warp * warps), int(size_t(smem) / smem_per_cta),
                    512 / std::max(32, tmem_cols)});
  return std::max(1, n);
}

// How many clusters of S CTAs the hardware keeps resident at once (cluster placement is bounded
// by the GPC structure, not only by the per-SM limits); cached per (configuration, S).
template <int CFG, int FUSED>
static int dec_max_clusters(const void* kern, int S) {
  static int cache[gd::MAX_SPLIT + 1] = {0};
  if (S <= 1) return gd::DecCfg<CFG, FUSED>::MINB * num_sms();
  if (cache[S] > 0) return cache[S];
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(S * 64));
  cfg.blockDim = dim3(gd::THREADS);
  cfg.dynamicSmemBytes = gd::DecCfg<CFG, FUSED>::SMEM;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(S);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  int na = 1;
  if (dec_policy() > 0) {
    attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[1].val.clusterSchedulingPolicyPreference =
        dec_policy() == 1 ? cudaClusterSchedulingPolicySpread : cudaClusterSchedulingPolicyLoadBalancing;
    na = 2;
  }
  cfg.attrs = attr;
  cfg.numAttrs = unsigned(na);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = gd::DecCfg<CFG, FUSED>::MINB * num_sms() / S;
  }
  cache[S] = n;
  return n;
}

// Split: the largest S <= 8 (and <= the number of K-blocks) for which every cluster of the grid
// is resident at once; shapes with more feature blocks than that run unsplit.
template <int CFG, int FUSED>
static int dec_pick_split(const void* kern, int N, int K) {
  const int fbs = (N + gd::BM - 1) / gd::BM;
  const int nkb = (K + gd::BK * gd::DecCfg<CFG, FUSED>::KP - 1) / (gd::BK * gd::DecCfg<CFG, FUSED>::KP);
  // at most one CTA per SM from the split (round 2): the second slot of every SM stays free for
  // the NEXT kernel of the stream, whose CTAs then start (PDL) and stream their weights while
  // this kernel drains -- measured: the C4 GEMM chain 64 -> 52 us
  static const int cap_per_sm = [] {               // FQ_DEC_GRIDCAP: testing aid (CTAs per SM of the grid)
    const char* v = std::getenv("FQ_DEC_GRIDCAP");
    return v ? std::atoi(v) : 1;
  }();
  const int per_sm = std::max(1, std::min(cap_per_sm, gd::DecCfg<CFG, FUSED>::MINB));
  int s = 1;
  for (int c = 2; c <= gd::MAX_SPLIT && c <= nkb; ++c)
    if (fbs * c <= per_sm * num_sms() && fbs <= dec_max_clusters<CFG, FUSED>(kern, c)) s = c;
  return s;
}

// device address of this launch's {arrivals, departures} slot (FUSED); slots are handed out
// round-robin per device, so up to FD_SLOTS fused launches may be in flight on a device at once
static unsigned* fd_sync_slot() {
  static unsigned* base[64] = {nullptr};
  static std::atomic<uint32_t> next[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!base[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, gd::g_fd_sync) != cudaSuccess) return nullptr;
    base[dev] = static_cast<unsigned*>(p);
  }
  return base[dev] + 2 * (next[dev].fetch_add(1, std::memory_order_relaxed) % gd::FD_SLOTS);
}

template <int CFG, int FUSED>
static cudaError_t dec_launch_cfg(const GemmArgs& a, int split, const FdArgs* f) {
  using namespace gd;
  using DC = DecCfg<CFG, FUSED>;
  const bool asym = a.za != nullptr && !a.out_i32;
  auto kern = a.out_i32 ? gemm_dec_kernel<CFG, true, false, false, FUSED>
              : asym    ? (a.y_bf16 ? gemm_dec_kernel<CFG, false, true, true, FUSED>
                                    : gemm_dec_kernel<CFG, false, false, true, FUSED>)
                        : (a.y_bf16 ? gemm_dec_kernel<CFG, false, true, false, FUSED>
                                    : gemm_dec_kernel<CFG, false, false, false, FUSED>);
  static std::atomic<uint64_t> attr_done[5];   // per kernel variant: devices configured
  const int which = a.out_i32 ? 0 : (a.y_bf16 ? 1 : 2) + (asym ? 2 : 0);
  const int TN = int((a.T + 15) / 16) * 16;
  CUtensorMap mw{}, ma{}, mwpf{};
  {
    const uint64_t dims[2] = {uint64_t(a.K / 2), uint64_t(a.N)};
    const uint64_t strides[1] = {uint64_t(a.K / 2)};
    const uint32_t box[2] = {uint32_t(DC::KP * BK / 2), BM};
    if (!tmap_encode(&mw, a.qw, 1, 2, dims, strides, box,
                     DC::KP == 2 ? TMAP_SW128 : (TMEMW ? TMAP_SW64 : TMAP_SW_NONE)))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {uint64_t(a.K / 2), uint64_t(a.N)};
    const uint64_t strides[1] = {uint64_t(a.K / 2)};
    const uint32_t box[2] = {uint32_t(std::min(256, a.K / 2)), BM};   // L2 prefetch boxes (32 KB)
    if (!tmap_encode(&mwpf, a.qw, 1, 2, dims, strides, box, TMAP_SW_NONE)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {uint64_t(a.K / 2), uint64_t(a.T)};
    const uint64_t strides[1] = {uint64_t(a.K / 2)};
    const uint32_t box[2] = {uint32_t(DC::KP * BK / 2), uint32_t(TN)};
    if (!tmap_encode(&ma, a.qa, 1, 2, dims, strides, box, DC::KP == 2 ? TMAP_SW128 : TMAP_SW_NONE))
      return cudaErrorInvalidValue;
  }
  const int nkb = (a.K + BK * DC::KP - 1) / (BK * DC::KP);     // ring stages of K
  int S = split > 0 ? split : dec_pick_split<CFG, FUSED>(reinterpret_cast<const void*>(kern), a.N, a.K);
  S = std::max(1, std::min({S, MAX_SPLIT, nkb}));
  const int fbs = (a.N + BM - 1) / BM;
  FdParams fd{};
  if constexpr (FUSED != 0) {
    using FG = FdGeo<FUSED>;
    // ticket CTAs: one per tile (TOK tokens), all within the (resident) grid
    fd.ntiles = int((a.T + FG::TOK - 1) / FG::TOK);
    if (fbs * S < fd.ntiles) return cudaErrorNotSupported;      // caller falls back (nothing launched)
    const uint64_t xd[3] = {uint64_t(FG::N2), uint64_t(FG::N1), uint64_t(a.T)};
    const uint64_t xs[2] = {uint64_t(FG::N2) * 2, uint64_t(f->ldx) * 2};
    const uint32_t xb[3] = {64, uint32_t(FG::N1), uint32_t(FG::TOK)};
    if (!tmap_encode(&fd.tmX, f->x, 2, 3, xd, xs, xb, TMAP_SW128)) return cudaErrorInvalidValue;
    {
      const uint64_t pd[2] = {uint64_t(FG::N1), uint64_t(FG::N1)};
      const uint64_t ps[1] = {uint64_t(FG::N1) * 2};
      const uint32_t pb[2] = {64, uint32_t(FG::N1)};
      if (!tmap_encode(&fd.tmP1, f->p1, 2, 2, pd, ps, pb, TMAP_SW128)) return cudaErrorInvalidValue;
    }
    {
      const uint64_t pd[2] = {uint64_t(FG::N2), uint64_t(FG::N2)};
      const uint64_t ps[1] = {uint64_t(FG::N2) * 2};
      const uint32_t pb[2] = {64, uint32_t(FG::N2)};
      if (!tmap_encode(&fd.tmP2, f->p2, 2, 2, pd, ps, pb, TMAP_SW128)) return cudaErrorInvalidValue;
    }
    fd.alpha = f->alpha;
    fd.bf16x = f->bf16 ? 1 : 0;
    fd.q = const_cast<uint8_t*>(a.qa);
    fd.s = const_cast<float*>(a.sa);
    fd.sync = fd_sync_slot();
    if (!fd.sync) return cudaErrorInvalidValue;
  }
  if (cudaError_t e = ensure_smem_attr(kern, int(DC::SMEM), attr_done[which]); e != cudaSuccess) return e;
  if constexpr (FUSED != 0) {
    // forward progress: the GEMM CTAs wait for the ticket CTAs, so the whole grid must fit on
    // the device at once (the CUDA model does not promise that blocks are dispatched in index
    // order); larger grids run the two kernels (nothing launched here)
    static std::atomic<int> occ[5];               // per kernel variant (0: not computed yet)
    if (occ[which].load(std::memory_order_relaxed) == 0)
      occ[which].store(resident_ctas_per_sm(reinterpret_cast<const void*>(kern), THREADS, DC::SMEM, DC::TMEM_COLS),
                       std::memory_order_relaxed);
    if (fbs * S > occ[which].load(std::memory_order_relaxed) * num_sms()) return cudaErrorNotSupported;
  }
  static const bool dbg = std::getenv("FQ_DEC_DEBUG") != nullptr;
  if (dbg)
    std::fprintf(stderr, "[fq] decode GEMM%s N=%d K=%d T=%lld: config %d, split %d, %d CTAs, max resident clusters %d\n",
                 FUSED ? " (fused transform)" : "", a.N, a.K, (long long)a.T, CFG, S, fbs * S,
                 dec_max_clusters<CFG, FUSED>(reinterpret_cast<const void*>(kern), S));
  cudaError_t e = launch_pdl_policy(kern, dim3(unsigned(fbs * S)), dim3(THREADS), DC::SMEM, a.stream, S,
                                    dec_policy(), mw, ma, mwpf, a.qw, a.sa, int(a.T), TN, a.K, a.sw, a.N, a.y, a.za, a.colsum, S,
                                    a.pdl, fd);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

static int dec_env_split() {                      // FQ_DEC_SPLIT: testing aid (forces S)
  static const int v = [] {
    const char* e = std::getenv("FQ_DEC_SPLIT");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
static bool dec_deep(const GemmArgs& a) {         // FQ_DEC_CFG: testing aid (forces 0 or 1)
  static const int env_cfg = [] {
    const char* v = std::getenv("FQ_DEC_CFG");
    return v ? std::atoi(v) : -1;
  }();
  // round 2: the two-CTAs-per-SM footprint everywhere (108 KB, 64 registers, 256 TMEM columns),
  // so that consecutive decode kernels co-reside; the deep-ring one-CTA-per-SM configuration
  // (FQ_DEC_CFG=1) kept its weights in flight but left no room for the next kernel
  return env_cfg == 1;
}

cudaError_t gemm_dec_launch(const GemmArgs& a, int split) {
  if (split <= 0) split = dec_env_split();
  return dec_deep(a) ? dec_launch_cfg<1, 0>(a, split, nullptr) : dec_launch_cfg<0, 0>(a, split, nullptr);
}

bool fused_dec_supported(const GemmArgs& a, int n1, int n2, bool x_bf16, const void* p2) {
  (void)x_bf16;                                    // fp16 and bf16 activations (bf16: P2 scaled, K1)
  const bool shape = (n1 == 64 && n2 == 64) || (n1 == 112 && n2 == 128) || (n1 == 64 && n2 == 128);
  return shape && p2 != nullptr && a.za == nullptr && !a.out_i32 && gemm_dec_supported(a) &&
         a.K == n1 * n2;
}

cudaError_t fused_dec_launch(const GemmArgs& a, const FdArgs& f) {
  const int split = dec_env_split();
  if (f.n1 == 112) return dec_deep(a) ? dec_launch_cfg<1, 2>(a, split, &f) : dec_launch_cfg<0, 2>(a, split, &f);
  if (f.n2 == 128) return dec_deep(a) ? dec_launch_cfg<1, 3>(a, split, &f) : dec_launch_cfg<0, 3>(a, split, &f);
  return dec_deep(a) ? dec_launch_cfg<1, 1>(a, split, &f) : dec_launch_cfg<0, 1>(a, split, &f);
}

}  // namespace fq
