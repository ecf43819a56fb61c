// fq_gemm_tc05_pair.cu -- W4A4 GEMM + dequant on a CTA PAIR (tcgen05.mma.cta_group::2 kind::i8).
//
//   acc[t,o] = sum_k qa[t,k] qw[o,k]               (Eq.3; PAPER.md:315 INT4 GEMM)
//   y[t,o]   = cvt_rn(float(acc) * sa[t] * sw[o])  (per-token x per-channel)
//
// Same int4 -> int8 widening contract as fq_gemm_tc05.cu (x16 per operand, acc/256 exact).
// Two SMs of a TPC cooperate on a 256 (tokens) x 192 (features) tile: each CTA holds its own
// 128 activation rows as the A operand in TMEM (widened by converter warps straight from
// registers with tcgen05.st) and HALF of the 192 weight rows (96) as the B operand in shared
// memory; the leader CTA issues one M=256 N=192 K=32 MMA for both.  Per SM this halves the
// shared-memory and L1 traffic per MAC relative to a single-CTA tile.
//   warps 0-3  : epilogue (own TMEM lanes -> dequant -> swizzled smem -> TMA bulk store)
//   warp  4    : TMEM allocator (both CTAs) + MMA issuer (leader CTA only)
//   warps 5-8  : A converters (FQ_GEMM_AWARPS), one activation row per thread: packed row from the
//                TMA ring (SWIZZLE_128B, conflict-free) -> widened in registers -> tcgen05.st into TMEM
//   warps 9-12 : B converters (FQ_GEMM_BWARPS), 16-byte packed chunks of the weight rows from the
//                ring -> widened SWIZZLE_128B K-major operand in shared memory
//   warp  13   : TMA producer of the packed A+B ring (PSTAGES K-blocks deep)
// (Round 2 measured the converter warp counts: 4 A + 4 B warps beat 8 + 6 by 3-8% on every C3
// shape -- fewer warps contend less for the shared-memory pipe -- scripts/gemm_shapes.py.)
// Loads are fully asynchronous (TMA, no registers, no LSU queue); per K-block and SM the shared-
// memory traffic is 14 KB (TMA) + 14 KB (converter reads) + 12 KB (widened B) + 12 KB (MMA read of
// B), the A operand never touches shared memory after conversion.
// Synchronisation: converters of both CTAs arrive (release.cluster) on the leader's `full`
// barrier; the leader's tcgen05.commit multicasts to both CTAs' `empty` / `tfull` barriers;
// both CTAs' epilogues arrive on the leader's `tempty` barrier.
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"
#include "fq_tc05.cuh"

namespace fq {
namespace g3 {

// Optional device timeline of the first CTA pair (build with -DFQ_TRACE; scripts/trace_gemm.py).
#ifdef FQ_TRACE
__device__ unsigned long long g_trace[2 * 256];
FQ_DEVICE void trace(int ev) {
  if (blockIdx.x < 2 && ev < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    g_trace[blockIdx.x * 256 + ev] = t;
  }
}
#else
FQ_DEVICE void trace(int) {}
#endif

constexpr int BM = 256, BM_CTA = 128;     // tokens per pair tile / per CTA
#ifndef FQ_GEMM_MAX_STAGES
#define FQ_GEMM_MAX_STAGES 4
#endif
#ifndef FQ_GEMM_PSTAGES
#define FQ_GEMM_PSTAGES 4       // cap on the packed ring depth (shared memory permitting)
#endif
#ifndef FQ_GEMM_BWARPS
#define FQ_GEMM_BWARPS 4     // measured best (round 2: 2-10 tried; fewer B warps, less contention)
#endif
#ifndef FQ_GEMM_BK
#define FQ_GEMM_BK 256
#endif
constexpr int BK = FQ_GEMM_BK;            // int8 K per stage: 256 (two 128-byte K atoms) or 128 (one)
static_assert(BK == 256 || BK == 128, "BK");
// the packed A ring row of one K-block is BK/2 bytes: SWIZZLE_128B rows (BK 256) or SWIZZLE_64B
constexpr int A_ROW = BK / 2;
constexpr int UK = 32;
constexpr int AP_BYTES = BM_CTA * BK / 2; // 8 KB packed A per ring stage
constexpr int EPI_BYTES = 32 * 128;       // per epilogue warp: 32 rows x 64 fp16 columns (SW128)
constexpr int A_COLS = BK / 4;            // TMEM columns per A stage
constexpr int TMEM_ACC0 = 0;              // two accumulators [0, 2*BN)
constexpr int TMEM_COLS = 512;
constexpr int NUM_EPI_WARPS = 4, MMA_WARP = 4;
#ifndef FQ_GEMM_AWARPS
#define FQ_GEMM_AWARPS 4     // measured best (round 2: 4 > 8 > 16; one full row per thread)
#endif
constexpr int A_WARP0 = 5, NUM_A_WARPS = FQ_GEMM_AWARPS;   // 4 warps per K part (one per TMEM lane quarter)
constexpr int A_PARTS = NUM_A_WARPS / 4;                   // K parts of a row: 2 (halves) or 4 (quarters)
constexpr int A_CH = (BK / 32) / A_PARTS;                  // packed 16-byte chunks per thread and K-block
static_assert(A_CH == 2 || A_CH == 4 || A_CH == 8, "A chunks per thread");
static_assert(NUM_A_WARPS == 4 || NUM_A_WARPS == 8 || NUM_A_WARPS == 16, "A converter warps: 4, 8 or 16");
constexpr int B_WARP0 = A_WARP0 + NUM_A_WARPS, NUM_B_WARPS = FQ_GEMM_BWARPS;
constexpr int NUM_CONV_WARPS = NUM_A_WARPS + NUM_B_WARPS;
constexpr int TMA_WARP = B_WARP0 + NUM_B_WARPS;
constexpr int THREADS = (TMA_WARP + 1) * 32;
constexpr int B_CHUNKS = BK / 32;                          // 16-byte packed chunks per weight row

// Tile width BN (features per pair tile) is a template parameter: the host picks it per shape to
// fill the last wave (fewer, narrower waves when N / 192 tiles would leave most clusters idle).
template <int BN>
struct Geo {
  static_assert(BN % 16 == 0 && BN >= 64 && BN <= 256, "BN: multiple of 16 in [64, 256] (MMA N at M = 256)");
  // up to 192 columns two accumulators fit beside the A stages (epilogue of tile i overlaps the
  // main loop of tile i+1); a 256-wide tile has one, and its epilogue is not overlapped
  static constexpr int NACC = BN <= 192 ? 2 : 1;
  static constexpr int BN_CTA = BN / 2;                    // B rows per CTA
  static constexpr int B_BYTES = BN_CTA * BK;              // widened B per stage per CTA
  static constexpr int BP_BYTES = BN_CTA * BK / 2;         // packed B per ring stage
  static constexpr int P_BYTES = AP_BYTES + BP_BYTES;
  static constexpr int TMEM_A0 = NACC * BN;                // A stages after the accumulator(s)
  static constexpr int B_ATOM = BN_CTA * 128;              // one 128-byte K atom of the widened B stage
  static constexpr int B_TOTAL = BN_CTA * B_CHUNKS;        // B conversion tasks per stage
  static constexpr int B_TASKS = (B_TOTAL + NUM_B_WARPS * 32 - 1) / (NUM_B_WARPS * 32);
  // MMA stages (TMEM A / widened smem B): as many as the TMEM left beside the accumulators holds
  // (192: 2, 160: 3, 128 and 256: 4); the packed TMA ring gets the shared memory that is left
  static constexpr int STAGES_FIT = (TMEM_COLS - NACC * BN) / A_COLS;
  static constexpr int STAGES = STAGES_FIT < FQ_GEMM_MAX_STAGES ? STAGES_FIT : FQ_GEMM_MAX_STAGES;
  static constexpr int SMEM_AVAIL = 232448 - 1024 - 512 - NUM_EPI_WARPS * EPI_BYTES - STAGES * B_BYTES;
  static constexpr int PSTAGES = SMEM_AVAIL / P_BYTES < FQ_GEMM_PSTAGES ? SMEM_AVAIL / P_BYTES : FQ_GEMM_PSTAGES;
  static constexpr size_t SMEM_BYTES =
      size_t(STAGES) * B_BYTES + size_t(PSTAGES) * P_BYTES + NUM_EPI_WARPS * EPI_BYTES + 1024 + 512;
  static_assert(STAGES >= 2 && PSTAGES >= 2, "pipeline depth");
  static constexpr uint32_t IDESC = tc::idesc_i8(BM, BN);
  static_assert(TMEM_A0 + STAGES * A_COLS <= TMEM_COLS, "TMEM budget");
  static_assert(B_ATOM % 1024 == 0 && P_BYTES % 1024 == 0, "SWIZZLE_128B atoms stay 1024-B aligned");
};

FQ_DEVICE void widen8(uint32_t p, uint32_t& lo, uint32_t& hi) {   // 8 nibbles -> 8 x (16 q) int8
  lo = (p << 4) & 0xF0F0F0F0u;
  hi = p & 0xF0F0F0F0u;
}

FQ_DEVICE void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

struct Sched {
  int num_m, num_n, num_tiles, num_kb, cluster, num_clusters;
  FQ_DEVICE void tile(int id, int& mb, int& nb) const {
    mb = id % num_m;
    nb = id / num_m;
  }
};

// Walks this cluster's (tile, k-block) job sequence without per-step divisions.
struct Cursor {
  int tile, kb, mb, nb;
  bool valid;
  FQ_DEVICE void init(const Sched& s) {
    tile = s.cluster;
    kb = 0;
    valid = tile < s.num_tiles;
    if (valid) s.tile(tile, mb, nb);
  }
  FQ_DEVICE void next(const Sched& s) {
    if (++kb == s.num_kb) {
      kb = 0;
      tile += s.num_clusters;
      valid = tile < s.num_tiles;
      if (valid) s.tile(tile, mb, nb);
    }
  }
};

template <int BN, bool OUT_I32, bool BF16, bool ASYM>
__global__ void __launch_bounds__(THREADS, 1)
gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmY32,
                 const __grid_constant__ CUtensorMap tmY16,
                 const float* __restrict__ sa, int T, int K, const float* __restrict__ sw, int N,
                 void* __restrict__ yv, const int8_t* __restrict__ za, const int32_t* __restrict__ colsum,
                 int pdl) {
  using GE = Geo<BN>;
  constexpr int BN_CTA = GE::BN_CTA, B_BYTES = GE::B_BYTES, P_BYTES = GE::P_BYTES, TMEM_A0 = GE::TMEM_A0;
  constexpr int B_ATOM = GE::B_ATOM, B_TASKS = GE::B_TASKS;
  constexpr int STAGES = GE::STAGES, PSTAGES = GE::PSTAGES;
  constexpr uint32_t IDESC = GE::IDESC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sP = smem + size_t(STAGES) * B_BYTES;                  // packed ring: [A 8 KB | B 6 KB]
  uint8_t* sEpi = sP + size_t(PSTAGES) * P_BYTES;                  // epilogue staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + NUM_EPI_WARPS * EPI_BYTES);
  uint64_t* full = bars;                 // [STAGES] leader: converters of both CTAs -> MMA
  uint64_t* empty = bars + STAGES;       // [STAGES] each CTA: MMA commit -> converters
  uint64_t* tfull = bars + 2 * STAGES;   // [2]      each CTA: MMA commit -> epilogue
  uint64_t* tempty = tfull + 2;          // [2]      leader: epilogues of both CTAs -> MMA
  uint64_t* pfull = tempty + 2;          // [PSTAGES] each CTA: TMA -> converters
  uint64_t* pempty = pfull + PSTAGES;    // [PSTAGES] each CTA: converter warps -> TMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + PSTAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) trace(250);
  const uint32_t rank = tc::cluster_ctarank();
  Sched sc;
  sc.num_m = (T + BM - 1) / BM;
  sc.num_n = (N + BN - 1) / BN;
  sc.num_tiles = sc.num_m * sc.num_n;
  sc.num_kb = (K + BK - 1) / BK;
  sc.cluster = blockIdx.x >> 1;
  sc.num_clusters = gridDim.x >> 1;
  const int KB = K / 2;

  if (warp == MMA_WARP) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        tc::mbar_init(&full[s], 2 * NUM_CONV_WARPS);  // one arrival per converter warp of the pair
        tc::mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        tc::mbar_init(&tfull[b], 1);
        tc::mbar_init(&tempty[b], 2);
      }
      for (int s = 0; s < PSTAGES; ++s) {
        tc::mbar_init(&pfull[s], 1);
        tc::mbar_init(&pempty[s], NUM_CONV_WARPS);
      }
      tc::fence_barrier_init();
      if constexpr (!OUT_I32) {
        tc::tma_prefetch_desc(&tmY);
        if constexpr (BN % 64 != 0) tc::tma_prefetch_desc(&tmY32);
      }
      tc::tma_prefetch_desc(&tmA);
      tc::tma_prefetch_desc(&tmB);
    }
    __syncwarp();
    tc::tmem_alloc2(tmem_slot, TMEM_COLS);
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();            // peer barriers initialised before any remote arrive
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL (round 2c): only the TMA thread waits for the preceding kernel -- after it has requested
  // the weight (B) halves of its first ring stages, when the host found the weights are not
  // written by that kernel (PDL_P).  Everything else in this kernel is ordered after the wait
  // through the ring: the converters, the MMAs, and the epilogue (which reads sa and writes y)
  // all consume activation data the TMA thread requested after its wait.

  // Every converter warp signals the leader's `full` barrier on its own (CTA-scope arrive in the
  // leader, release.cluster remote arrive from the peer), so the A and B paths and the warps of
  // each path run decoupled, up to STAGES K-blocks apart; no CTA-wide barrier per stage.
  int jtrace = 0;
  auto signal_full = [&](uint64_t* bar) {
    __syncwarp();
    if (lane == 0) {
      if (rank == 0) tc::mbar_arrive(bar);
      else tc::mbar_arrive_cluster(bar, 0);
    }
    if (threadIdx.x == A_WARP0 * 32) {
      if (jtrace < 64) trace(jtrace);
      ++jtrace;
    }
  };

  if (warp == TMA_WARP) {
    // ================================ TMA producer (packed A + B ring) ================================
    if (lane == 0) {
      Cursor ld;
      ld.init(sc);
      int pre = 0;                                   // ring stages whose B half left before the wait
#ifndef FQ_PAIR_PREB
#define FQ_PAIR_PREB 1                                 // (experiment builds: 0 = no early weights)
#endif
      if (FQ_PAIR_PREB && (pdl & PDL_P)) {
        Cursor pb = ld;
        for (; pre < PSTAGES && pb.valid; ++pre, pb.next(sc)) {
          tc::mbar_expect_tx(&pfull[pre], P_BYTES);
          tc::tma_load_2d(sP + size_t(pre) * P_BYTES + AP_BYTES, &tmB, &pfull[pre], pb.kb * (BK / 2),
                          pb.nb * BN + int(rank) * BN_CTA);
        }
      }
      tc::griddep_wait();                        // qa / sa written by the previous kernel are visible
      tc::griddep_launch();                      // dependents launch only after the wait (fq_internal.h)
      for (int j = 0; ld.valid; ++j, ld.next(sc)) {
        const int sp = j % PSTAGES;
        uint8_t* dst = sP + size_t(sp) * P_BYTES;
        if (j >= pre) {
          tc::mbar_wait(&pempty[sp], ((j / PSTAGES) & 1) ^ 1);
          tc::mbar_expect_tx(&pfull[sp], P_BYTES);
          tc::tma_load_2d(dst + AP_BYTES, &tmB, &pfull[sp], ld.kb * (BK / 2), ld.nb * BN + int(rank) * BN_CTA);
        }
        tc::tma_load_2d(dst, &tmA, &pfull[sp], ld.kb * (BK / 2), ld.mb * BM + int(rank) * BM_CTA);
      }
    }
    __syncwarp();
  } else if (warp >= A_WARP0) {
    // ================================ converters ================================
    const bool is_a = warp < B_WARP0;
    int stage = 0;
    uint32_t phase = 0;
    Cursor cv;
    cv.init(sc);
    int job = 0;
    if (is_a) {
      // row r_local of the CTA's 128 activation rows, K part kpart of the 256-element K-block:
      // 128 / A_PARTS packed bytes = chunks A_CH kpart .. A_CH kpart + A_CH - 1 of the SWIZZLE_128B row
      const int aw = warp - A_WARP0;
      const int quarter = warp & 3, kpart = aw >> 2;
      const int r_local = quarter * 32 + lane;                   // == TMEM lane of this row
      const uint32_t tl = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(TMEM_A0 + kpart * (A_COLS / A_PARTS));
      // 16-byte chunk c of the row sits at c ^ swizzle: SW128 (row % 8) or SW64 ((row / 2) % 4)
      const uint32_t sw = BK == 256 ? uint32_t(r_local & 7) : uint32_t((r_local >> 1) & 3);
      const uint32_t roff = uint32_t(r_local * A_ROW);
      // Two K-blocks per iteration: both are converted and their tcgen05.st issued before one
      // tcgen05.wait::st + signal, which halves the per-K-block synchronisation latency (the
      // A path is latency-bound, not throughput-bound).
      auto prep = [&](int jb, int st, uint32_t ph) {
        const int sp = jb % PSTAGES;
        tc::mbar_wait(&empty[st], ph ^ 1);
        tc::mbar_wait(&pfull[sp], (jb / PSTAGES) & 1);
        const uint32_t src = smem_u32(sP + size_t(sp) * P_BYTES) + roff;
        uint32_t w[8 * A_CH];
#ifdef FQ_EXP_SKIP_A      // experiment build only: A conversion removed (garbage A) to bound the rest
        if (true) {
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&pempty[sp]);
          return;
        }
#endif
#pragma unroll
        for (int c = 0; c < A_CH; ++c) {
          const uint4 pk = tc::lds128(src + ((uint32_t(A_CH * kpart + c) ^ sw) << 4));
          widen8(pk.x, w[8 * c + 0], w[8 * c + 1]);
          widen8(pk.y, w[8 * c + 2], w[8 * c + 3]);
          widen8(pk.z, w[8 * c + 4], w[8 * c + 5]);
          widen8(pk.w, w[8 * c + 6], w[8 * c + 7]);
        }
        if constexpr (A_CH == 8) {
          tc::tmem_st32(tl + uint32_t(st * A_COLS), *reinterpret_cast<uint32_t(*)[32]>(w));
          tc::tmem_st32(tl + uint32_t(st * A_COLS + 32), *reinterpret_cast<uint32_t(*)[32]>(w + 32));
        } else if constexpr (A_CH == 4) {
          tc::tmem_st32(tl + uint32_t(st * A_COLS), *reinterpret_cast<uint32_t(*)[32]>(w));
        } else {
          tmem_st16(tl + uint32_t(st * A_COLS), *reinterpret_cast<uint32_t(*)[16]>(w));
        }
        // release the ring slot only after the loaded values were consumed (the tcgen05.st reads
        // them): mbarrier.arrive does not wait for an outstanding ld.shared, so an arrive right
        // after the loads lets the TMA overwrite the slot before a delayed load has read it
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&pempty[sp]);
      };
      while (cv.valid) {
        const int jt = jtrace;
        const bool trA = threadIdx.x == A_WARP0 * 32 && jt >= 16 && jt < 26;
        if (trA) trace(160 + (jt - 16) * 5 + 0);
        const int st0 = stage;
        prep(job, stage, phase);
        ++job;
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        cv.next(sc);
        const bool two = STAGES > 2 && cv.valid;         // batch two K-blocks only with spare stages
        const int st1 = stage;
        if (two) {
          prep(job, stage, phase);
          ++job;
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          cv.next(sc);
        }
        if (trA) trace(160 + (jt - 16) * 5 + 2);
        tc::tmem_st_wait();
        tc::fence_before();
        if (trA) trace(160 + (jt - 16) * 5 + 3);
        signal_full(&full[st0]);
        if (two) signal_full(&full[st1]);
        if (trA) trace(160 + (jt - 16) * 5 + 4);
      }
    } else {
      // 4 threads per weight row (16 packed bytes each) -> widened SWIZZLE_128B K-major rows
      const int ct = threadIdx.x - B_WARP0 * 32;
      while (cv.valid) {
        const int sp = job % PSTAGES;
        tc::mbar_wait(&empty[stage], phase ^ 1);
        tc::mbar_wait(&pfull[sp], (job / PSTAGES) & 1);
        const bool trB = threadIdx.x == B_WARP0 * 32 && job >= 16 && job < 26;
        if (trB) trace(210 + (job - 16) * 3 + 0);
        const uint32_t src = smem_u32(sP + size_t(sp) * P_BYTES + AP_BYTES);
        const uint32_t dst = smem_u32(smem + size_t(stage) * B_BYTES);
        uint32_t o[B_TASKS][8];
#ifdef FQ_EXP_SKIP_B      // experiment build only: B conversion removed (garbage B)
#pragma unroll
        for (int i = 0; i < B_TASKS; ++i) o[i][0] = 0;
        if (true) {
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&pempty[sp]);
          signal_full(&full[stage]);
          ++job;
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          cv.next(sc);
          continue;
        }
#endif
#pragma unroll
        for (int i = 0; i < B_TASKS; ++i) {
          const int task = ct + i * NUM_B_WARPS * 32;
          if (GE::B_TOTAL % (NUM_B_WARPS * 32) != 0 && task >= GE::B_TOTAL) break;
          const uint4 pk = tc::lds128(src + uint32_t(task * 16));      // row task/8, packed chunk task%8
          widen8(pk.x, o[i][0], o[i][1]);
          widen8(pk.y, o[i][2], o[i][3]);
          widen8(pk.z, o[i][4], o[i][5]);
          widen8(pk.w, o[i][6], o[i][7]);
        }
#pragma unroll
        for (int i = 0; i < B_TASKS; ++i) {
          const int task = ct + i * NUM_B_WARPS * 32, rl = task / B_CHUNKS, c = task % B_CHUNKS;
          if (GE::B_TOTAL % (NUM_B_WARPS * 32) != 0 && task >= GE::B_TOTAL) break;
          const uint32_t rowp = dst + uint32_t((c >> 2) * B_ATOM + rl * 128);
          const int cc = c & 3;
          tc::sts128(rowp + uint32_t(((2 * cc) ^ (rl & 7)) << 4), o[i][0], o[i][1], o[i][2], o[i][3]);
          tc::sts128(rowp + uint32_t(((2 * cc + 1) ^ (rl & 7)) << 4), o[i][4], o[i][5], o[i][6], o[i][7]);
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&pempty[sp]);               // packed B consumed (stored above)
        if (trB) trace(210 + (job - 16) * 3 + 1);
        tc::fence_proxy_async_smem();
        if (trB) trace(210 + (job - 16) * 3 + 2);
        signal_full(&full[stage]);
        ++job;
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        cv.next(sc);
      }
    }
  } else if (warp == MMA_WARP) {
    // ================================ MMA issuer (leader CTA) ================================
    if (rank == 0 && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = sc.cluster; tile < sc.num_tiles; tile += sc.num_clusters, ++it) {
        const int buf = GE::NACC == 2 ? (it & 1) : 0;
        tc::mbar_wait_cluster(&tempty[buf], ((GE::NACC == 2 ? (it >> 1) : it) & 1) ^ 1);
        tc::fence_after();
        const uint32_t tmem_d = tmem_base + uint32_t(TMEM_ACC0 + buf * BN);
        for (int kb = 0; kb < sc.num_kb; ++kb) {
          tc::mbar_wait_cluster(&full[stage], phase);
          tc::fence_after();
          if (it * sc.num_kb + kb < 64) trace(64 + it * sc.num_kb + kb);
          const uint32_t a_t = tmem_base + uint32_t(TMEM_A0 + stage * A_COLS);
          const uint32_t b0 = smem_u32(smem + size_t(stage) * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            tc::mma_ts_i8_pair(tmem_d, a_t + k * (UK / 4),
                               tc::sdesc_sw128(b0 + (k >> 2) * B_ATOM + (k & 3) * UK, 16, 1024), IDESC,
                               (kb | k) != 0);
          tc::mma_commit_pair(&empty[stage], 0x3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit_pair(&tfull[buf], 0x3);
        if (it < 8) trace(128 + it);
      }
    }
    __syncwarp();
  } else {
    // ================================ epilogue ================================
    // fp16/bf16: each warp dequantizes its 32 rows in 64-column chunks into a SWIZZLE_128B smem
    // box and TMA-stores it (coalesced; rows >= T and columns >= N are clipped by the TMA unit).
    const int r_local = warp * 32 + lane;
    const uint32_t stg = smem_u32(sEpi + warp * EPI_BYTES);
    int it = 0;
    for (int tile = sc.cluster; tile < sc.num_tiles; tile += sc.num_clusters, ++it) {
      int mb, nb;
      sc.tile(tile, mb, nb);
      const int buf = GE::NACC == 2 ? (it & 1) : 0;
      tc::mbar_wait(&tfull[buf], (GE::NACC == 2 ? (it >> 1) : it) & 1);
      tc::fence_after();
      if (threadIdx.x == 0 && it < 8) trace(136 + it);
      const int row = mb * BM + int(rank) * BM_CTA + r_local;
      const bool row_ok = row < T;
      const uint32_t tacc = tmem_base + (uint32_t(warp * 32) << 16) + uint32_t(TMEM_ACC0 + buf * BN);
      if constexpr (OUT_I32) {
#pragma unroll 1
        for (int cc = 0; cc < (BN + 31) / 32; ++cc) {
          uint32_t v[32];
          if (BN % 32 != 0 && cc == BN / 32) {                 // 16-column tail (BN = 240)
            tc::tmem_ld16(tacc + uint32_t(cc * 32), *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
          } else {
            tc::tmem_ld32(tacc + uint32_t(cc * 32), v);
          }
          tc::tmem_ld_wait();
          const int col0 = nb * BN + cc * 32;
          if (row_ok) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              const int col = col0 + j;
              if (col >= N || cc * 32 + j >= BN) break;
              int32_t* dst = static_cast<int32_t*>(yv) + size_t(row) * N + col;
              reinterpret_cast<int4*>(dst)[0] =
                  make_int4(int(v[j]) >> 8, int(v[j + 1]) >> 8, int(v[j + 2]) >> 8, int(v[j + 3]) >> 8);
              reinterpret_cast<int4*>(dst)[1] =
                  make_int4(int(v[j + 4]) >> 8, int(v[j + 5]) >> 8, int(v[j + 6]) >> 8, int(v[j + 7]) >> 8);
            }
          }
        }
      } else {
        // the TMEM holds 256 acc exactly (|256 acc| <= 2^14 K < 2^31 for K < 131072).  Symmetric:
        // float(256 acc) * (s_a / 256) is exactly float(acc) * s_a (power-of-two scaling).
        // Asymmetric: acc_true = acc - (z - 8) colsum_w is formed after the exact >> 8, in int32
        // (|acc_true| <= 120 K), so it cannot wrap for any supported K.
        // (L2 loads: this thread did not execute the PDL wait itself, see the TMA producer)
        const float s_a = row_ok ? __ldcg(sa + row) * (ASYM ? 1.0f : 1.0f / 256.0f) : 0.f;
        const int zc = (ASYM && row_ok) ? int(__ldcg(za + row)) : 0;
        // one chunk of NC (64 or 32) columns: TMEM -> dequant -> swizzled staging -> TMA store
        auto emit = [&](auto nc_tag, int c0off) {
          constexpr int NC = decltype(nc_tag)::value;
          uint32_t v[NC];
          if constexpr (NC == 16) {
            tc::tmem_ld16(tacc + uint32_t(c0off), *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
          } else {
            tc::tmem_ld32(tacc + uint32_t(c0off), *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
          }
          if constexpr (NC == 64)
            tc::tmem_ld32(tacc + uint32_t(c0off + 32), *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
          if (lane == 0) tc::bulk_wait_read0();          // previous chunk's store has left the buffer
          __syncwarp();
          tc::tmem_ld_wait();
          const int col0 = nb * BN + c0off;
#pragma unroll
          for (int c8 = 0; c8 < NC / 8; ++c8) {
            const int col = col0 + c8 * 8;
            float4 w0 = make_float4(0.f, 0.f, 0.f, 0.f), w1 = w0;
            if (col < N) {                                  // N % 8 == 0: a group is all in or all out
              w0 = __ldg(reinterpret_cast<const float4*>(sw + col));
              w1 = __ldg(reinterpret_cast<const float4*>(sw + col + 4));
            }
            uint32_t* vv = &v[c8 * 8];
            if constexpr (ASYM) {
              int4 c0 = make_int4(0, 0, 0, 0), c1 = c0;
              if (col < N) {
                c0 = __ldg(reinterpret_cast<const int4*>(colsum + col));
                c1 = __ldg(reinterpret_cast<const int4*>(colsum + col + 4));
              }
              vv[0] = uint32_t((int(vv[0]) >> 8) - zc * c0.x);
              vv[1] = uint32_t((int(vv[1]) >> 8) - zc * c0.y);
              vv[2] = uint32_t((int(vv[2]) >> 8) - zc * c0.z);
              vv[3] = uint32_t((int(vv[3]) >> 8) - zc * c0.w);
              vv[4] = uint32_t((int(vv[4]) >> 8) - zc * c1.x);
              vv[5] = uint32_t((int(vv[5]) >> 8) - zc * c1.y);
              vv[6] = uint32_t((int(vv[6]) >> 8) - zc * c1.z);
              vv[7] = uint32_t((int(vv[7]) >> 8) - zc * c1.w);
            }
            const float f0 = float(int(vv[0])) * s_a * w0.x, f1 = float(int(vv[1])) * s_a * w0.y;
            const float f2 = float(int(vv[2])) * s_a * w0.z, f3 = float(int(vv[3])) * s_a * w0.w;
            const float f4 = float(int(vv[4])) * s_a * w1.x, f5 = float(int(vv[5])) * s_a * w1.y;
            const float f6 = float(int(vv[6])) * s_a * w1.z, f7 = float(int(vv[7])) * s_a * w1.w;
            uint32_t o[4];
            if constexpr (BF16) {
              __nv_bfloat162 h0 = __floats2bfloat162_rn(f0, f1), h1 = __floats2bfloat162_rn(f2, f3);
              __nv_bfloat162 h2 = __floats2bfloat162_rn(f4, f5), h3 = __floats2bfloat162_rn(f6, f7);
              o[0] = *reinterpret_cast<uint32_t*>(&h0);
              o[1] = *reinterpret_cast<uint32_t*>(&h1);
              o[2] = *reinterpret_cast<uint32_t*>(&h2);
              o[3] = *reinterpret_cast<uint32_t*>(&h3);
            } else {
              o[0] = pack_half2(f0, f1);
              o[1] = pack_half2(f2, f3);
              o[2] = pack_half2(f4, f5);
              o[3] = pack_half2(f6, f7);
            }
            if constexpr (NC == 64)      // 32 rows x 128 B, SWIZZLE_128B: chunk ^= row % 8
              tc::sts128(stg + uint32_t(lane * 128 + ((c8 ^ (lane & 7)) << 4)), o[0], o[1], o[2], o[3]);
            else if constexpr (NC == 32) // 32 rows x 64 B, SWIZZLE_64B: chunk ^= (row / 2) % 4
              tc::sts128(stg + uint32_t(lane * 64 + ((c8 ^ ((lane >> 1) & 3)) << 4)), o[0], o[1], o[2], o[3]);
            else                         // 32 rows x 32 B, no swizzle (the 16-column tail of BN = 240)
              tc::sts128(stg + uint32_t(lane * 32 + (c8 << 4)), o[0], o[1], o[2], o[3]);
          }
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tc::tma_store_2d(NC == 64 ? &tmY : (NC == 32 ? &tmY32 : &tmY16), stg, col0,
                             mb * BM + int(rank) * BM_CTA + warp * 32);
            tc::bulk_commit();
          }
        };
#pragma unroll 1
        for (int q = 0; q < BN / 64; ++q) emit(std::integral_constant<int, 64>{}, q * 64);
        if constexpr (BN % 64 >= 32) emit(std::integral_constant<int, 32>{}, (BN / 64) * 64);
        if constexpr (BN % 32 != 0) emit(std::integral_constant<int, 16>{}, (BN / 32) * 32);
      }
      tc::fence_before();
      named_bar_sync(2, NUM_EPI_WARPS * 32);
      if (threadIdx.x == 0) {
        if (rank == 0) tc::mbar_arrive(&tempty[buf]);
        else tc::mbar_arrive_cluster(&tempty[buf], 0);
        if (it < 8) trace(144 + it);
      }
    }
    if (lane == 0) tc::bulk_wait0();
  }

  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  if (warp == MMA_WARP) {
    tc::fence_after();
    tc::tmem_dealloc2(tmem_base, TMEM_COLS);
    if (lane == 0) trace(251);
  }
}

}  // namespace g3

#ifdef FQ_TRACE
extern "C" int fq_debug_trace_gemm(unsigned long long* out) {
  return int(cudaMemcpyFromSymbol(out, g3::g_trace, sizeof(unsigned long long) * 512));
}
#endif

bool gemm_pair_supported(const GemmArgs& a) {
  return a.K % 32 == 0 && a.K < 131072 && a.N % 8 == 0 && a.T <= int64_t(1) << 30 && tmap_available();
}

// Tile width per shape: cost = waves x measured per-wave cost (scripts/gemm_shapes.py with the
// widths forced; round 2, 4 A + 4 B converter warps; 192 and 160 run 2 and 3 MMA stages, 128 and
// the single-accumulator 256 run 4).  Relative to 128: 1.19 at 160, 1.23 at 192, and
// 1.23 x (1.12 + 0.2 x 4096 / K) at 256 (its epilogue is not overlapped, which costs more at short
// K).  256 wins where it saves waves: qkv 4 -> 3, o_proj / C2 3 -> 2, down_proj 3 -> 2, 8192^3;
// 192 keeps gate/up (17 vs 13 waves, equal time).
int gemm_pair_pick_bn(int64_t T, int N, int K, int clusters) {
  using g3::BM;
  // (a 224-wide single-accumulator tile was measured too: gate/up 176 us in 14 waves vs 169 us in 17
  // waves of 192 -- not a candidate)
  const int cands[4] = {192, 160, 128, 256};
  const double rel[4] = {1.23, 1.19, 1.07, 1.23 * (1.12 + 0.2 * 4096.0 / double(K > 0 ? K : 1))};
  int best = 192;
  double best_cost = 0;
  for (int i = 0; i < 4; ++i) {
    const int bn = cands[i];
    const int64_t tiles = ((T + BM - 1) / BM) * ((N + bn - 1) / bn);
    const double cost = double((tiles + clusters - 1) / clusters) * rel[i];
    if (i == 0 || cost < best_cost - 1e-9) {
      best = bn;
      best_cost = cost;
    }
  }
  return best;
}

template <int BN>
static cudaError_t launch_bn(const GemmArgs& a) {
  using namespace g3;
  using GE = Geo<BN>;
  const bool asym = a.za != nullptr && !a.out_i32;
  auto kern = a.out_i32 ? gemm_pair_kernel<BN, true, false, false>
              : asym    ? (a.y_bf16 ? gemm_pair_kernel<BN, false, true, true> : gemm_pair_kernel<BN, false, false, true>)
                        : (a.y_bf16 ? gemm_pair_kernel<BN, false, true, false>
                                    : gemm_pair_kernel<BN, false, false, false>);
  static std::atomic<uint64_t> attr_done[5];   // per kernel variant: devices configured
  const int which = a.out_i32 ? 0 : (a.y_bf16 ? 1 : 2) + (asym ? 2 : 0);
  if (cudaError_t e = ensure_smem_attr(kern, int(GE::SMEM_BYTES), attr_done[which]); e != cudaSuccess) return e;
  CUtensorMap ma{}, mb{}, my{}, my32{}, my16{};
  {
    const uint64_t dims[2] = {uint64_t(a.K / 2), uint64_t(a.T)};
    const uint64_t strides[1] = {uint64_t(a.K / 2)};
    const uint32_t box[2] = {BK / 2, BM_CTA};
    if (!tmap_encode(&ma, a.qa, 1, 2, dims, strides, box, BK == 256 ? TMAP_SW128 : TMAP_SW64))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {uint64_t(a.K / 2), uint64_t(a.N)};
    const uint64_t strides[1] = {uint64_t(a.K / 2)};
    const uint32_t box[2] = {BK / 2, uint32_t(GE::BN_CTA)};
    if (!tmap_encode(&mb, a.qw, 1, 2, dims, strides, box, TMAP_SW_NONE)) return cudaErrorInvalidValue;
  }
  if (!a.out_i32) {
    const uint64_t dims[2] = {uint64_t(a.N), uint64_t(a.T)};
    const uint64_t strides[1] = {uint64_t(a.N) * 2};
    const uint32_t box[2] = {64, 32};
    if (!tmap_encode(&my, a.y, 2, 2, dims, strides, box, TMAP_SW128)) return cudaErrorInvalidValue;
    const uint32_t box32[2] = {32, 32};
    if (BN % 64 != 0 && !tmap_encode(&my32, a.y, 2, 2, dims, strides, box32, TMAP_SW64)) return cudaErrorInvalidValue;
    const uint32_t box16[2] = {16, 32};
    if (BN % 32 != 0 && !tmap_encode(&my16, a.y, 2, 2, dims, strides, box16, TMAP_SW_NONE)) return cudaErrorInvalidValue;
  }
  const int num_tiles = int((a.T + BM - 1) / BM) * ((a.N + BN - 1) / BN);
  const int clusters = std::max(1, std::min(num_tiles, num_sms() / 2));
  cudaError_t e = launch_pdl(kern, dim3(unsigned(2 * clusters)), dim3(THREADS), GE::SMEM_BYTES, a.stream, 2, ma, mb,
                             my, my32, my16, a.sa, int(a.T), a.K, a.sw, a.N, a.y, a.za, a.colsum, a.pdl);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t gemm_pair_launch(const GemmArgs& a, int bn) {
  static const int env_bn = [] {                    // FQ_PAIR_BN: testing aid (forces the width)
    const char* v = std::getenv("FQ_PAIR_BN");
    return v ? std::atoi(v) : 0;
  }();
  if (bn == 0) bn = env_bn;
  if (bn == 0) bn = gemm_pair_pick_bn(a.T, a.N, a.K, std::max(1, num_sms() / 2));
  switch (bn) {
    case 256: return launch_bn<256>(a);
    case 240: return launch_bn<240>(a);
    case 160: return launch_bn<160>(a);
    case 128: return launch_bn<128>(a);
    case 96: return launch_bn<96>(a);
    case 64: return launch_bn<64>(a);
    default: return launch_bn<192>(a);
  }
}

// colsum[o] = sum_k qw[o,k] over the signed nibbles of packed row o (one warp per row).
__global__ void weight_colsum_kernel(const uint8_t* __restrict__ qw, int N, int KB, int32_t* __restrict__ colsum) {
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= N) return;
  const uint8_t* p = qw + size_t(row) * KB;
  int acc = 0;
  for (int i = lane; i < KB; i += 32) {
    const int b = p[i];
    acc += ((b & 15) ^ 8) - 8 + ((b >> 4) ^ 8) - 8;     // sign-extended nibbles
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) colsum[row] = acc;
}

cudaError_t weight_colsum_launch(const uint8_t* qw, int N, int K, int32_t* colsum, cudaStream_t stream) {
  const int rows_per_block = 8;
  weight_colsum_kernel<<<(N + rows_per_block - 1) / rows_per_block, 32 * rows_per_block, 0, stream>>>(
      qw, N, K / 2, colsum);
  count_launch();
  return cudaGetLastError();
}

}  // namespace fq
