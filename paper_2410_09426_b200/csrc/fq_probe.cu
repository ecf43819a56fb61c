// fq_probe.cu -- tensor-core issue-rate microbenchmark (instrumented build only, -DFQ_TRACE):
// one elected thread issues a long chain of tcgen05.mma.kind::i8 on garbage operands (TMEM A or
// shared-memory A, CTA pair or single CTA, several N) and the kernel reports cycles per MMA.
// Used to pin the MMA pacing of the W4A4 GEMM design (scripts/probe_mma.py).  Not part of the
// product library.
#ifdef FQ_TRACE
#include <cstdint>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"
#include "fq_tc05.cuh"

namespace fq {
namespace probe {

__device__ unsigned long long g_probe[4];

template <bool PAIR, bool TS, int N>
__global__ void __launch_bounds__(128, 1) mma_probe_kernel(int iters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) {
    if (PAIR) tc::tmem_alloc2(&slot, 512);
    else tc::tmem_alloc(&slot, 512);
  }
  tc::fence_before();
  __syncthreads();
  if (PAIR) tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem = slot;
  constexpr int M = PAIR ? 256 : 128;
  constexpr uint32_t IDESC = tc::idesc_i8(M, N);
  if (threadIdx.x == 0 && rank == 0) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0)::"memory");
    const uint32_t b0 = smem_u32(smem);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t bd = tc::sdesc_sw128(b0 + k * 32, 16, 1024);
        if constexpr (TS) {
          if constexpr (PAIR) tc::mma_ts_i8_pair(tmem, tmem + 384 + k * 8, bd, IDESC, 1);
          else tc::mma_ts<true>(tmem, tmem + 384 + k * 8, bd, IDESC, 1);
        } else {
          const uint64_t ad = tc::sdesc_sw128(b0 + 65536 + k * 32, 16, 1024);
          if constexpr (PAIR) {
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(IDESC), "r"(1));
          } else {
            tc::mma_ss<true>(tmem, ad, bd, IDESC, 1);
          }
        }
      }
    }
    if constexpr (PAIR) tc::mma_commit_pair(&bar, 0x3);
    else tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)::"memory");
    if (blockIdx.x == 0) {
      g_probe[0] = t1 - t0;
      g_probe[1] = uint64_t(iters) * 4;
    }
  } else if (PAIR && rank == 1 && threadIdx.x == 0) {
    tc::mbar_wait(&bar, 0);
  }
  tc::fence_before();
  __syncthreads();
  if (PAIR) tc::cluster_sync();
  if (warp == 0) {
    tc::fence_after();
    if (PAIR) tc::tmem_dealloc2(tmem, 512);
    else tc::tmem_dealloc(tmem, 512);
  }
}

template <bool PAIR, bool TS, int N>
static int launch(int iters, int ctas) {
  auto kern = mma_probe_kernel<PAIR, TS, N>;
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(ctas));
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, iters);
  return int(cudaDeviceSynchronize());
}

}  // namespace probe
}  // namespace fq

// variant: bit0 = pair, bit1 = TS (A in TMEM); n in {128, 192, 256}.  out[0] = ns, out[1] = #MMAs
extern "C" int fq_debug_mma_probe(int variant, int n, int iters, int ctas, unsigned long long* out) {
  using namespace fq::probe;
  const bool pair = variant & 1, ts = variant & 2;
  int e = -1;
#define FQ_PROBE_CASE(P, S, NN) \
  if (pair == P && ts == S && n == NN) e = launch<P, S, NN>(iters, ctas);
  FQ_PROBE_CASE(true, true, 128) FQ_PROBE_CASE(true, true, 192) FQ_PROBE_CASE(true, true, 256)
  FQ_PROBE_CASE(true, false, 128) FQ_PROBE_CASE(true, false, 192) FQ_PROBE_CASE(true, false, 256)
  FQ_PROBE_CASE(false, true, 128) FQ_PROBE_CASE(false, true, 192) FQ_PROBE_CASE(false, true, 256)
  FQ_PROBE_CASE(false, false, 128) FQ_PROBE_CASE(false, false, 192) FQ_PROBE_CASE(false, false, 256)
#undef FQ_PROBE_CASE
  if (e != 0) return e;
  return int(cudaMemcpyFromSymbol(out, g_probe, sizeof(unsigned long long) * 2));
}
#endif  // FQ_TRACE
