// fq_probe_cp.cu -- semantics probe for the hardware INT4 -> 8-bit decompression path
// (instrumented build only, -DFQ_TRACE; scripts/probe_cp.py):
//   TMA with CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B (packed 4-bit global -> 16 elements per
//   16-byte smem unit) and tcgen05.cp ... .b8x16.b4x16_p64 (padded 4-bit smem -> 8-bit TMEM).
// Dumps the shared-memory image and the TMEM image so the host can read off where each nibble
// lands.  Not part of the product library.
#ifdef FQ_TRACE
#include <cuda.h>
#include <cstdint>
#include <cuda_runtime.h>
#include "fq_device.cuh"
#include "fq_internal.h"
#include "fq_tc05.cuh"

namespace fq {
namespace probe_cp {

constexpr int ROWS = 128, KEL = 256;          // 128 rows x 256 4-bit elements (128 packed bytes)
constexpr int SM_BYTES = ROWS * KEL;          // padded image: one byte per element = 32 KB

template <bool PAIR>
__global__ void __launch_bounds__(128, 1)
cp_probe_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* __restrict__ packed, int mode,
                uint8_t* __restrict__ smem_dump, uint32_t* __restrict__ tmem_dump) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_tma, bar_cp;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0;
  const uint8_t* src = packed + size_t(rank) * ROWS * (KEL / 2);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar_tma, 1);
    tc::mbar_init(&bar_cp, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) {
    if (PAIR) tc::tmem_alloc2(&slot, 128);
    else tc::tmem_alloc(&slot, 128);
  }
  // clear the image (so padding bytes written by nobody read as 0xEE)
  for (int i = threadIdx.x; i < SM_BYTES / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0xEEEEEEEEu;
  tc::fence_before();
  __syncthreads();
  if (PAIR) tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem = slot;
  if ((mode & 3) == 1) {
    // TMA, 16U4_ALIGN16B, SWIZZLE_128B, two boxes of {128 elements, 128 rows} (16 KB each)
    if (threadIdx.x == 0) {
      tc::mbar_expect_tx(&bar_tma, (mode & 8) ? SM_BYTES / 2 : SM_BYTES);
      tc::tma_load_2d(smem, &tm, &bar_tma, 0, int(rank) * ROWS);
      tc::tma_load_2d(smem + SM_BYTES / 2, &tm, &bar_tma, 128, int(rank) * ROWS);
    }
    // bounded wait: report instead of hanging if the transaction count never completes
    uint32_t done = 0;
    for (int it = 0; it < (1 << 22) && !done; ++it)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bar_tma)) : "memory");
    if (!done) {
      if (threadIdx.x == 0) tmem_dump[0] = 0xDEADBEEFu;
      asm volatile("trap;");
    }
  } else {
    // manual SW128 K-major image: row r, group g (16 elements = 8 packed bytes): 16-byte unit at
    // half (g / 8) * 16 KB + r * 128 + ((g % 8) ^ (r % 8)) * 16; packed bytes in the first 8
    // (mode 0) or the last 8 (mode 2) bytes of the unit, the other 8 bytes zero
    const int r = threadIdx.x;
    for (int g = 0; g < KEL / 16; ++g) {
      uint32_t w0 = *reinterpret_cast<const uint32_t*>(src + r * (KEL / 2) + g * 8);
      uint32_t w1 = *reinterpret_cast<const uint32_t*>(src + r * (KEL / 2) + g * 8 + 4);
      uint8_t* u = smem + (g / 8) * (SM_BYTES / 2) + r * 128 + (((g % 8) ^ (r % 8)) * 16);
      uint32_t* u32 = reinterpret_cast<uint32_t*>(u);
      if ((mode & 3) == 0) { u32[0] = w0; u32[1] = w1; u32[2] = 0; u32[3] = 0; }
      else { u32[0] = 0; u32[1] = 0; u32[2] = w0; u32[3] = w1; }
    }
    tc::fence_proxy_async_smem();
  }
  __syncthreads();
  if (PAIR) tc::cluster_sync();
  // dump the smem image
  uint8_t* sd = smem_dump + size_t(rank) * SM_BYTES;
  for (int i = threadIdx.x; i < SM_BYTES / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sd)[i] = reinterpret_cast<const uint4*>(smem)[i];
  // decompress: 16 copies of 128 rows x 128 bits (16 elements) -> TMEM columns 4g .. 4g+3
  if (threadIdx.x == 0 && rank == 0) {
    for (int g = 0; g < KEL / 16; ++g) {
      const uint32_t a = smem_u32(smem + (g / 8) * (SM_BYTES / 2) + (g % 8) * 16);
      const uint64_t d = tc::sdesc_sw128(a, 16, 1024);
      if constexpr (PAIR)
        asm volatile("tcgen05.cp.cta_group::2.128x128b.b8x16.b4x16_p64 [%0], %1;\n" ::"r"(tmem + uint32_t(4 * g)),
                     "l"(d) : "memory");
      else
        asm volatile("tcgen05.cp.cta_group::1.128x128b.b8x16.b4x16_p64 [%0], %1;\n" ::"r"(tmem + uint32_t(4 * g)),
                     "l"(d) : "memory");
    }
    if constexpr (PAIR) tc::mma_commit_pair(&bar_cp, 0x3);
    else tc::mma_commit(&bar_cp);
  }
  tc::mbar_wait(&bar_cp, 0);
  tc::fence_after();
  uint32_t v[32];
  uint32_t* td = tmem_dump + size_t(rank) * ROWS * 64;
  for (int h = 0; h < 2; ++h) {
    tc::tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + uint32_t(h * 32), v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) td[(warp * 32 + lane) * 64 + h * 32 + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (PAIR) tc::cluster_sync();
  if (warp == 0) {
    tc::fence_after();
    if (PAIR) tc::tmem_dealloc2(tmem, 128);
    else tc::tmem_dealloc(tmem, 128);
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace probe_cp
}  // namespace fq

// packed: [2 * 128, 128] bytes (device).  mode bit0-1: 0 manual (data first 8 B), 1 TMA
// 16U4_ALIGN16B, 2 manual (data last 8 B); bit2: CTA pair; bit3: TMA expect_tx = packed bytes.  smem_dump [2 * 32768] bytes,
// tmem_dump [2 * 128 * 64] u32.  Returns 0 on success, else a CUDA / driver error code.
extern "C" int fq_debug_cp_probe(const uint8_t* packed, int mode, uint8_t* smem_dump, uint32_t* tmem_dump) {
  using namespace fq::probe_cp;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult qr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess || !p) return -1;
  EncodeTiled enc = reinterpret_cast<EncodeTiled>(p);
  CUtensorMap tm{};
  const cuuint64_t dims[2] = {cuuint64_t(KEL), cuuint64_t(2 * ROWS)};
  const cuuint64_t strides[1] = {cuuint64_t(KEL / 2)};
  const cuuint32_t box[2] = {128, ROWS};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 2, const_cast<uint8_t*>(packed), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return 1000 + int(r);
  const bool pair = mode & 4;
  const int smem = SM_BYTES + 1024;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pair ? 2 : 1);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (pair) {
    cudaFuncSetAttribute(cp_probe_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    e = cudaLaunchKernelEx(&cfg, cp_probe_kernel<true>, tm, packed, mode & 11, smem_dump, tmem_dump);
  } else {
    cudaFuncSetAttribute(cp_probe_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    e = cudaLaunchKernelEx(&cfg, cp_probe_kernel<false>, tm, packed, mode & 11, smem_dump, tmem_dump);
  }
  if (e != cudaSuccess) return int(e);
  return int(cudaDeviceSynchronize());
}
#endif  // FQ_TRACE
