// probe: does a tcgen05.alloc in the kernel limit residency to one CTA per SM?
// (the occupancy calculator says 1 for any kernel containing tcgen05.alloc; this measures what
// the hardware does: every CTA records its SM and [start, end) on the global timer)
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__global__ void __launch_bounds__(512, 2) k_plain(unsigned long long* rec, int spin_ns) {
  const unsigned long long t0 = gtime();
  while (gtime() - t0 < (unsigned long long)spin_ns) {}
  if (threadIdx.x == 0) { rec[3 * blockIdx.x] = smid(); rec[3 * blockIdx.x + 1] = t0; rec[3 * blockIdx.x + 2] = gtime(); }
}
template <int COLS>
__global__ void __launch_bounds__(512, 2) k_tmem(unsigned long long* rec, int spin_ns) {
  __shared__ unsigned slot;
  const unsigned long long t0 = gtime();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        (unsigned)__cvta_generic_to_shared(&slot)), "n"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  while (gtime() - t0 < (unsigned long long)spin_ns) {}
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "n"(COLS));
  if (threadIdx.x == 0) { rec[3 * blockIdx.x] = smid(); rec[3 * blockIdx.x + 1] = t0; rec[3 * blockIdx.x + 2] = gtime(); }
}
static int max_conc(const std::vector<unsigned long long>& h, int n) {
  int best = 0;
  for (int i = 0; i < n; ++i) {
    int c = 0;
    for (int j = 0; j < n; ++j)
      if (h[3 * j] == h[3 * i] && h[3 * j + 1] <= h[3 * i + 1] && h[3 * j + 2] > h[3 * i + 1]) ++c;
    best = std::max(best, c);
  }
  return best;
}
template <typename K>
static void run(const char* name, K k, int grid) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * 3 * grid);
  k<<<grid, 512>>>(d, 50000);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<grid, 512>>>(d, 50000);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  std::vector<unsigned long long> h(3 * grid);
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  int o = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, 512, 0);
  printf("%-10s grid %d: %.1f us (50 us spin per CTA), max CTAs concurrently on one SM %d, occupancy API %d, %s\n",
         name, grid, ms * 1e3, max_conc(h, grid), o, cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run("plain", k_plain, 2 * sms);
  run("tmem64", k_tmem<64>, 2 * sms);
  run("tmem256", k_tmem<256>, 2 * sms);
  run("tmem64x4", k_tmem<64>, 4 * sms);
  return 0;
}
