// fq_internal.h -- internal (non-ABI) declarations shared by the library's translation units.
#pragma once
#include <cstdint>
#include <algorithm>
#include <atomic>
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>

namespace fq {

// TMA tensor maps (fq_tmap.cu).  dims / box innermost first; strides_bytes has rank-1 entries.
bool tmap_available();
enum TmapSwizzle { TMAP_SW_NONE = 0, TMAP_SW64 = 64, TMAP_SW128 = 128 };
bool tmap_encode(CUtensorMap* m, const void* base, int elem_bytes, int rank, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, TmapSwizzle swizzle);

// Programmatic dependent launch protocol of every PDL kernel in this library:
//   * a kernel signals its dependents (griddepcontrol.launch_dependents) only AFTER its own
//     griddepcontrol.wait has returned, so while a kernel runs before its wait, the only kernel
//     that can still be running is its immediate predecessor on the stream;
//   * before its wait a kernel may read parameters (PDL_P), read activations (PDL_X) and write
//     its outputs (PDL_OUT) only when the host found that the predecessor -- the last kernel
//     this library enqueued on the stream -- neither writes those inputs nor touches those
//     outputs (fq_abi.cu).  Anything else runs after the wait.
constexpr int PDL_P = 1, PDL_X = 2, PDL_OUT = 4;

struct TQArgs {
  const void* x;
  int64_t T, ldx;
  int n1, n2;
  const void* p1;
  const void* p2;
  float alpha;
  uint8_t* q;
  float* scale;
  float* y;         // optional fp32 export of the transformed activations (debug / parity)
  int8_t* zero;     // FQ_ASYM: per-token zero point - 8 (output); nullptr for FQ_SYM
  bool bf16;
  int pdl;            // PDL_* flags (fq_abi.cu hazard check): what may happen before griddepcontrol.wait
  cudaStream_t stream;
};

struct GemmArgs {
  const uint8_t* qa;
  const float* sa;
  int64_t T;
  int K;
  const uint8_t* qw;
  const float* sw;
  int N;
  void* y;          // fp16/bf16 output, or int32 accumulators when out_i32
  const int8_t* za;         // asymmetric activations: z - 8 per token (nullptr: symmetric)
  const int32_t* colsum;    // asymmetric activations: sum_k qw[o,k] per output channel
  bool y_bf16;
  bool out_i32;
  int pdl;            // PDL_* flags (fq_abi.cu hazard check)
  cudaStream_t stream;
};

struct KVArgs {     // KV-cache quantization (fq_kv_quant)
  const void* x;    // [R, D] head vectors, row stride ldx elements
  int64_t R, ldx;
  int D;
  const void* p;    // P_h [D, D] row-major, same dtype as x
  float alpha;
  uint8_t* q;       // [R, D/2]
  float* scale;     // [R]
  int8_t* zero;     // [R] z - 8
  bool bf16;
  int pdl;          // PDL_* flags (the KV kernel waits before any access regardless)
  cudaStream_t stream;
};

int num_sms();
void count_launch();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies per device context: set it once per
// device for one kernel; `done` (a static at the launch site, one per kernel variant) holds a bit
// per device id < 64 already configured (larger ids are configured on every launch).
template <typename K>
cudaError_t ensure_smem_attr(K kern, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? uint64_t(1) << dev : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_release);
  return e;
}
bool pdl_enabled();      // FQ_PDL=0 in the environment disables programmatic dependent launch

// Launch with programmatic stream serialization (PDL: the kernel may start while the previous
// kernel of the stream finishes; it calls griddepcontrol.wait before touching global inputs) and
// an optional cluster size.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_policy(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              int cluster_x, int cluster_policy, Args&&... args);

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       int cluster_x, Args&&... args) {
  return launch_pdl_policy(kern, grid, block, smem, stream, cluster_x, 0, std::forward<Args>(args)...);
}

// cluster_policy: 0 default, 1 spread, 2 load balancing (cudaClusterSchedulingPolicy)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_policy(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              int cluster_x, int cluster_policy, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[3];
  int na = 0;
  if (cluster_x > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = unsigned(cluster_x);
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (cluster_policy > 0) {
      attr[na].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
      attr[na].val.clusterSchedulingPolicyPreference =
          cluster_policy == 1 ? cudaClusterSchedulingPolicySpread : cudaClusterSchedulingPolicyLoadBalancing;
      ++na;
    }
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = unsigned(na);
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

cudaError_t transform_quant_launch(const TQArgs& a);   // impl selection (fq_set_tq_impl)
bool tq_kernel_available(const TQArgs& a);             // some kernel serves this call
bool tq_is_pdl(const TQArgs& a);                       // the kernel it picks uses PDL (tcgen05 kernels)
bool tq_simt_supported(int n1, int n2);
bool tq_mma_supported(int n1, int n2);                 // legacy mma.sync kernel instantiations
cudaError_t tq_mma_launch(const TQArgs& a);
bool tq_ident2_supported(int n1, int n2);             // P2 = I (p2 == nullptr), mma.sync kernel
cudaError_t tq_ident2_launch(const TQArgs& a);
cudaError_t tq_simt_launch(const TQArgs& a);
bool tq_tc05_supported(const TQArgs& a);               // tcgen05 / TMA kernel
bool tq_asym_supported(const TQArgs& a);               // FQ_ASYM available for this shape
cudaError_t tq_tc05_launch(const TQArgs& a);
bool tq_wide_supported(const TQArgs& a);               // tcgen05, n1 = 128, n2 in {160, 192, 224, 256}
cudaError_t tq_wide_launch(const TQArgs& a);
int tq_impl();

cudaError_t weight_colsum_launch(const uint8_t* qw, int N, int K, int32_t* colsum, cudaStream_t stream);
cudaError_t gemm_mma_launch(const GemmArgs& a);      // legacy mma.sync cross-check kernel
cudaError_t gemm_tc05_launch(const GemmArgs& a);     // tcgen05 kind::i8, single CTA
bool gemm_tc05_supported(const GemmArgs& a);
cudaError_t gemm_pair_launch(const GemmArgs& a, int bn = 0);   // tcgen05 kind::i8, CTA pair (cta_group::2);
                                                          // bn: tile width 192/160/128, 0 = per shape
int gemm_pair_pick_bn(int64_t T, int N, int K, int clusters);
cudaError_t gemm_dec_launch(const GemmArgs& a, int split = 0);  // decode (T <= 64): swapped operands,
bool gemm_dec_supported(const GemmArgs& a);                     // cluster split-K; split 0 = per shape
bool gemm_pair_supported(const GemmArgs& a);
// fused decode linear (T <= 64, (n1, n2) = (64, 64) or (112, 128), fp16 or bf16 x, P2 given, symmetric): the transform +
// quantize of x (into the codes/scales buffers named by the GemmArgs) runs inside the decode GEMM
// launch (fq_gemm_dec.cu, FUSED); cudaErrorNotSupported (nothing launched) when the grid for the
// shape has fewer CTAs than two-token tiles
struct FdArgs {
  const void* x;
  int64_t ldx;
  int n1, n2;                // (64, 64) or (112, 128)
  const void* p1;
  const void* p2;
  float alpha;
  bool bf16;                 // x, p1, p2 bf16 (else fp16)
};
bool fused_dec_supported(const GemmArgs& a, int n1, int n2, bool x_bf16, const void* p2);
cudaError_t fused_dec_launch(const GemmArgs& a, const FdArgs& f);
size_t weight_prep_workspace(int n1, int n2);
cudaError_t inverse_t_launch(const void* p, int n, bool bf16, void* aug, void* out, int* status,
                             cudaStream_t stream);
bool kv_quant_supported(const KVArgs& a);            // tcgen05 KV-cache kernel
cudaError_t kv_quant_launch(const KVArgs& a);

}  // namespace fq
