// fq_internal.h -- internal (non-ABI) declarations shared by the library's translation units.
#pragma once
#include <cstdint>
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>

namespace fq {

// TMA tensor maps (fq_tmap.cu).  dims / box innermost first; strides_bytes has rank-1 entries.
bool tmap_available();
enum TmapSwizzle { TMAP_SW_NONE = 0, TMAP_SW64 = 64, TMAP_SW128 = 128 };
bool tmap_encode(CUtensorMap* m, const void* base, int elem_bytes, int rank, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, TmapSwizzle swizzle);

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
  bool bf16;
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
  bool y_bf16;
  bool out_i32;
  cudaStream_t stream;
};

int num_sms();
void count_launch();

cudaError_t transform_quant_launch(const TQArgs& a);   // impl selection (fq_set_tq_impl)
bool tq_simt_supported(int n1, int n2);
bool tq_mma_supported(int n1, int n2);                 // legacy mma.sync kernel instantiations
cudaError_t tq_mma_launch(const TQArgs& a);
cudaError_t tq_simt_launch(const TQArgs& a);
bool tq_tc05_supported(const TQArgs& a);               // tcgen05 / TMA kernel
cudaError_t tq_tc05_launch(const TQArgs& a);
int tq_impl();

cudaError_t gemm_mma_launch(const GemmArgs& a);      // legacy mma.sync cross-check kernel
cudaError_t gemm_tc05_launch(const GemmArgs& a);     // tcgen05 kind::i8, single CTA
bool gemm_tc05_supported(const GemmArgs& a);
cudaError_t gemm_pair_launch(const GemmArgs& a);     // tcgen05 kind::i8, CTA pair (cta_group::2)
bool gemm_pair_supported(const GemmArgs& a);

}  // namespace fq
