// fq_abi.cu -- the extern "C" boundary declared in include/flatquant.h: argument validation,
// kernel selection and launch.  No computation happens here; every step runs in the kernels.
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>
#include <cuda_runtime.h>
#include "../../include/flatquant.h"
#include "fq_internal.h"

namespace fq {

static std::atomic<uint64_t> g_launches{0};
static std::atomic<int> g_last_cuda_error{0};
static std::atomic<int> g_gemm_impl{0};
static std::atomic<int> g_tq_impl{0};

int tq_impl() { return g_tq_impl.load(); }

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FQ_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 1;
  }
  return cached[dev];
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- programmatic dependent launch: host-side hazard check ------------------------------------
// Protocol (fq_internal.h): every PDL kernel of this library signals its dependents only after its
// own griddepcontrol.wait has returned, so a kernel running BEFORE its wait can overlap only its
// immediate predecessor on the stream.  Whatever else was enqueued earlier has completed by then;
// so has any work of other origin in between (copies, kernels that do not trigger PDL early),
// which a PDL kernel can never overlap.  The host therefore records, per stream, the buffers the
// last kernel this library enqueued reads and writes, and lets the next kernel
//   read its parameters early  (PDL_P)   if no parameter overlaps the predecessor's outputs,
//   read its activations early (PDL_X)   if no activation overlaps the predecessor's outputs,
//   write its outputs early    (PDL_OUT) if no output overlaps the predecessor's inputs or outputs.
// Weights and P stream in while the previous kernel finishes, and a kernel whose data is disjoint
// from its predecessor's (e.g. the next linear's transform after a GEMM) runs concurrently with it.
struct Span {
  uintptr_t lo, hi;
};
static Span span(const void* p, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  return Span{a, p ? a + bytes : a};
}
using Spans = std::initializer_list<Span>;
struct LaunchRec {
  std::vector<Span> in, out;
};
static std::mutex g_pdl_mu;
static std::unordered_map<void*, LaunchRec> g_pdl_rec;   // stream -> last PDL kernel's buffers

static bool overlap(Spans a, const std::vector<Span>& b) {
  for (const Span& x : a)
    for (const Span& y : b)
      if (x.lo < x.hi && y.lo < y.hi && x.lo < y.hi && y.lo < x.hi) return true;
  return false;
}
static int pdl_flags(cudaStream_t st, Spans params, Spans acts, Spans outs) {
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  auto it = g_pdl_rec.find(static_cast<void*>(st));
  if (it == g_pdl_rec.end()) return PDL_P | PDL_X | PDL_OUT;
  const LaunchRec& r = it->second;
  int f = 0;
  if (!overlap(params, r.out)) f |= PDL_P;
  if (!overlap(acts, r.out)) f |= PDL_X;
  if (!overlap(outs, r.out) && !overlap(outs, r.in)) f |= PDL_OUT;
  return f;
}
// after a launch: a PDL kernel becomes the stream's overlappable predecessor; after anything else
// (a kernel without early trigger, a copy) the next kernel cannot start before it completes
static void record_launch(cudaStream_t st, bool pdl_kernel, Spans ins, Spans outs) {
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  if (!pdl_kernel) {
    g_pdl_rec.erase(static_cast<void*>(st));
    return;
  }
  LaunchRec& r = g_pdl_rec[static_cast<void*>(st)];
  r.in.assign(ins.begin(), ins.end());
  r.out.assign(outs.begin(), outs.end());
}
static void clear_outputs(cudaStream_t st) { record_launch(st, false, {}, {}); }

static fq_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return FQ_OK;
  g_last_cuda_error.store(int(e));
  return FQ_ECUDA;
}

static fq_status validate_tq(const void* x, int32_t x_dtype, int64_t T, int64_t ldx, int32_t n1, int32_t n2,
                             const void* p1, const void* p2, float alpha, const uint8_t* q,
                             const float* scale) {
  if (x_dtype != FQ_F16 && x_dtype != FQ_BF16) return FQ_EINVAL;
  if (T < 0 || n1 < 1 || n2 < 1) return FQ_EINVAL;
  if (!(alpha > 0.0f && alpha <= 1.0f)) return FQ_EINVAL;   // also rejects NaN
  if (T == 0) return FQ_OK;
  if (!x || !p1 || !q || !scale) return FQ_EINVAL;        // p2 == NULL: P2 = I (fq_transform_quant)
  if (!p2 && !tq_ident2_supported(n1, n2)) return FQ_ENOTSUP;   // P2 = I: (32, 128), (64, 128)
  const int64_t n = int64_t(n1) * n2;
  if (n % 2 != 0) return FQ_ESHAPE;
  if (ldx < n) return FQ_ESHAPE;
  const bool tc = (n1 % 16 == 0) && (n2 % 16 == 0);
  if (tc) {
    // tensor-core kernel: 16-byte cp.async of x rows and 16-byte stores of packed rows
    if ((ldx * 2) % 16 != 0 || !aligned16(x) || !aligned16(q)) return FQ_ESHAPE;
  }
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(p1) | reinterpret_cast<uintptr_t>(p2)) & 1u)
    return FQ_ESHAPE;
  if ((reinterpret_cast<uintptr_t>(scale) & 3u) != 0) return FQ_ESHAPE;
  if (n1 > 256 || n2 > 256) return FQ_ENOTSUP;
  return FQ_OK;
}

static fq_status run_tq(const void* x, int32_t x_dtype, int64_t T, int64_t ldx, int32_t n1, int32_t n2,
                        const void* p1, const void* p2, float alpha, uint8_t* q, float* scale, float* y,
                        int8_t* zero, void* stream) {
  TQArgs a{};
  a.x = x;
  a.T = T;
  a.ldx = ldx;
  a.n1 = n1;
  a.n2 = n2;
  a.p1 = p1;
  a.p2 = p2;
  a.alpha = alpha;
  a.q = q;
  a.scale = scale;
  a.y = y;
  a.zero = zero;
  a.bf16 = (x_dtype == FQ_BF16);
  a.stream = static_cast<cudaStream_t>(stream);
  if (!tq_kernel_available(a)) return FQ_ENOTSUP;
  if (zero && !tq_asym_supported(a)) return FQ_ENOTSUP;
  const int64_t n = int64_t(n1) * n2;
  const Span sp1 = span(p1, size_t(n1) * n1 * 2), sp2 = span(p2, size_t(n2) * n2 * 2);
  const Span sx = span(x, size_t(T - 1) * size_t(ldx) * 2 + size_t(n) * 2);
  const Span sq = span(q, size_t(T) * size_t(n / 2)), ss = span(scale, size_t(T) * 4), sz = span(zero, size_t(T)),
             sy = span(y, y ? size_t(T) * size_t(n) * 4 : 0);
  a.pdl = pdl_flags(a.stream, {sp1, sp2}, {sx}, {sq, ss, sz, sy});
  const fq_status s = cuda_status(transform_quant_launch(a));
  if (s == FQ_OK) record_launch(a.stream, tq_is_pdl(a), {sp1, sp2, sx}, {sq, ss, sz, sy});
  return s;
}

static fq_status validate_gemm(const uint8_t* qa, int64_t T, int32_t K, const uint8_t* qw, int32_t N,
                               const void* y) {
  if (T < 0 || K < 0 || N < 0) return FQ_EINVAL;
  if (T == 0 || N == 0) return FQ_OK;
  if (!qa || !qw || !y) return FQ_EINVAL;
  if (K == 0 || K % 32 != 0 || N % 8 != 0) return FQ_ESHAPE;
  if (!aligned16(qa) || !aligned16(qw) || !aligned16(y)) return FQ_ESHAPE;
  if (K >= 131072) return FQ_ENOTSUP;   // 256 |acc| <= 2^14 K must stay < 2^31 (widened x16 operands)
  if (T > (int64_t(1) << 30)) return FQ_ENOTSUP;
  return FQ_OK;
}

static fq_status launch_gemm(GemmArgs& a, bool& pdl_kernel);

static fq_status run_gemm(const uint8_t* qa, const float* sa, int64_t T, int32_t K, const uint8_t* qw,
                          const float* sw, int32_t N, void* y, bool y_bf16, bool out_i32, void* stream,
                          const int8_t* za = nullptr, const int32_t* colsum = nullptr) {
  GemmArgs a{};
  a.qa = qa;
  a.sa = sa;
  a.T = T;
  a.K = K;
  a.qw = qw;
  a.sw = sw;
  a.N = N;
  a.y = y;
  a.y_bf16 = y_bf16;
  a.out_i32 = out_i32;
  a.za = za;
  a.colsum = colsum;
  a.stream = static_cast<cudaStream_t>(stream);
  const Span sqw = span(qw, size_t(N) * size_t(K / 2)), ssw = span(sw, sw ? size_t(N) * 4 : 0),
             scs = span(colsum, colsum ? size_t(N) * 4 : 0);
  const Span sqa = span(qa, size_t(T) * size_t(K / 2)), ssa = span(sa, sa ? size_t(T) * 4 : 0),
             sza = span(za, za ? size_t(T) : 0);
  const Span sy = span(y, size_t(T) * size_t(N) * (out_i32 ? 4 : 2));
  a.pdl = pdl_flags(a.stream, {sqw, ssw, scs}, {sqa, ssa, sza}, {sy});
  bool pdl_kernel = false;
  const fq_status s = launch_gemm(a, pdl_kernel);
  if (s == FQ_OK) record_launch(a.stream, pdl_kernel, {sqw, ssw, scs, sqa, ssa, sza}, {sy});
  return s;
}

static fq_status launch_gemm(GemmArgs& a, bool& pdl_kernel) {
  const int impl = g_gemm_impl.load();
  const bool za = a.za != nullptr;
  pdl_kernel = true;                               // decode and pair kernels use PDL
  // impl 0: decode kernel for T <= 64, else the pair kernel with the tile width picked per shape;
  // 3 / 4 / 5: pair kernel with the width forced to 192 / 160 / 128; 6: decode kernel forced
  if (impl == 6 || (impl == 0 && gemm_dec_supported(a))) {
    if (!gemm_dec_supported(a)) return FQ_ENOTSUP;
    return cuda_status(gemm_dec_launch(a));
  }
  const bool pair = impl == 0 || (impl >= 3 && impl <= 5) || impl == 7;
  const int bn = impl == 3 ? 192 : impl == 4 ? 160 : impl == 5 ? 128 : impl == 7 ? 256 : 0;
  if (za) {                                        // asymmetric activations: pair or decode kernel
    if (!pair || !gemm_pair_supported(a)) return FQ_ENOTSUP;
    return cuda_status(gemm_pair_launch(a, bn));
  }
  if (pair && gemm_pair_supported(a)) return cuda_status(gemm_pair_launch(a, bn));
  if (impl >= 3) return FQ_ENOTSUP;   // a forced pair width the shape does not support
  pdl_kernel = false;                              // cross-check kernels: plain launches
  if (impl == 2 && gemm_tc05_supported(a)) return cuda_status(gemm_tc05_launch(a));
  return cuda_status(gemm_mma_launch(a));
}

}  // namespace fq

using namespace fq;

extern "C" {

fq_status fq_transform_quant(const void* x, int32_t x_dtype, int64_t T, int64_t ldx, int32_t n1, int32_t n2,
                             const void* p1, const void* p2, float alpha, int32_t qmode, uint8_t* q,
                             float* scale, int8_t* zero, void* stream) {
  if (qmode != FQ_SYM && qmode != FQ_ASYM) return FQ_EINVAL;
  if ((qmode == FQ_SYM) != (zero == nullptr)) return FQ_EINVAL;   // zero iff asymmetric

  fq_status s = validate_tq(x, x_dtype, T, ldx, n1, n2, p1, p2, alpha, q, scale);
  if (s != FQ_OK || T == 0) return s;
  return run_tq(x, x_dtype, T, ldx, n1, n2, p1, p2, alpha, q, scale, nullptr, zero, stream);
}

fq_status fq_transform_f32(const void* x, int32_t x_dtype, int64_t T, int64_t ldx, int32_t n1, int32_t n2,
                           const void* p1, const void* p2, float alpha, uint8_t* q, float* scale, float* y,
                           void* stream) {
  fq_status s = validate_tq(x, x_dtype, T, ldx, n1, n2, p1, p2, alpha, q, scale);
  if (s != FQ_OK || T == 0) return s;
  if (!y) return FQ_EINVAL;
  if ((reinterpret_cast<uintptr_t>(y) & 7u) != 0) return FQ_ESHAPE;
  return run_tq(x, x_dtype, T, ldx, n1, n2, p1, p2, alpha, q, scale, y, nullptr, stream);
}

fq_status fq_w4a4_linear(const uint8_t* qa, const float* sa, const int8_t* za, int64_t T, int32_t K,
                         const uint8_t* qw, const float* sw, const int32_t* colsum_w, int32_t N, void* y,
                         int32_t y_dtype, void* stream) {
  if (y_dtype != FQ_F16 && y_dtype != FQ_BF16) return FQ_EINVAL;
  if ((za == nullptr) != (colsum_w == nullptr)) return FQ_EINVAL;   // both or neither
  fq_status s = validate_gemm(qa, T, K, qw, N, y);
  if (s != FQ_OK || T == 0 || N == 0) return s;
  if (!sa || !sw) return FQ_EINVAL;
  if (!aligned16(sw) || (colsum_w && !aligned16(colsum_w))) return FQ_ESHAPE;
  return run_gemm(qa, sa, T, K, qw, sw, N, y, y_dtype == FQ_BF16, false, stream, za, colsum_w);
}

fq_status fq_w4a4_gemm_i32(const uint8_t* qa, int64_t T, int32_t K, const uint8_t* qw, int32_t N,
                           int32_t* acc, void* stream) {
  fq_status s = validate_gemm(qa, T, K, qw, N, acc);
  if (s != FQ_OK || T == 0 || N == 0) return s;
  return run_gemm(qa, nullptr, T, K, qw, nullptr, N, acc, false, true, stream);
}

}  // extern "C"

namespace fq {
// every check fq_flatquant_linear makes, before anything is enqueued (also for the host-buffer
// entry points, which must not start a copy for a call that is then rejected)
static fq_status validate_linear(const void* x, int32_t x_dtype, int64_t T, int32_t n1, int32_t n2,
                                 const void* p1, const void* p2, float alpha, const uint8_t* qw,
                                 const float* sw, int32_t N, const void* y, int32_t y_dtype,
                                 const uint8_t* q_ws, const float* s_ws) {
  if (T < 0 || n1 < 1 || n2 < 1 || N < 0) return FQ_EINVAL;
  const int64_t n = int64_t(n1) * n2;
  if (n > INT32_MAX) return FQ_ESHAPE;
  if (y_dtype != FQ_F16 && y_dtype != FQ_BF16) return FQ_EINVAL;
  fq_status s = validate_tq(x, x_dtype, T, n, n1, n2, p1, p2, alpha, q_ws, s_ws);
  if (s != FQ_OK || T == 0) return s;
  s = validate_gemm(q_ws, T, int32_t(n), qw, N, y);
  if (s != FQ_OK || N == 0) return s;
  if (!sw) return FQ_EINVAL;
  if (!aligned16(sw)) return FQ_ESHAPE;
  return FQ_OK;
}

bool fused_enabled() {                             // FQ_FUSED=0: testing aid (two kernels always)
  static const bool on = [] {
    const char* e = std::getenv("FQ_FUSED");
    return !(e && e[0] == '0');
  }();
  return on;
}

// one launch for the whole linear (transform + quantize + GEMM + dequant) where a fused kernel
// exists: FQ_ENOTSUP (nothing enqueued) otherwise
static fq_status run_fused(const void* x, int32_t x_dtype, int64_t T, int32_t n1, int32_t n2, const void* p1,
                           const void* p2, float alpha, const uint8_t* qw, const float* sw, int32_t N, void* y,
                           bool y_bf16, uint8_t* q_ws, float* s_ws, void* stream) {
  const int64_t n = int64_t(n1) * n2;
  GemmArgs a{};
  a.qa = q_ws;
  a.sa = s_ws;
  a.T = T;
  a.K = int32_t(n);
  a.qw = qw;
  a.sw = sw;
  a.N = N;
  a.y = y;
  a.y_bf16 = y_bf16;
  a.stream = static_cast<cudaStream_t>(stream);
  if (!fused_dec_supported(a, n1, n2, x_dtype == FQ_BF16, p2)) return FQ_ENOTSUP;
  FdArgs f{x, n, n1, n2, p1, p2, alpha, x_dtype == FQ_BF16};
  const Span sqw = span(qw, size_t(N) * size_t(n / 2)), ssw = span(sw, size_t(N) * 4);
  const Span sp1 = span(p1, size_t(n1) * n1 * 2), sp2 = span(p2, size_t(n2) * n2 * 2);
  const Span sx = span(x, size_t(T) * size_t(n) * 2);
  const Span sq = span(q_ws, size_t(T) * size_t(n / 2)), ss = span(s_ws, size_t(T) * 4);
  const Span sy = span(y, size_t(T) * size_t(N) * 2);
  a.pdl = pdl_flags(a.stream, {sqw, ssw, sp1, sp2}, {sx}, {sq, ss, sy});
  const cudaError_t e = fused_dec_launch(a, f);
  if (e == cudaErrorNotSupported) return FQ_ENOTSUP;
  const fq_status s = cuda_status(e);
  if (s == FQ_OK) record_launch(a.stream, true, {sqw, ssw, sp1, sp2, sx}, {sq, ss, sy});
  return s;
}

}  // namespace fq

extern "C" {

fq_status fq_flatquant_linear(const void* x, int32_t x_dtype, int64_t T, int32_t n1, int32_t n2,
                              const void* p1, const void* p2, float alpha, const uint8_t* qw, const float* sw,
                              int32_t N, void* y, int32_t y_dtype, uint8_t* q_ws, float* s_ws, void* stream) {
  fq_status s = validate_linear(x, x_dtype, T, n1, n2, p1, p2, alpha, qw, sw, N, y, y_dtype, q_ws, s_ws);
  if (s != FQ_OK || T == 0 || N == 0) return s;
  const int64_t n = int64_t(n1) * n2;
  if (fused_enabled() && g_gemm_impl.load() == 0 && g_tq_impl.load() == 0) {
    // decode sizes: the transform runs inside the GEMM launch (NEXT-4(i)); FQ_ENOTSUP-free
    // fallback to the two kernels below when the shape has no fused kernel
    s = run_fused(x, x_dtype, T, n1, n2, p1, p2, alpha, qw, sw, N, y, y_dtype == FQ_BF16, q_ws, s_ws, stream);
    if (s != FQ_ENOTSUP) return s;
  }
  s = run_tq(x, x_dtype, T, n, n1, n2, p1, p2, alpha, q_ws, s_ws, nullptr, nullptr, stream);
  if (s != FQ_OK) return s;
  return run_gemm(q_ws, s_ws, T, int32_t(n), qw, sw, N, y, y_dtype == FQ_BF16, false, stream);
}

fq_status fq_flatquant_linear_host(const void* x_host, void* x_dev, int32_t x_dtype, int64_t T, int32_t n1,
                                   int32_t n2, const void* p1, const void* p2, float alpha, const uint8_t* qw,
                                   const float* sw, int32_t N, void* y_host, void* y_dev, int32_t y_dtype,
                                   uint8_t* q_ws, float* s_ws, void* stream) {
  fq_status s = fq_flatquant_linear_host_async(x_host, x_dev, x_dtype, T, n1, n2, p1, p2, alpha, qw, sw, N, y_host,
                                               y_dev, y_dtype, q_ws, s_ws, stream);
  if (s != FQ_OK || T == 0) return s;
  return cuda_status(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
}

fq_status fq_flatquant_linear_host_async(const void* x_host, void* x_dev, int32_t x_dtype, int64_t T, int32_t n1,
                                         int32_t n2, const void* p1, const void* p2, float alpha, const uint8_t* qw,
                                         const float* sw, int32_t N, void* y_host, void* y_dev, int32_t y_dtype,
                                         uint8_t* q_ws, float* s_ws, void* stream) {
  fq_status s = validate_linear(x_dev, x_dtype, T, n1, n2, p1, p2, alpha, qw, sw, N, y_dev, y_dtype, q_ws, s_ws);
  if (s != FQ_OK || T == 0) return s;
  if (!x_host || !x_dev || !y_host || !y_dev) return FQ_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t xbytes = size_t(T) * size_t(n1) * size_t(n2) * 2;
  const size_t ybytes = size_t(T) * size_t(N) * 2;
  s = cuda_status(cudaMemcpyAsync(x_dev, x_host, xbytes, cudaMemcpyHostToDevice, st));
  if (s != FQ_OK) return s;
  clear_outputs(st);               // the copy completes before any later kernel starts
  if (N > 0) {
    s = fq_flatquant_linear(x_dev, x_dtype, T, n1, n2, p1, p2, alpha, qw, sw, N, y_dev, y_dtype, q_ws, s_ws, stream);
    if (s != FQ_OK) return s;
  }
  s = cuda_status(cudaMemcpyAsync(y_host, y_dev, ybytes, cudaMemcpyDeviceToHost, st));
  if (s == FQ_OK) clear_outputs(st);
  return s;
}

fq_status fq_weight_colsum(const uint8_t* qw, int32_t N, int32_t K, int32_t* colsum, void* stream) {
  if (N < 0 || K < 0) return FQ_EINVAL;
  if (N == 0) return FQ_OK;
  if (!qw || !colsum) return FQ_EINVAL;
  if (K % 2 != 0) return FQ_ESHAPE;
  if ((reinterpret_cast<uintptr_t>(colsum) & 3u) != 0) return FQ_ESHAPE;
  const fq_status s = cuda_status(weight_colsum_launch(qw, N, K, colsum, static_cast<cudaStream_t>(stream)));
  if (s == FQ_OK) clear_outputs(static_cast<cudaStream_t>(stream));   // plain launch: completes before the next
  return s;
}

uint64_t fq_prepare_weight_workspace_size(int32_t n1, int32_t n2) {
  if (n1 < 1 || n2 < 1 || n1 > 256 || n2 > 256) return 0;
  return uint64_t(weight_prep_workspace(n1, n2));
}

fq_status fq_prepare_weight(const void* w, int32_t w_dtype, int32_t N, int64_t ldw, int32_t n1, int32_t n2,
                            const void* p1, const void* p2, float alpha_w, uint8_t* qw, float* sw,
                            int32_t* colsum_w, void* workspace, uint64_t workspace_bytes, void* stream) {
  fq_status s = validate_tq(w, w_dtype, N, ldw, n1, n2, p1, p2, alpha_w, qw, sw);
  if (s != FQ_OK || N == 0) return s;
  if (n1 > 256 || n2 > 256) return FQ_ENOTSUP;
  if (!workspace) return FQ_EINVAL;
  if (workspace_bytes < weight_prep_workspace(n1, n2)) return FQ_EINVAL;
  if ((reinterpret_cast<uintptr_t>(workspace) & 255u) != 0) return FQ_ESHAPE;
  if (colsum_w && (reinterpret_cast<uintptr_t>(colsum_w) & 3u) != 0) return FQ_ESHAPE;
  const size_t nm = size_t(n1 > n2 ? n1 : n2);
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  void* aug = ws;
  uint8_t* inv1 = ws + up(nm * 2 * nm * sizeof(double));
  uint8_t* inv2 = inv1 + up(size_t(n1) * n1 * 2);
  int* status = reinterpret_cast<int*>(inv2 + up(size_t(n2) * n2 * 2));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool bf16 = w_dtype == FQ_BF16;
  int h_status[2] = {0, 0};
  s = cuda_status(inverse_t_launch(p1, n1, bf16, aug, inv1, status, st));
  if (s != FQ_OK) return s;
  if (p2) {                                        // P2 = I: its inverse transpose is I as well
    s = cuda_status(inverse_t_launch(p2, n2, bf16, aug, inv2, status + 1, st));
    if (s != FQ_OK) return s;
  }
  s = cuda_status(cudaMemcpyAsync(h_status, status, sizeof(h_status), cudaMemcpyDeviceToHost, st));
  if (s != FQ_OK) return s;
  s = cuda_status(cudaStreamSynchronize(st));
  if (s != FQ_OK) return s;
  if (h_status[0] != 0 || (p2 && h_status[1] != 0)) return FQ_ESINGULAR;
  s = run_tq(w, w_dtype, N, ldw, n1, n2, inv1, p2 ? inv2 : nullptr, alpha_w, qw, sw, nullptr, nullptr, stream);
  if (s != FQ_OK) return s;
  if (colsum_w) {
    s = cuda_status(weight_colsum_launch(qw, N, n1 * n2, colsum_w, st));
    if (s != FQ_OK) return s;
  }
  // return once the prepared weights are written (the caller may hand them to another stream)
  s = cuda_status(cudaStreamSynchronize(st));
  if (s == FQ_OK) clear_outputs(st);
  return s;
}

fq_status fq_kv_quant(const void* kv, int32_t kv_dtype, int64_t R, int64_t ldkv, int32_t head_dim,
                      const void* p_h, float alpha, uint8_t* q, float* scale, int8_t* zero, void* stream) {
  if (kv_dtype != FQ_F16 && kv_dtype != FQ_BF16) return FQ_EINVAL;
  if (R < 0 || head_dim < 1 || ldkv < head_dim) return FQ_EINVAL;
  if (!(alpha > 0.f && alpha <= 1.f)) return FQ_EINVAL;
  if (R == 0) return FQ_OK;
  if (!kv || !p_h || !q || !scale || !zero) return FQ_EINVAL;
  if (head_dim != 64 && head_dim != 128) return FQ_ENOTSUP;
  KVArgs a{};
  a.x = kv;
  a.R = R;
  a.ldx = ldkv;
  a.D = head_dim;
  a.p = p_h;
  a.alpha = alpha;
  a.q = q;
  a.scale = scale;
  a.zero = zero;
  a.bf16 = kv_dtype == FQ_BF16;
  a.stream = static_cast<cudaStream_t>(stream);
  if (!kv_quant_supported(a)) return FQ_ESHAPE;
  const Span sq = span(q, size_t(R) * size_t(head_dim / 2)), ss = span(scale, size_t(R) * 4), sz = span(zero, size_t(R));
  const Span skv = span(kv, size_t(R - 1) * size_t(ldkv) * 2 + size_t(head_dim) * 2),
             sp = span(p_h, size_t(head_dim) * head_dim * 2);
  a.pdl = pdl_flags(a.stream, {sp}, {skv}, {sq, ss, sz});      // (the KV kernel waits before any access)
  const fq_status s = cuda_status(kv_quant_launch(a));
  if (s == FQ_OK) record_launch(a.stream, true, {skv, sp}, {sq, ss, sz});
  return s;
}

fq_status fq_choose_decomposition(int64_t n, int32_t* n1, int32_t* n2) {
  if (n < 1 || !n1 || !n2) return FQ_EINVAL;
  if (n > INT32_MAX) return FQ_ENOTSUP;
  int64_t b1 = 1, b2 = n;
  for (int64_t a = 1; a * a <= n; ++a)
    if (n % a == 0 && a + n / a < b1 + b2) {
      b1 = a;
      b2 = n / a;
    }
  *n1 = int32_t(b1);
  *n2 = int32_t(b2);
  return FQ_OK;
}

fq_status fq_set_tq_impl(int32_t impl) {
  if (impl < 0 || impl > 2) return FQ_EINVAL;
  g_tq_impl.store(impl);
  return FQ_OK;
}

fq_status fq_set_gemm_impl(int32_t impl) {
  if (impl < 0 || impl > 7) return FQ_EINVAL;
  g_gemm_impl.store(impl);
  return FQ_OK;
}

uint64_t fq_launch_count(void) { return g_launches.load(); }

const char* fq_status_string(int32_t status) {
  switch (status) {
    case FQ_OK: return "FQ_OK";
    case FQ_EINVAL: return "FQ_EINVAL: invalid argument";
    case FQ_ESHAPE: return "FQ_ESHAPE: unsupported shape, stride or alignment";
    case FQ_ENOTSUP: return "FQ_ENOTSUP: no kernel for this configuration";
    case FQ_ECUDA: return "FQ_ECUDA: CUDA error (see fq_last_cuda_error)";
    case FQ_ESINGULAR: return "FQ_ESINGULAR: transform matrix singular or its inverse overflows the dtype";
    default: return "unknown fq_status";
  }
}

int32_t fq_abi_version(void) { return FQ_ABI_VERSION; }
int32_t fq_last_cuda_error(void) { return g_last_cuda_error.load(); }

}  // extern "C"
