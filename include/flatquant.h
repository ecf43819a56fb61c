/*
 * flatquant.h -- C ABI of the B200-native FlatQuant online hot path
 * (arXiv 2410.09426, "FlatQuant: Flatness Matters for LLM Quantization").
 *
 * One linear layer Y = X W^T executed as
 *
 *   fq_transform_quant   a1-a5: y_t = vec_row(P1^T . reshape(x_t, n1, n2) . P2)   (Eq.3)
 *                               s_t = alpha . max|y_t| / 7                       (Eq.1 PAPER.md:90-93;
 *                               q   = clamp(rint(y / s_t), -8, 7), packed int4    PAPER.md:258-259, 367)
 *   fq_w4a4_linear       a6-a7: acc = Q_a Q_w^T (int32, exact), Y = acc . s_a[t] . s_w[o]
 *                               (INT4 GEMM PAPER.md:315, per-channel weights PAPER.md:367)
 *
 * Conventions common to every entry point
 *  - Pointers named x, p1, p2, q, scale, qa, sa, qw, sw, y, acc are DEVICE pointers
 *    (cudaMalloc / torch CUDA storage) unless the name ends in _host.  All buffers are
 *    caller-allocated; the library never allocates, frees or retains them.  They must stay
 *    valid until the work queued on `stream` has completed.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Every call
 *    is asynchronous with respect to the host unless stated otherwise.
 *  - Stream order.  Every call is ordered after the work already enqueued on `stream`, as
 *    with any CUDA library.  The kernels use programmatic dependent launch (PDL) to overlap
 *    with the kernel before them: each kernel lets its dependents launch only after its own
 *    griddepcontrol.wait has returned, so a kernel that has not yet waited can overlap only its
 *    immediate predecessor on the stream.  The library records, per stream, the buffers its last
 *    kernel reads and writes; the next kernel reads its parameters (p1, p2, qw, sw, colsum_w)
 *    or its activations (x, qa, sa, za) before the wait only if the predecessor does not write
 *    them, and writes its outputs before the wait only if the predecessor neither reads nor
 *    writes them -- otherwise it waits first.  So weights and transforms stream in while the
 *    previous kernel finishes, and a call whose buffers are disjoint from the previous call's
 *    (e.g. the next layer linear's transform after a GEMM) runs concurrently with it, while
 *    any real dependency (read-after-write, write-after-read, write-after-write) is ordered.
 *    Work of other origin between two calls (copies, kernels without an early PDL trigger)
 *    completes before a PDL kernel may start.  The one case the library cannot see: a kernel
 *    of ANOTHER library that triggers its dependents early and touches this library's buffers
 *    immediately before a call; synchronise or record an event between them in that case.
 *  - Argument validation is synchronous: on any error nothing is launched and a non-zero
 *    fq_status is returned.  T == 0 returns FQ_OK without launching.  A failed launch
 *    returns FQ_ECUDA; fq_last_cuda_error() returns the cudaError_t value.  Device faults
 *    surface at the caller's next synchronisation, as with any CUDA library.
 *  - Layouts are row-major.  INT4 codes are two's-complement nibbles, element 2i in the
 *    LOW nibble of byte i of its row (reading R7).  Alignment: every pointer
 *    is aligned to its element size; in addition the tensor-core paths (the GEMM, and the
 *    transform when n1 % 16 == 0 and n2 % 16 == 0) need x, q, qa, qw, y and sw 16-byte
 *    aligned and row strides that are multiples of 16 bytes (FQ_ESHAPE otherwise).
 *  - Re-entrant.  Per-device kernel attributes are set once per (kernel, device), thread-safely;
 *    the host state is the per-stream record of the last launch's buffers (see Stream order),
 *    guarded by a mutex.  Device state: the transform kernel's dynamic tile schedule and the
 *    fused decode linear count through per-launch counter pairs taken round-robin from rings of
 *    1024 slots per device in the library's own (module) device memory; each launch's last CTA
 *    resets its slot, so CUDA-graph replays are safe.  At most 1024 such launches of each kind
 *    may be in flight on one device at a time; a captured launch keeps the slot it was given at
 *    capture, so one graph must not be replayed concurrently with itself (on two streams).
 *  - Non-finite inputs give unspecified codes (the oracle's precondition is finite x).
 */
#ifndef FLATQUANT_H_
#define FLATQUANT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FQ_ABI_VERSION 5   /* 2: FQ_ASYM + fq_weight_colsum; 3: fq_kv_quant, fq_prepare_weight; 4: p2 = NULL (P2 = I);
                              5: K < 131072, PDL hazard check on inputs/outputs, bf16 P2 scaled into fp16 range */

typedef enum {
  FQ_OK = 0,
  FQ_EINVAL = 1,   /* null pointer, bad enum, alpha outside (0, 1], negative size          */
  FQ_ESHAPE = 2,   /* n1*n2 != K, odd K, K % 32 != 0 for the GEMM, misaligned pointer/stride */
  FQ_ENOTSUP = 3,  /* well-formed but no kernel for it (e.g. n1 or n2 > 256)                 */
  FQ_ECUDA = 4,    /* a CUDA launch/runtime call failed; see fq_last_cuda_error()            */
  FQ_ESINGULAR = 5 /* fq_prepare_weight: P1 or P2 singular, or its inverse overflows the dtype */
} fq_status;

typedef enum { FQ_F16 = 0, FQ_BF16 = 1 } fq_dtype;

/* FQ_SYM: per-token symmetric (the paper's setting).
 * FQ_ASYM: per-token asymmetric min-max (DESIGN.md reading
 *   R19): lo = min(alpha min y, 0), hi = max(alpha max y, 0), s = (hi - lo) / 15 (1 if hi == lo),
 *   z = rint(-lo / s) in [0, 15], q = clamp(rint(y / s) + z, 0, 15); the nibble stores q - 8
 *   (two's complement, so the GEMM's signed widening is unchanged) and zero[t] stores z - 8. */
typedef enum { FQ_SYM = 0, FQ_ASYM = 1 } fq_qmode;

/* ---------------------------------------------------------------------------------------
 * fq_transform_quant -- fused Kronecker transform + clip + per-token INT4 quantize + pack.
 *   PAPER.md:236-244 (Eq.3, activation factor Q(P1^T x_1 X~ x_2 P2))
 *   (clipping ratio after the transform), PAPER.md:367 (per-token symmetric), Eq.1.
 *
 *   x      [T, ldx] elements of x_dtype; row t holds x_t (n = n1*n2 used), ldx >= n.
 *          Viewed as V_t = reshape(x_t, n1, n2) in C order.
 *   p1     [n1, n1] row-major, x_dtype.     p2 [n2, n2] row-major, x_dtype, or NULL for
 *          P2 = I_{n2}: the paper's online o_proj transform P_o (a x a) applied across the a
 *          heads of the attention output, identity inside each head of d_head = n2
 *          (PAPER.md:297 P_v fused, PAPER.md:726 a^2 parameters); stage 2 is skipped and the
 *          fp32 result of P1^T V is quantized directly (tcgen05 kernel; FQ_SYM and FQ_ASYM).
 *          Shapes (n1, n2) in {(32, 128), (64, 128)}; FQ_ENOTSUP otherwise.
 *   alpha  post-sigmoid clipping ratio in (0, 1]; 1 = no clipping.
 *   qmode  FQ_SYM or FQ_ASYM.
 *   q      [T, n/2] uint8 packed codes (output).     scale [T] fp32 (output), s_t.
 *   zero   FQ_SYM: must be NULL.  FQ_ASYM: [T] int8 (output), z_t - 8.
 *   FQ_ASYM runs on the tcgen05 kernel shapes and the CUDA-core kernel (n1 n2 <= 25600);
 *   other shapes return FQ_ENOTSUP.
 *   Supported (FQ_ENOTSUP otherwise): n even, 1 <= n1, n2 <= 256, and a kernel for the shape:
 *   tcgen05 for (64, 64), (64, 128), ({80, 96, 112, 128}, 128), (128, {160, 192, 224, 256});
 *   mma.sync for the other multiples of 16 listed in DESIGN.md (Fig. 5 decompositions); the
 *   CUDA-core fp32 kernel for any shape with n1 n2 <= 25600.
 *   Precision: X and P in x_dtype; stage 1 (P1^T V) accumulates in fp32; the intermediate is
 *   re-fed to the second stage as fp16 after an exact per-token power-of-two prescale (never
 *   bf16, R9).  A bf16 P2 is likewise scaled by a power of two into fp16 range (its
 *   largest entry to [2^14, 2^15)), so no entry overflows; 2^-e is divided out exactly.
 * ------------------------------------------------------------------------------------- */
fq_status fq_transform_quant(const void* x, int32_t x_dtype, int64_t T, int64_t ldx,
                             int32_t n1, int32_t n2, const void* p1, const void* p2,
                             float alpha, int32_t qmode, uint8_t* q, float* scale,
                             int8_t* zero, void* stream);

/* fq_transform_f32 -- same kernel as fq_transform_quant, additionally exporting the
 * transformed activations y [T, n] fp32 (before clipping/quantization; 8-byte aligned) so
 * that the "transformed activations rel 1e-3" bar can be checked on the production code
 * path.  q and scale are written exactly as by fq_transform_quant (both required). */
fq_status fq_transform_f32(const void* x, int32_t x_dtype, int64_t T, int64_t ldx,
                           int32_t n1, int32_t n2, const void* p1, const void* p2,
                           float alpha, uint8_t* q, float* scale, float* y, void* stream);

/* ---------------------------------------------------------------------------------------
 * fq_w4a4_linear -- W4A4 GEMM + dequant epilogue.
 *   Y[t, o] = cvt_rn( float(acc[t, o]) * sa[t] * sw[o] ),  acc = sum_k qa[t,k] qw[o,k]
 *   PAPER.md:241 (weights pre-transformed offline, P1^{-1} x_1 W~ x_2 P2^{-T})
 *   (INT4 GEMM), PAPER.md:367 (per-token x per-channel scales).
 *
 *   qa [T, K/2] uint8 packed activation codes (from fq_transform_quant), sa [T] fp32.
 *   qw [N, K/2] uint8 packed weight codes (K contiguous, same nibble order), sw [N] fp32.
 *   za, colsum_w: both NULL (symmetric activations) or both set (FQ_ASYM activations):
 *      za [T] int8 = z_t - 8 from fq_transform_quant, colsum_w [N] int32 = sum_k qw[o,k]
 *      (fq_weight_colsum, computed once per weight).  Then
 *      Y[t,o] = cvt_rn( float(acc[t,o] - za[t] colsum_w[o]) * sa[t] * sw[o] ), i.e. the
 *      dequantized product s_a (q - z) . s_w q_w.  Asymmetric inputs need the default GEMM
 *      implementation (fq_set_gemm_impl 0) or a tcgen05 pair / decode one (3-6); FQ_ENOTSUP
 *      otherwise.
 *   y  [T, N] of y_dtype (FQ_F16 or FQ_BF16), row-major.
 *   Requires K % 32 == 0, K < 131072 and N % 8 == 0 (FQ_ESHAPE / FQ_ENOTSUP otherwise).
 *   Exact integer accumulation: the tensor core accumulates 256 acc (operands widened to 16 q),
 *   |256 acc| <= 2^14 K < 2^31; the asymmetric correction is applied after the exact division
 *   by 256, |acc - za colsum_w| <= 120 K.
 * ------------------------------------------------------------------------------------- */
fq_status fq_w4a4_linear(const uint8_t* qa, const float* sa, const int8_t* za, int64_t T,
                         int32_t K, const uint8_t* qw, const float* sw,
                         const int32_t* colsum_w, int32_t N, void* y, int32_t y_dtype,
                         void* stream);

/* fq_weight_colsum -- colsum[o] = sum_k qw[o,k] (int32, exact) of packed weight codes [N, K/2];
 * offline preparation for asymmetric activations (fq_w4a4_linear's colsum_w). */
fq_status fq_weight_colsum(const uint8_t* qw, int32_t N, int32_t K, int32_t* colsum, void* stream);

/* fq_w4a4_gemm_i32 -- the same GEMM kernel exporting the raw int32 accumulators
 * acc [T, N] (bit-exactness bar).  Same shape requirements as fq_w4a4_linear. */
fq_status fq_w4a4_gemm_i32(const uint8_t* qa, int64_t T, int32_t K, const uint8_t* qw,
                           int32_t N, int32_t* acc, void* stream);

/* ---------------------------------------------------------------------------------------
 * fq_flatquant_linear -- the whole hot path a1-a7 for one linear layer: transform+quant of
 * x into the caller's workspace (q_ws [T, n/2] uint8, s_ws [T] fp32), then the W4A4 GEMM.
 * Equivalent to fq_transform_quant followed by fq_w4a4_linear on the same stream: q_ws, s_ws
 * and y hold bit-identical results either way.
 * Decode sizes run FUSED in ONE launch (PAPER.md:312-314 fuses the
 * transform and quantization into one kernel, here it is fused into the GEMM as well): for
 * 1 <= T <= 64, (n1, n2) = (64, 64), (64, 128) or (112, 128), fp16 or bf16 x and p2 != NULL, the
 * first CTAs of the decode GEMM transform one tile each (two tokens at 64 x 64 and 64 x 128, one at
 * 112 x 128) into q_ws/s_ws
 * (L2-resident at these sizes) while the other CTAs already stream their weights, and the GEMM
 * reads the codes once all tiles are published.  Tile
 * publication uses a {arrivals, departures} counter pair from a ring of 1024 slots per device in
 * the library's own device memory, reset by the last CTA of each launch (so CUDA-graph replay is
 * safe); at most 1024 fused launches may be in flight on one device at a time.  The fused
 * launch also needs its whole grid resident at once (N <= 37888: 128 outputs per CTA, two
 * CTAs per SM) and at least one CTA per tile.  Every other shape, dtype, T or N runs the two kernels.
 * Fused launches running concurrently on several streams also rely on each grid's first blocks
 * (the tickets) being dispatched no later than its others, as the hardware does (tests run three
 * streams); a CTA that waits more than ~35 s for the tiles traps (a launch error), it does not hang.
 * ------------------------------------------------------------------------------------- */
fq_status fq_flatquant_linear(const void* x, int32_t x_dtype, int64_t T, int32_t n1,
                              int32_t n2, const void* p1, const void* p2, float alpha,
                              const uint8_t* qw, const float* sw, int32_t N, void* y,
                              int32_t y_dtype, uint8_t* q_ws, float* s_ws, void* stream);

/* fq_flatquant_linear_host -- as fq_flatquant_linear but x_host [T, n] and y_host [T, N]
 * are HOST buffers (page-locked strongly recommended): copies x_host -> x_dev, runs the hot
 * path, copies y_dev -> y_host, all on `stream`, then synchronises the stream before
 * returning (so y_host is valid on return).  x_dev/y_dev are caller-provided device staging
 * buffers of the same shapes. */
fq_status fq_flatquant_linear_host(const void* x_host, void* x_dev, int32_t x_dtype,
                                   int64_t T, int32_t n1, int32_t n2, const void* p1,
                                   const void* p2, float alpha, const uint8_t* qw,
                                   const float* sw, int32_t N, void* y_host, void* y_dev,
                                   int32_t y_dtype, uint8_t* q_ws, float* s_ws, void* stream);

/* fq_flatquant_linear_host_async -- fq_flatquant_linear_host WITHOUT the final
 * synchronisation: the H2D copy, the hot path and the D2H copy are only enqueued on `stream`;
 * y_host is valid once the caller has synchronised the stream.  With page-locked buffers the
 * copies are asynchronous, so linears issued on different streams overlap their transfers
 * (PCIe is full duplex) with each other's compute. */
fq_status fq_flatquant_linear_host_async(const void* x_host, void* x_dev, int32_t x_dtype,
                                         int64_t T, int32_t n1, int32_t n2, const void* p1,
                                         const void* p2, float alpha, const uint8_t* qw,
                                         const float* sw, int32_t N, void* y_host, void* y_dev,
                                         int32_t y_dtype, uint8_t* q_ws, float* s_ws, void* stream);

/* ---------------------------------------------------------------------------------------
 * fq_prepare_weight -- offline weight side of Eq. 3 on the GPU:
 *   W'_o = P1^{-1} W~_o P2^{-T}     (W~_o = row o of W reshaped n1 x n2)
 *   then per-output-channel symmetric INT4 with clipping alpha_w:
 *   sw[o] = alpha_w max|W'_o| / 7, qw[o] = clamp(rint(W'_o / sw[o]), -8, 7), packed as the
 *   activations are (R7).  Steps, all on `stream`: P1^{-T} and P2^{-T} by Gauss-Jordan with
 *   partial pivoting in float64 (rounded to w_dtype), then the fq_transform_quant kernel with
 *   (P1^{-T}, P2^{-T}, alpha_w) -- (P1^{-T})^T W~ P2^{-T} is the weight factor -- and, if
 *   colsum_w is not NULL, fq_weight_colsum.
 *   w       [N, n1 n2] fp16/bf16 (w_dtype), row stride ldw elements.
 *   p1, p2  [n1, n1], [n2, n2] row-major, same dtype (the activation-side transforms);
 *           p2 NULL = I_{n2} as in fq_transform_quant (then P2^{-T} = I).
 *   qw      [N, n1 n2 / 2] uint8 (output).  sw [N] fp32 (output).  colsum_w [N] int32 or NULL.
 *   workspace  device buffer of fq_prepare_weight_workspace_size(n1, n2) bytes, 256-byte
 *           aligned; scratch, contents undefined on return.
 *   SYNCHRONOUS: waits for `stream` to read the inversion status; returns FQ_ESINGULAR if a
 *   pivot is zero/non-finite or the inverse does not fit the dtype (nothing else launched).
 *   n1, n2 <= 256 and the shape rules of fq_transform_quant.
 * ------------------------------------------------------------------------------------- */
fq_status fq_prepare_weight(const void* w, int32_t w_dtype, int32_t N, int64_t ldw, int32_t n1,
                            int32_t n2, const void* p1, const void* p2, float alpha_w,
                            uint8_t* qw, float* sw, int32_t* colsum_w, void* workspace,
                            uint64_t workspace_bytes, void* stream);

/* Workspace bytes fq_prepare_weight needs for (n1, n2); 0 for invalid sizes. */
uint64_t fq_prepare_weight_workspace_size(int32_t n1, int32_t n2);

/* ---------------------------------------------------------------------------------------
 * fq_kv_quant -- KV-cache quantization: per-head transform and
 * group-wise asymmetric INT4 with one group per head vector.
 *   y_r = kv_r . P_h   (§3.2: P_h transforms the keys head by head; values
 *                       use P = I since P_v is merged into the weights)
 *   s_r = alpha (hi - lo) / 15, z_r = rint(-alpha lo / s_r), q = clamp(rint(y / s) + z, 0, 15)
 *   with hi = max(max_j y_rj, 0), lo = min(min_j y_rj, 0) (reading R19); group size =
 *   head_dim ("group-wise asymmetric ... size of 128" = head dim).
 *   kv     [R, head_dim] fp16/bf16 (kv_dtype), row stride ldkv elements; R = tokens x heads.
 *   p_h    [head_dim, head_dim] row-major, same dtype as kv (identity for values).
 *   alpha  KV clipping threshold in (0, 1].
 *   q      [R, head_dim/2] uint8 packed nibbles q - 8 (output).   scale [R] fp32 (output).
 *   zero   [R] int8, z - 8 (output).       Dequantization: s (q - z) = s ((q-8) - (z-8)).
 *   head_dim 64 or 128 (FQ_ENOTSUP otherwise); kv, p_h, q 16-byte aligned and ldkv * 2 a
 *   multiple of 16 (FQ_ESHAPE otherwise).  One tcgen05 kernel launch.
 * ------------------------------------------------------------------------------------- */
fq_status fq_kv_quant(const void* kv, int32_t kv_dtype, int64_t R, int64_t ldkv,
                      int32_t head_dim, const void* p_h, float alpha, uint8_t* q,
                      float* scale, int8_t* zero, void* stream);

/* ---------------------------------------------------------------------------------------
 * Helpers
 * ------------------------------------------------------------------------------------- */
/* (n1, n2) = argmin(n1 + n2) s.t. n1 n2 = n, n1 <= n2.  Host-only, sync. */
fq_status fq_choose_decomposition(int64_t n, int32_t* n1, int32_t* n2);

/* Selects the GEMM implementation for subsequent calls in this process (testing aid):
 * 0 = default (T <= 64: the decode kernel; otherwise tcgen05 kind::i8 on a CTA pair,
 * cta_group::2, tile width 192/160/128 features picked per shape to fill the last wave),
 * 1 = legacy mma.sync cross-check kernel, 2 = tcgen05 kind::i8 on a single CTA, 3 / 4 / 5 = the
 * pair kernel with the tile width forced to 192 / 160 / 128 (7: 256, one accumulator), 6 = the
 * decode kernel forced
 * (swapped operands: 128 weight rows x T tokens per CTA, K split across a cluster and reduced
 * through distributed shared memory; T <= 64, FQ_ENOTSUP otherwise).  All bit-identical.
 * Returns FQ_EINVAL otherwise. */
fq_status fq_set_gemm_impl(int32_t impl);

/* Selects the transform+quant implementation for subsequent calls in this process (testing
 * aid): 0 = default (tcgen05/TMEM/TMA kernel for n2 in {64,128} with n1 = 64, or n2 = 128 with
 * n1 in {80,96,112,128}; the wide tcgen05 kernel for n1 = 128, n2 in {160,192,224,256}; the
 * CUDA-core kernel for n1 n2 <= 1024; otherwise the legacy mma.sync kernel where instantiated,
 * else the CUDA-core kernel), 1 = legacy mma.sync kernel (else CUDA cores), 2 = CUDA-core
 * kernel.  p2 = NULL (P2 = I) runs the tcgen05 kernel's stage-1-only variant (impl 0) or the
 * mma.sync one (impl 1, symmetric only).  Returns FQ_EINVAL otherwise.
 * All implementations compute the same function. */
fq_status fq_set_tq_impl(int32_t impl);

/* Number of kernel launches issued by this library since process start (bench accounting). */
uint64_t fq_launch_count(void);

const char* fq_status_string(int32_t status);
int32_t fq_abi_version(void);
int32_t fq_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FLATQUANT_H_ */
