// fq_device.cuh -- small sm_100a device helpers (PTX wrappers) shared by the kernels.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

#define FQ_DEVICE __device__ __forceinline__

namespace fq {

FQ_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- cp.async (LDGSTS) -------------------------------------------------------------------
FQ_DEVICE void cp_async16(void* smem, const void* gmem, bool pred) {
  const int n = pred ? 16 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(n));
}
FQ_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
FQ_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- named barriers ----------------------------------------------------------------------
FQ_DEVICE void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- ldmatrix ------------------------------------------------------------------------------
FQ_DEVICE void ldsm_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
FQ_DEVICE void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// ---- legacy warp MMA (HMMA / IMMA) -----------------------------------------------------
template <bool BF16>
FQ_DEVICE void mma_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (BF16) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
}

FQ_DEVICE void mma_s8_16832(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// ---- conversions --------------------------------------------------------------------------
FQ_DEVICE uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <typename T>
FQ_DEVICE float to_f32(T v);
template <>
FQ_DEVICE float to_f32<__half>(__half v) { return __half2float(v); }
template <>
FQ_DEVICE float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
FQ_DEVICE T from_f32(float v);
template <>
FQ_DEVICE __half from_f32<__half>(float v) { return __float2half_rn(v); }
template <>
FQ_DEVICE __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Sign-extend the 8 two's-complement nibbles of w (element 2i in the low nibble of byte i)
// into 8 int8 values, in natural element order: lo word = e0..e3, hi word = e4..e7.
FQ_DEVICE void widen_int4x8(uint32_t w, uint32_t& lo, uint32_t& hi) {
  // even elements (low nibbles) and odd elements (high nibbles) as zero-extended bytes
  uint32_t ev = w & 0x0F0F0F0Fu;          // bytes: e0 e2 e4 e6
  uint32_t od = (w >> 4) & 0x0F0F0F0Fu;   // bytes: e1 e3 e5 e7
  // sign extension per byte: s = (u + 0x78) ^ 0x78 maps 0..7 -> 0..7, 8..15 -> 0xF8..0xFF
  ev = (ev + 0x78787878u) ^ 0x78787878u;
  od = (od + 0x78787878u) ^ 0x78787878u;
  // interleave: lo = e0 e1 e2 e3 ; hi = e4 e5 e6 e7
  lo = __byte_perm(ev, od, 0x5140);
  hi = __byte_perm(ev, od, 0x7362);
}

FQ_DEVICE float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Exponent e with max * 2^e in [2^14, 2^15) for a finite max >= 0 (biased-exponent arithmetic,
// exact); 0 for max == 0; clamped to [-126, 126].
FQ_DEVICE int p2_scale_exp(uint32_t max_bits) {
  const int be = int(max_bits >> 23);
  if (max_bits == 0) return 0;
  const int e = 14 - ((be == 0 ? 1 : be) - 127);
  return e < -126 ? -126 : (e > 126 ? 126 : e);
}

// A bf16 matrix P (row-major, `elems` entries at p, 16-byte aligned, in shared memory) becomes
// fp16 P * 2^e IN PLACE, with e from p2_scale_exp(max |P|) so that the largest entry lands in
// [2^14, 2^15): every bf16 entry >= 2^-17 of that range is exact in fp16 (8-bit bf16 mantissa),
// none can overflow, and the caller divides 2^e out of the result exactly (DESIGN.md reading
// R9: the second Kronecker stage runs in fp16 with its fp16 intermediate).  Whole block; `red`
// is one shared word; returns e.  Ends with the smem writes visible to the async proxy and
// the block synchronised.
FQ_DEVICE int bf16_to_f16_pow2(uint8_t* p, int elems, uint32_t* red) {
  uint4* v4 = reinterpret_cast<uint4*>(p);
  const int n4 = elems / 8;
  if (threadIdx.x == 0) *red = 0u;
  __syncthreads();
  uint32_t m = 0;
  for (int i = threadIdx.x; i < n4; i += blockDim.x) {
    const uint4 v = v4[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) m = max(m, max((w[h] << 16) & 0x7FFFFFFFu, w[h] & 0x7FFF0000u));
  }
  m = __reduce_max_sync(0xffffffffu, m);        // |x| bit patterns order like the values
  if ((threadIdx.x & 31) == 0) atomicMax(red, m);
  __syncthreads();
  const int e = p2_scale_exp(*red);
  const float sc = __int_as_float((127 + e) << 23);
  for (int i = threadIdx.x; i < n4; i += blockDim.x) {
    uint4 v = v4[i];
    uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
    for (int h = 0; h < 4; ++h)
      w[h] = pack_half2(__uint_as_float(w[h] << 16) * sc, __uint_as_float(w[h] & 0xFFFF0000u) * sc);
    v4[i] = v;
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  return e;
}

// bf16_to_f16_pow2 for one group of `nthreads` threads (this thread is `tid`) that synchronises
// through named barrier `bar` instead of the whole block (the fused decode linear's epilogue warps):
// the same maximum, exponent and conversion, so the result is bit-identical.
FQ_DEVICE int bf16_to_f16_pow2_group(uint8_t* p, int elems, uint32_t* red, int tid, int nthreads, int bar) {
  uint4* v4 = reinterpret_cast<uint4*>(p);
  const int n4 = elems / 8;
  if (tid == 0) *red = 0u;
  named_bar_sync(bar, nthreads);
  uint32_t m = 0;
  for (int i = tid; i < n4; i += nthreads) {
    const uint4 v = v4[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) m = max(m, max((w[h] << 16) & 0x7FFFFFFFu, w[h] & 0x7FFF0000u));
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if ((tid & 31) == 0) atomicMax(red, m);
  named_bar_sync(bar, nthreads);
  const int e = p2_scale_exp(*red);
  const float sc = __int_as_float((127 + e) << 23);
  for (int i = tid; i < n4; i += nthreads) {
    uint4 v = v4[i];
    uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
    for (int h = 0; h < 4; ++h)
      w[h] = pack_half2(__uint_as_float(w[h] << 16) * sc, __uint_as_float(w[h] & 0xFFFF0000u) * sc);
    v4[i] = v;
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  named_bar_sync(bar, nthreads);
  return e;
}

}  // namespace fq
