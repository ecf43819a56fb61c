// fq_quant.cuh -- per-token INT4 quantization arithmetic shared by the transform kernel
// (fq_tq_tc05.cu) and the fused decode linear (fq_gemm_dec.cu), so both produce bit-identical
// codes and scales from the same transformed values.
//   s_t = alpha max|y_t| / 7 (1 if y_t == 0), q = clamp(rint(y / s_t), -8, 7)   (Eq.1,
//   PAPER.md:258-259 clipping, PAPER.md:367 per-token symmetric; readings R4-R7)
#pragma once
#include <cstdint>
#include "fq_device.cuh"

namespace fq {
namespace qz {

constexpr float MAGIC = 12582912.0f;   // 1.5 * 2^23: fma(y, c, MAGIC) rounds y*c half-to-even

// per-token exact power-of-two exponent e with m * 2^e in [2^14, 2^15) (fp16-safe); m >= 0 and
// finite.  A subnormal (or zero) m gets the largest scale 2^126.
FQ_DEVICE int prescale_exp(float m) {
  const int be = int(__float_as_uint(m) >> 23);       // biased exponent (sign bit is 0)
  if (be == 0) return 126;
  const int e = 14 - (be - 127);
  return e < -126 ? -126 : (e > 126 ? 126 : e);
}

FQ_DEVICE float exp2i(int e) { return __int_as_float((127 + e) << 23); }

FQ_DEVICE float max3f(float a, float b, float c) {   // FMNMX3 (sm_100); |.| folds into operand modifiers
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
FQ_DEVICE float fma_sat(float a, float b, float c) {  // FFMA.SAT: clamp to [0, 1]
  float r;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// 8 quantized values in MAGIC form (low nibble of the bit pattern = two's-complement code)
// -> one 32-bit word, element 2m in the low nibble of byte m.
FQ_DEVICE uint32_t pack8(const float (&v)[8]) {
  const uint32_t e = __byte_perm(__byte_perm(__float_as_uint(v[0]), __float_as_uint(v[2]), 0x0040),
                                 __byte_perm(__float_as_uint(v[4]), __float_as_uint(v[6]), 0x0040), 0x5410);
  const uint32_t o = __byte_perm(__byte_perm(__float_as_uint(v[1]), __float_as_uint(v[3]), 0x0040),
                                 __byte_perm(__float_as_uint(v[5]), __float_as_uint(v[7]), 0x0040), 0x5410);
  return (e & 0x0F0F0F0Fu) | ((o << 4) & 0xF0F0F0F0u);
}

// symmetric quantizer constants from the token statistic m = max|y| (prescaled values):
// code = clamp(rint(y * 7 / (alpha m)), -8, 7) = fma(sat(y c15 + 8/15), 15, MAGIC - 8)
FQ_DEVICE float sym_c15(float alpha, float m) { return m > 0.f ? __fdividef(7.0f / 15.0f, alpha * m) : 0.f; }
FQ_DEVICE float sym_code(float y, float c15) {
  return fmaf(fma_sat(y, c15, 8.0f / 15.0f), 15.0f, MAGIC - 8.0f);
}

}  // namespace qz
}  // namespace fq
