// Small device-side float helpers shared by the kernels (header-only).
#pragma once

namespace rsdb {

// max that propagates NaN (IEEE 754-2019 maximum): one NaN element makes a
// block's absmax NaN (readings R27 / R28)
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

constexpr float FLT_MAX_F = 3.402823466e38f;

}  // namespace rsdb
