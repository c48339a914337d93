// Plane sets of the densify stage: up to three H x W planes, each stored as
// f32 or f64 (the pipeline keeps the flow numerators in f32 and the
// indicator, whose ratio against the 1e-4 floor must not flip, in f64).
#pragma once
#include "hdr_internal.h"

namespace hdr {

__device__ __forceinline__ double ldp(const DtPlanes& P, int k, int64_t i) {
  return P.f64[k] ? reinterpret_cast<const double*>(P.p[k])[i]
                  : (double)reinterpret_cast<const float*>(P.p[k])[i];
}

__device__ __forceinline__ void stp(const DtPlanes& P, int k, int64_t i, double v) {
  if (P.f64[k]) reinterpret_cast<double*>(P.p[k])[i] = v;
  else reinterpret_cast<float*>(P.p[k])[i] = (float)v;
}

}  // namespace hdr
