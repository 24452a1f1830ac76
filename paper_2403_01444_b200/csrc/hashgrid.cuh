// Hash-grid encoding shared by the NTC kernels (ntc.cu) and the fused
// gather + tcgen05 decoder (mlp_tc.cu).  Reference: ntc.py:161-203.
#pragma once

#include "common.cuh"

namespace ss {

// ------------------------------------------------------------------ encode
// Normalised position in float64, exactly (x - lo) / (hi - lo), clipped
// (ntc.py:166-169).  Returns false when outside by more than 1e-9.
__device__ inline bool normalise(const ss_grid& g, const float* m, double xn[3]) {
  bool ok = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double lo = g.aabb_min[d], hi = g.aabb_max[d];
    double v = __ddiv_rn(__dsub_rn((double)m[d], lo), __dsub_rn(hi, lo));
    ok &= (v >= -1e-9) && (v <= 1.0 + 1e-9);
    xn[d] = fmin(fmax(v, 0.0), 1.0);
  }
  return ok;
}

// Corner rows and trilinear weights of one level (ntc.py:176-186, :192-203).
// Corner k = (k&1, k>>1&1, k>>2&1), x fastest (ntc.py:25-27).
__device__ inline void level_corners(const ss_grid& g, int l, const double xn[3],
                                     uint32_t idx[8], float w[8]) {
  const int res = g.resolution[l];
  const uint32_t T = 1u << g.log2_table;
  double fr[3];
  uint32_t c0[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double pos = __dmul_rn(xn[d], (double)res);
    double f = fmin(floor(pos), (double)(res - 1));
    c0[d] = (uint32_t)f;
    fr[d] = __dsub_rn(pos, f);
  }
  const int64_t side = (int64_t)res + 1;
  const bool dense = side * side * side <= (int64_t)T;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t ox = k & 1, oy = (k >> 1) & 1, oz = (k >> 2) & 1;
    double tx = ox ? fr[0] : __dsub_rn(1.0, fr[0]);
    double ty = oy ? fr[1] : __dsub_rn(1.0, fr[1]);
    double tz = oz ? fr[2] : __dsub_rn(1.0, fr[2]);
    w[k] = (float)__dmul_rn(__dmul_rn(tx, ty), tz);
    uint32_t cx = c0[0] + ox, cy = c0[1] + oy, cz = c0[2] + oz;
    if (dense) {
      idx[k] = cx + (uint32_t)side * (cy + (uint32_t)side * cz);
    } else {
      // int64 (x*1 ^ y*2654435761 ^ z*805459861) % T == uint32-wrap & (T-1)
      idx[k] = (cx ^ (cy * 2654435761u) ^ (cz * 805459861u)) & (T - 1u);
    }
  }
}

}  // namespace ss
