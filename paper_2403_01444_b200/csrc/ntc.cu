// Neural Transformation Cache on sm_100a: hash-grid encode (K1f), fused
// decoder + transform (K2f/K3f), fused transform/decoder backward with the
// hash-table scatter (K3b/K2b/K1b), and the lazy Adam step (KA).
//
// Reference: ntc.py:161-293, transform.py:53-135, optim.py:33-66
// (/root/reference/pkg/src/splatstream/).
#include <mutex>

#include "common.cuh"

namespace ss {

constexpr int HID = 64;
constexpr int OUTP = 8;
constexpr int kChunk = 128;  // Gaussians per CTA pass in the backward

__constant__ ShRotConst c_shrot;
static std::mutex g_const_mu;
static int g_const_device = -1;

int ensure_shrot_const() {
  int dev = 0;
  SS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_const_mu);
  if (g_const_device == dev) return SS_OK;
  ShRotConst h{};
  build_shrot_host(&h);
  SS_CUDA(cudaMemcpyToSymbol(c_shrot, &h, sizeof(h)));
  g_const_device = dev;
  return SS_OK;
}

template <int IN, int NL>
struct Lay {
  static constexpr int W0 = 0, B0 = IN * HID, W1 = B0 + HID;
  static constexpr int B1 = W1 + (NL == 2 ? HID * HID : 0);
  static constexpr int W2 = B1 + (NL == 2 ? HID : 0);
  static constexpr int B2 = W2 + HID * OUTP;
  static constexpr int TOTAL = B2 + OUTP;
};

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

// Interpolated features (ntc.py:205-216), zero-padded to IN.
template <int IN>
__device__ inline void gather_features(const ss_grid& g, const float* __restrict__ tables,
                                       const double xn[3], float (&x)[IN]) {
#pragma unroll
  for (int i = 0; i < IN; ++i) x[i] = 0.f;
  const int F = g.n_features;
  const size_t T = (size_t)1 << g.log2_table;
  if (F == 2) {
#pragma unroll
    for (int l = 0; l < IN / 2; ++l) {
      if (l < g.n_levels) {
        uint32_t idx[8];
        float w[8];
        level_corners(g, l, xn, idx, w);
        const float2* tl = reinterpret_cast<const float2*>(tables + (size_t)l * T * 2);
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float2 v = __ldg(tl + idx[k]);
          a0 = fmaf(w[k], v.x, a0);
          a1 = fmaf(w[k], v.y, a1);
        }
        x[2 * l] = a0;
        x[2 * l + 1] = a1;
      }
    }
    return;
  }
  for (int l = 0; l < g.n_levels; ++l) {
    uint32_t idx[8];
    float w[8];
    level_corners(g, l, xn, idx, w);
    const float* tl = tables + (size_t)l * T * F;
    for (int f = 0; f < F; ++f) {
      float a = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) a = fmaf(w[k], __ldg(tl + (size_t)idx[k] * F + f), a);
#pragma unroll
      for (int i = 0; i < IN; ++i)
        if (i == l * F + f) x[i] = a;
    }
  }
}

// Hash-table scatter of a feature gradient (ntc.py:278-288).
template <int IN>
__device__ inline void scatter_features(const ss_grid& g, float* __restrict__ g_tables,
                                        const double xn[3], const float (&dx)[IN]) {
  const int F = g.n_features;
  const size_t T = (size_t)1 << g.log2_table;
  if (F == 2) {
#pragma unroll
    for (int l = 0; l < IN / 2; ++l) {
      if (l < g.n_levels) {
        uint32_t idx[8];
        float w[8];
        level_corners(g, l, xn, idx, w);
        float* gl = g_tables + (size_t)l * T * 2;
        const float f0 = dx[2 * l], f1 = dx[2 * l + 1];
#pragma unroll
        for (int k = 0; k < 8; ++k) red_add_v2(gl + 2 * (size_t)idx[k], w[k] * f0, w[k] * f1);
      }
    }
    return;
  }
  for (int l = 0; l < g.n_levels; ++l) {
    uint32_t idx[8];
    float w[8];
    level_corners(g, l, xn, idx, w);
    float* gl = g_tables + (size_t)l * T * F;
    for (int f = 0; f < F; ++f) {
      float fv = 0.f;
#pragma unroll
      for (int k = 0; k < IN; ++k)
        if (k == l * F + f) fv = dx[k];
#pragma unroll
      for (int k = 0; k < 8; ++k) atomicAdd(gl + (size_t)idx[k] * F + f, w[k] * fv);
    }
  }
}

// Features of one point written into a shared-memory row (zero-padded to
// `width`); the level loop is deliberately not unrolled.
__device__ inline void gather_to_row(const ss_grid& g, const float* __restrict__ tables,
                                     const double xn[3], float* row, int width) {
  const int F = g.n_features;
  const size_t T = (size_t)1 << g.log2_table;
#pragma unroll 1
  for (int l = 0; l < g.n_levels; ++l) {
    uint32_t idx[8];
    float w[8];
    level_corners(g, l, xn, idx, w);
    const float* tl = tables + (size_t)l * T * F;
    if (F == 2) {
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(tl) + idx[k]);
        a0 = fmaf(w[k], v.x, a0);
        a1 = fmaf(w[k], v.y, a1);
      }
      row[2 * l] = a0;
      row[2 * l + 1] = a1;
    } else {
      for (int f = 0; f < F; ++f) {
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) a = fmaf(w[k], __ldg(tl + (size_t)idx[k] * F + f), a);
        row[l * F + f] = a;
      }
    }
  }
  for (int k = g.n_levels * F; k < width; ++k) row[k] = 0.f;
}

// dx_j = W0[j,:] . d1 for the features of each level, scattered with vector
// reductions into the table gradient (level loop not unrolled).
template <int IN>
__device__ inline void scatter_rows(const ss_grid& g, const float* __restrict__ w0,
                                    const float (&d1)[HID], const double xn[3],
                                    float* __restrict__ g_tables) {
  const int F = g.n_features;
  const size_t T = (size_t)1 << g.log2_table;
#pragma unroll 1
  for (int l = 0; l < g.n_levels; ++l) {
    uint32_t idx[8];
    float w[8];
    level_corners(g, l, xn, idx, w);
    float* gl = g_tables + (size_t)l * T * F;
    for (int f0 = 0; f0 < F; f0 += 2) {
      float dv[2] = {0.f, 0.f};
      for (int u = 0; u < 2 && f0 + u < F; ++u) {
        const float4* w4 = reinterpret_cast<const float4*>(w0 + (l * F + f0 + u) * HID);
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < HID / 4; ++q) {
          const float4 ww = w4[q];
          s = fmaf(ww.x, d1[4 * q], s);
          s = fmaf(ww.y, d1[4 * q + 1], s);
          s = fmaf(ww.z, d1[4 * q + 2], s);
          s = fmaf(ww.w, d1[4 * q + 3], s);
        }
        dv[u] = s;
      }
      if (F - f0 >= 2 && (F % 2) == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          red_add_v2(gl + (size_t)idx[k] * F + f0, w[k] * dv[0], w[k] * dv[1]);
      } else {
        for (int u = 0; u < 2 && f0 + u < F; ++u)
#pragma unroll
          for (int k = 0; k < 8; ++k) atomicAdd(gl + (size_t)idx[k] * F + f0 + u, w[k] * dv[u]);
      }
    }
  }
}

// ------------------------------------------------------------------ decoder
template <int IN, int NL>
__device__ inline void mlp_forward(const float* __restrict__ sp, const float (&x)[IN],
                                   float (&h1)[HID], float (&h2)[HID], float (&out)[OUTP]) {
  using L = Lay<IN, NL>;
#pragma unroll
  for (int j = 0; j < HID; ++j) h1[j] = sp[L::B0 + j];
#pragma unroll
  for (int i = 0; i < IN; ++i) {
    const float4* w4 = reinterpret_cast<const float4*>(sp + L::W0 + i * HID);
    const float xi = x[i];
#pragma unroll
    for (int q = 0; q < HID / 4; ++q) {
      float4 w = w4[q];
      h1[4 * q] = fmaf(xi, w.x, h1[4 * q]);
      h1[4 * q + 1] = fmaf(xi, w.y, h1[4 * q + 1]);
      h1[4 * q + 2] = fmaf(xi, w.z, h1[4 * q + 2]);
      h1[4 * q + 3] = fmaf(xi, w.w, h1[4 * q + 3]);
    }
  }
#pragma unroll
  for (int j = 0; j < HID; ++j) h1[j] = fmaxf(h1[j], 0.f);
  if (NL == 2) {
#pragma unroll
    for (int j = 0; j < HID; ++j) h2[j] = sp[L::B1 + j];
#pragma unroll
    for (int i = 0; i < HID; ++i) {
      const float4* w4 = reinterpret_cast<const float4*>(sp + L::W1 + i * HID);
      const float hi = h1[i];
#pragma unroll
      for (int q = 0; q < HID / 4; ++q) {
        float4 w = w4[q];
        h2[4 * q] = fmaf(hi, w.x, h2[4 * q]);
        h2[4 * q + 1] = fmaf(hi, w.y, h2[4 * q + 1]);
        h2[4 * q + 2] = fmaf(hi, w.z, h2[4 * q + 2]);
        h2[4 * q + 3] = fmaf(hi, w.w, h2[4 * q + 3]);
      }
    }
#pragma unroll
    for (int j = 0; j < HID; ++j) h2[j] = fmaxf(h2[j], 0.f);
  } else {
#pragma unroll
    for (int j = 0; j < HID; ++j) h2[j] = h1[j];
  }
#pragma unroll
  for (int o = 0; o < OUTP; ++o) out[o] = sp[L::B2 + o];
#pragma unroll
  for (int i = 0; i < HID; ++i) {
    const float4* w4 = reinterpret_cast<const float4*>(sp + L::W2 + i * OUTP);
    float4 a = w4[0], b = w4[1];
    const float hv = h2[i];
    out[0] = fmaf(hv, a.x, out[0]);
    out[1] = fmaf(hv, a.y, out[1]);
    out[2] = fmaf(hv, a.z, out[2]);
    out[3] = fmaf(hv, a.w, out[3]);
    out[4] = fmaf(hv, b.x, out[4]);
    out[5] = fmaf(hv, b.y, out[5]);
    out[6] = fmaf(hv, b.z, out[6]);
    out[7] = fmaf(hv, b.w, out[7]);
  }
}

template <int TOTAL>
__device__ inline void load_params(float* sp, const float* __restrict__ params) {
  for (int i = threadIdx.x; i < TOTAL / 4; i += blockDim.x)
    reinterpret_cast<float4*>(sp)[i] = __ldg(reinterpret_cast<const float4*>(params) + i);
  __syncthreads();
}

// ------------------------------------------------------------------ SH band rotation
// band values / vjp for degree-2/3 bands at direction e
template <int B>
__device__ inline void band_vals(float x, float y, float z, float* v) {
  float b[16];
  sh_basis<float>(B == 5 ? 2 : 3, x, y, z, b);
  const int off = B == 5 ? 4 : 9;
#pragma unroll
  for (int m = 0; m < B; ++m) v[m] = b[off + m];
}
template <int B>
__device__ inline void band_vjp(float x, float y, float z, const float* gv, float g[3]) {
  float gb[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) gb[m] = 0.f;
  const int off = B == 5 ? 4 : 9;
#pragma unroll
  for (int m = 0; m < B; ++m) gb[off + m] = gv[m];
  // degree-1 terms are zero in gb, so the lower bands contribute nothing
  sh_basis_vjp<float>(B == 5 ? 2 : 3, x, y, z, gb, g);
}

// M = S^{-1} E with E[k][b] = Y_b(R^T d_k); sample dirs / S^{-1} in c_shrot.
template <int B>
__device__ inline void band_matrix(const float R[3][3], float M[B][B]) {
  const float(*dirs)[3] = B == 5 ? c_shrot.dirs2 : c_shrot.dirs3;
  const float* sinv = B == 5 ? &c_shrot.binvT2[0][0] : &c_shrot.binvT3[0][0];
  float E[B][B];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    float e[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
      e[i] = R[0][i] * dirs[k][0] + R[1][i] * dirs[k][1] + R[2][i] * dirs[k][2];
    band_vals<B>(e[0], e[1], e[2], E[k]);
  }
#pragma unroll
  for (int a = 0; a < B; ++a)
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < B; ++k) s = fmaf(sinv[a * B + k], E[k][b], s);
      M[a][b] = s;
    }
}

// g_R += d(sum g_M . M)/dR for M = S^{-1} E(R)
template <int B>
__device__ inline void band_matrix_vjp(const float R[3][3], const float gM[B][B],
                                       float gR[3][3]) {
  const float(*dirs)[3] = B == 5 ? c_shrot.dirs2 : c_shrot.dirs3;
  const float* sinv = B == 5 ? &c_shrot.binvT2[0][0] : &c_shrot.binvT3[0][0];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    float e[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
      e[i] = R[0][i] * dirs[k][0] + R[1][i] * dirs[k][1] + R[2][i] * dirs[k][2];
    float gE[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < B; ++a) s = fmaf(sinv[a * B + k], gM[a][b], s);
      gE[b] = s;
    }
    float ge[3] = {0.f, 0.f, 0.f};
    band_vjp<B>(e[0], e[1], e[2], gE, ge);
    // e_i = sum_j R_ji d_j  ->  dL/dR_ji += d_j ge_i
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 3; ++i) gR[j][i] = fmaf(dirs[k][j], ge[i], gR[j][i]);
  }
}

__device__ __constant__ int c_perm[3] = {1, 2, 0};  // (y, z, x) basis order, sh.py:30-32

// sh_out bands 1..deg = M_l(R) sh_in (transform.py:80-84; band 1 = P R P^T)
__device__ inline void rotate_sh_bands(int deg, const float R[3][3], const float* __restrict__ in,
                                 float* __restrict__ out) {
  if (deg >= 1) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float s = 0.f;
#pragma unroll
        for (int b = 0; b < 3; ++b) s = fmaf(R[c_perm[a]][c_perm[b]], in[(1 + b) * 3 + c], s);
        out[(1 + a) * 3 + c] = s;
      }
  }
  if (deg >= 2) {
    float M[5][5];
    band_matrix<5>(R, M);
    for (int a = 0; a < 5; ++a)
      for (int c = 0; c < 3; ++c) {
        float s = 0.f;
#pragma unroll
        for (int b = 0; b < 5; ++b) s = fmaf(M[a][b], in[(4 + b) * 3 + c], s);
        out[(4 + a) * 3 + c] = s;
      }
  }
  if (deg >= 3) {
    float M[7][7];
    band_matrix<7>(R, M);
    for (int a = 0; a < 7; ++a)
      for (int c = 0; c < 3; ++c) {
        float s = 0.f;
#pragma unroll
        for (int b = 0; b < 7; ++b) s = fmaf(M[a][b], in[(9 + b) * 3 + c], s);
        out[(9 + a) * 3 + c] = s;
      }
  }
}

// g_R from g_out (bands >= 1) and the source coefficients (transform.py:120-127)
__device__ inline void rotate_sh_bands_vjp(int deg, const float R[3][3], const float* __restrict__ g,
                                     const float* __restrict__ in, float gR[3][3]) {
  if (deg >= 1) {
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < 3; ++c) s = fmaf(g[(1 + a) * 3 + c], in[(1 + b) * 3 + c], s);
        gR[c_perm[a]][c_perm[b]] += s;  // P^T gM P
      }
  }
  if (deg >= 2) {
    float gM[5][5];
    for (int a = 0; a < 5; ++a)
      for (int b = 0; b < 5; ++b) {
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < 3; ++c) s = fmaf(g[(4 + a) * 3 + c], in[(4 + b) * 3 + c], s);
        gM[a][b] = s;
      }
    band_matrix_vjp<5>(R, gM, gR);
  }
  if (deg >= 3) {
    float gM[7][7];
    for (int a = 0; a < 7; ++a)
      for (int b = 0; b < 7; ++b) {
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < 3; ++c) s = fmaf(g[(9 + a) * 3 + c], in[(9 + b) * 3 + c], s);
        gM[a][b] = s;
      }
    band_matrix_vjp<7>(R, gM, gR);
  }
}

// ------------------------------------------------------------------ kernels
__global__ void encode_kernel(ss_grid g, int64_t n, const float* __restrict__ means,
                              int32_t* __restrict__ corner_idx, float* __restrict__ corner_w,
                              uint32_t* status) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xn[3];
  if (!normalise(g, means + 3 * i, xn) && status) atomicOr(status, SS_FLAG_OUTSIDE);
  for (int l = 0; l < g.n_levels; ++l) {
    uint32_t idx[8];
    float w[8];
    level_corners(g, l, xn, idx, w);
    for (int k = 0; k < 8; ++k) {
      corner_idx[(i * g.n_levels + l) * 8 + k] = (int32_t)idx[k];
      corner_w[(i * g.n_levels + l) * 8 + k] = w[k];
    }
  }
}

__global__ void touched_kernel(ss_grid g, int64_t n, const float* __restrict__ means,
                               const int32_t* __restrict__ rows, uint8_t* __restrict__ mask) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t r = rows ? rows[i] : i;
  double xn[3];
  normalise(g, means + 3 * r, xn);
  const size_t T = (size_t)1 << g.log2_table;
  for (int l = 0; l < g.n_levels; ++l) {
    uint32_t idx[8];
    float w[8];
    level_corners(g, l, xn, idx, w);
#pragma unroll
    for (int k = 0; k < 8; ++k) mask[l * T + idx[k]] = 1;
  }
}

// transform (transform.py:70-84): mu' = mu + d_mu, q' = norm(d_q) (x) q_src,
// SH bands >= 1 rotated by R(norm(d_q)).
__device__ inline void apply_transform(const ss_cloud& src, int64_t gid, const float* o,
                                       int rotate_sh, float* __restrict__ t_means,
                                       float* __restrict__ t_rot, float* __restrict__ t_sh,
                                       uint32_t* status) {
  float nq = sqrtf(o[3] * o[3] + o[4] * o[4] + o[5] * o[5] + o[6] * o[6]);
  if (nq < 1e-12f) {
    if (status) atomicOr(status, SS_FLAG_ZERO_QUAT);
    nq = 1.f;
  }
  const float u[4] = {o[3] / nq, o[4] / nq, o[5] / nq, o[6] / nq};
  const float* m = src.means + 3 * gid;
  t_means[3 * gid + 0] = m[0] + o[0];
  t_means[3 * gid + 1] = m[1] + o[1];
  t_means[3 * gid + 2] = m[2] + o[2];
  float qs[4], qo[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) qs[k] = src.rotations[4 * gid + k];
  quat_mul(u, qs, qo);
#pragma unroll
  for (int k = 0; k < 4; ++k) t_rot[4 * gid + k] = qo[k];
  const int K = src.sh_coeffs;
  const int deg = sh_degree_of(K);
  if (rotate_sh && deg >= 1) {
    float R[3][3];
    quat_to_rot(u[0], u[1], u[2], u[3], R);
    float in[48], outv[48];
    for (int k = 3; k < 3 * K; ++k) in[k] = src.sh[gid * 3 * K + k];
    rotate_sh_bands(deg, R, in, outv);
    for (int k = 3; k < 3 * K; ++k) t_sh[gid * 3 * K + k] = outv[k];
  }
}

// NTC forward (+ transform when `src` given).  One thread per Gaussian.
template <int IN, int NL>
__global__ void __launch_bounds__(128) ntc_forward_kernel(
    ss_grid g, int64_t n, const float* __restrict__ means, const int32_t* __restrict__ rows,
    const float* __restrict__ tables, const float* __restrict__ params, float* __restrict__ out7,
    float* __restrict__ feats, ss_cloud src, int rotate_sh, float* __restrict__ t_means,
    float* __restrict__ t_rot, float* __restrict__ t_sh, uint32_t* status) {
  extern __shared__ __align__(16) float smem[];
  load_params<Lay<IN, NL>::TOTAL>(smem, params);
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t gid = rows ? rows[i] : i;
  double xn[3];
  if (!normalise(g, means + 3 * gid, xn) && status) atomicOr(status, SS_FLAG_OUTSIDE);
  float x[IN], h1[HID], h2[HID], o[OUTP];
  gather_features<IN>(g, tables, xn, x);
  if (feats) {
    const int nf = g.n_levels * g.n_features;
#pragma unroll
    for (int k = 0; k < IN; ++k)
      if (k < nf) feats[i * nf + k] = x[k];
  }
  mlp_forward<IN, NL>(smem, x, h1, h2, o);
  if (out7) {
#pragma unroll
    for (int k = 0; k < 7; ++k) out7[i * 7 + k] = o[k];
  }
  if (!t_means) return;
  apply_transform(src, gid, o, rotate_sh, t_means, t_rot, t_sh, status);
}

// dL/d(out7) from transformed-cloud gradients (transform.py:111-134)
__device__ inline void transform_vjp(const ss_cloud& src, int64_t gid, const float o[OUTP],
                                     int rotate_sh, const float* __restrict__ d_means,
                                     const float* __restrict__ d_rot,
                                     const float* __restrict__ d_sh, float g7[OUTP]) {
  g7[0] = d_means[3 * gid];
  g7[1] = d_means[3 * gid + 1];
  g7[2] = d_means[3 * gid + 2];
  g7[7] = 0.f;
  float q[4], gr[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) q[k] = src.rotations[4 * gid + k], gr[k] = d_rot[4 * gid + k];
  // g_u = A(q_src)^T g_rot, A rows: [w,-x,-y,-z],[x,w,z,-y],[y,-z,w,x],[z,y,-x,w]
  const float w = q[0], x = q[1], y = q[2], z = q[3];
  float gu[4];
  gu[0] = w * gr[0] + x * gr[1] + y * gr[2] + z * gr[3];
  gu[1] = -x * gr[0] + w * gr[1] - z * gr[2] + y * gr[3];
  gu[2] = -y * gr[0] + z * gr[1] + w * gr[2] - x * gr[3];
  gu[3] = -z * gr[0] - y * gr[1] + x * gr[2] + w * gr[3];
  float nq = sqrtf(o[3] * o[3] + o[4] * o[4] + o[5] * o[5] + o[6] * o[6]);
  nq = nq < 1e-12f ? 1.f : nq;
  const float u[4] = {o[3] / nq, o[4] / nq, o[5] / nq, o[6] / nq};
  const int K = src.sh_coeffs;
  const int deg = sh_degree_of(K);
  if (rotate_sh && deg >= 1) {
    float R[3][3], gR[3][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
    quat_to_rot(u[0], u[1], u[2], u[3], R);
    float in[48], gs[48];
    for (int k = 3; k < 3 * K; ++k) in[k] = src.sh[gid * 3 * K + k], gs[k] = d_sh[gid * 3 * K + k];
    rotate_sh_bands_vjp(deg, R, gs, in, gR);
    float gq[4];
    quat_to_rot_vjp(u[0], u[1], u[2], u[3], gR, gq);
#pragma unroll
    for (int k = 0; k < 4; ++k) gu[k] += gq[k];
  }
  // (I - u u^T)/|q| (gaussians.py:109-117)
  const float dot = u[0] * gu[0] + u[1] * gu[1] + u[2] * gu[2] + u[3] * gu[3];
#pragma unroll
  for (int k = 0; k < 4; ++k) g7[3 + k] = (gu[k] - u[k] * dot) / nq;
}

__global__ void transform_apply_kernel(ss_cloud src, int64_t n, const int32_t* __restrict__ rows,
                                       const float* __restrict__ out7, int rotate_sh,
                                       float* __restrict__ tm, float* __restrict__ tr,
                                       float* __restrict__ ts, uint32_t* status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float o[OUTP];
#pragma unroll
  for (int k = 0; k < 7; ++k) o[k] = out7[i * 7 + k];
  o[7] = 0.f;
  apply_transform(src, rows ? rows[i] : i, o, rotate_sh, tm, tr, ts, status);
}

__global__ void transform_vjp_kernel(ss_cloud src, int64_t n, const int32_t* __restrict__ rows,
                                     const float* __restrict__ out7, int rotate_sh,
                                     const float* __restrict__ dm, const float* __restrict__ dr,
                                     const float* __restrict__ ds, float* __restrict__ g_out7) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float o[OUTP], g7[OUTP];
#pragma unroll
  for (int k = 0; k < 7; ++k) o[k] = out7[i * 7 + k];
  o[7] = 0.f;
  transform_vjp(src, rows ? rows[i] : i, o, rotate_sh, dm, dr, ds, g7);
#pragma unroll
  for (int k = 0; k < 7; ++k) g_out7[i * 7 + k] = g7[k];
}

// Backward: one thread per Gaussian per chunk; the decoder's weight gradient
// is a CTA-level GEMM over the chunk (register-blocked 4x4 tiles), the
// feature gradient is scattered into the tables with vector reductions.
template <int IN, int NL>
struct BwdSmem {
  static constexpr int SX = IN + 4, SH = HID + 4, SG = OUTP + 4;
  static constexpr int oX = Lay<IN, NL>::TOTAL;  // params first
  static constexpr int oH1 = oX + kChunk * SX;
  static constexpr int oH2 = oH1 + kChunk * SH;
  static constexpr int oD1 = oH2 + (NL == 2 ? kChunk * SH : 0);
  static constexpr int oD2 = oD1 + kChunk * SH;
  static constexpr int oG = oD2 + (NL == 2 ? kChunk * SH : 0);
  static constexpr int FLOATS = oG + kChunk * SG;
  // 4x4 weight-gradient tasks
  static constexpr int T0 = (IN / 4) * (HID / 4);
  static constexpr int T1 = NL == 2 ? (HID / 4) * (HID / 4) : 0;
  static constexpr int T2 = (HID / 4) * (OUTP / 4);
  static constexpr int TB = HID / 4 + (NL == 2 ? HID / 4 : 0) + OUTP / 4;
  static constexpr int TASKS = T0 + T1 + T2 + TB;
  static constexpr int PER_THREAD = (TASKS + kChunk - 1) / kChunk;
};

template <int IN, int NL>
struct TaskDesc {
  int a_off, a_stride, d_off, d_stride, dst, dst_cols;  // a_off < 0: ones (bias)
};

template <int IN, int NL>
__device__ inline TaskDesc<IN, NL> decode_task(int t) {
  using S = BwdSmem<IN, NL>;
  using L = Lay<IN, NL>;
  TaskDesc<IN, NL> d;
  if (t < S::T0) {
    int ib = t / (HID / 4), jb = t % (HID / 4);
    d = {S::oX + 4 * ib, S::SX, S::oD1 + 4 * jb, S::SH, L::W0 + 4 * ib * HID + 4 * jb, HID};
    return d;
  }
  t -= S::T0;
  if (t < S::T1) {
    int ib = t / (HID / 4), jb = t % (HID / 4);
    d = {S::oH1 + 4 * ib, S::SH, S::oD2 + 4 * jb, S::SH, L::W1 + 4 * ib * HID + 4 * jb, HID};
    return d;
  }
  t -= S::T1;
  const int oHlast = NL == 2 ? S::oH2 : S::oH1;
  if (t < S::T2) {
    int ib = t / (OUTP / 4), jb = t % (OUTP / 4);
    d = {oHlast + 4 * ib, S::SH, S::oG + 4 * jb, S::SG, L::W2 + 4 * ib * OUTP + 4 * jb, OUTP};
    return d;
  }
  t -= S::T2;
  if (t < HID / 4) {
    d = {-1, 0, S::oD1 + 4 * t, S::SH, L::B0 + 4 * t, 0};
    return d;
  }
  t -= HID / 4;
  if (NL == 2 && t < HID / 4) {
    d = {-1, 0, S::oD2 + 4 * t, S::SH, L::B1 + 4 * t, 0};
    return d;
  }
  if (NL == 2) t -= HID / 4;
  d = {-1, 0, S::oG + 4 * t, S::SG, L::B2 + 4 * t, 0};
  return d;
}

template <int IN, int NL>
__global__ void __launch_bounds__(kChunk, 1) ntc_backward_kernel(
    ss_grid g, int64_t n, const float* __restrict__ means, const int32_t* __restrict__ rows,
    const float* __restrict__ tables, const float* __restrict__ params,
    const float* __restrict__ g_out7,  // (n,7) upstream dL/d[d_mu | d_q]
    float* __restrict__ g_tables, float* __restrict__ g_params) {
  using S = BwdSmem<IN, NL>;
  using L = Lay<IN, NL>;
  extern __shared__ __align__(16) float smem[];
  load_params<L::TOTAL>(smem, params);
  const int tid = threadIdx.x;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t i = c * kChunk + tid;
    float* sX = smem + S::oX + tid * S::SX;
    float* sH1 = smem + S::oH1 + tid * S::SH;
    float* sH2 = smem + S::oH2 + tid * S::SH;
    float* sD1 = smem + S::oD1 + tid * S::SH;
    float* sD2 = smem + S::oD2 + tid * S::SH;
    float* sG = smem + S::oG + tid * S::SG;
    if (i < n) {
      const int64_t gid = rows ? rows[i] : i;
      double xn[3];
      normalise(g, means + 3 * gid, xn);
      // recompute the hidden activations, staging each layer through this
      // thread's shared-memory rows so at most two 64-vectors live in registers
      uint64_t mask1 = 0, mask2 = 0;
      gather_to_row(g, tables, xn, sX, IN);  // level loop not unrolled (register budget)
      {
        float h[HID];
#pragma unroll
        for (int j = 0; j < HID; ++j) h[j] = smem[L::B0 + j];
#pragma unroll 4
        for (int i2 = 0; i2 < IN; ++i2) {
          const float xi = sX[i2];
          const float4* w4 = reinterpret_cast<const float4*>(smem + L::W0 + i2 * HID);
#pragma unroll
          for (int q = 0; q < HID / 4; ++q) {
            const float4 w = w4[q];
            h[4 * q] = fmaf(xi, w.x, h[4 * q]);
            h[4 * q + 1] = fmaf(xi, w.y, h[4 * q + 1]);
            h[4 * q + 2] = fmaf(xi, w.z, h[4 * q + 2]);
            h[4 * q + 3] = fmaf(xi, w.w, h[4 * q + 3]);
          }
        }
#pragma unroll
        for (int k = 0; k < HID; ++k) {
          h[k] = fmaxf(h[k], 0.f);
          mask1 |= (uint64_t)(h[k] > 0.f) << k;
        }
#pragma unroll
        for (int k = 0; k < HID; k += 4)
          *reinterpret_cast<float4*>(sH1 + k) = make_float4(h[k], h[k + 1], h[k + 2], h[k + 3]);
      }
      if (NL == 2) {
        float h[HID];
#pragma unroll
        for (int j = 0; j < HID; ++j) h[j] = smem[L::B1 + j];
#pragma unroll 4
        for (int i2 = 0; i2 < HID; ++i2) {
          const float hi = sH1[i2];
          const float4* w4 = reinterpret_cast<const float4*>(smem + L::W1 + i2 * HID);
#pragma unroll
          for (int q = 0; q < HID / 4; ++q) {
            const float4 w = w4[q];
            h[4 * q] = fmaf(hi, w.x, h[4 * q]);
            h[4 * q + 1] = fmaf(hi, w.y, h[4 * q + 1]);
            h[4 * q + 2] = fmaf(hi, w.z, h[4 * q + 2]);
            h[4 * q + 3] = fmaf(hi, w.w, h[4 * q + 3]);
          }
        }
#pragma unroll
        for (int k = 0; k < HID; ++k) {
          h[k] = fmaxf(h[k], 0.f);
          mask2 |= (uint64_t)(h[k] > 0.f) << k;
        }
#pragma unroll
        for (int k = 0; k < HID; k += 4)
          *reinterpret_cast<float4*>(sH2 + k) = make_float4(h[k], h[k + 1], h[k + 2], h[k + 3]);
      } else {
        mask2 = mask1;
      }
      float g7[OUTP];
#pragma unroll
      for (int k = 0; k < 7; ++k) g7[k] = g_out7[i * 7 + k];
      g7[7] = 0.f;
      *reinterpret_cast<float4*>(sG) = make_float4(g7[0], g7[1], g7[2], g7[3]);
      *reinterpret_cast<float4*>(sG + 4) = make_float4(g7[4], g7[5], g7[6], g7[7]);
      // delta through the output layer: dl = (W2 g7) * (h_last > 0)
      float d1[HID];
      {
        float* sDl = NL == 2 ? sD2 : sD1;
#pragma unroll
        for (int j = 0; j < HID; ++j) {
          const float4* w4 = reinterpret_cast<const float4*>(smem + L::W2 + j * OUTP);
          const float4 a = w4[0], b = w4[1];
          const float sv = a.x * g7[0] + a.y * g7[1] + a.z * g7[2] + a.w * g7[3] + b.x * g7[4] +
                           b.y * g7[5] + b.z * g7[6];
          d1[j] = ((mask2 >> j) & 1) ? sv : 0.f;
        }
#pragma unroll
        for (int k = 0; k < HID; k += 4)
          *reinterpret_cast<float4*>(sDl + k) = make_float4(d1[k], d1[k + 1], d1[k + 2], d1[k + 3]);
        if (NL == 2) {
          // d1 = (W1 dl) * (h1 > 0), dl read back from its shared row
#pragma unroll
          for (int k = 0; k < HID; ++k) d1[k] = 0.f;
#pragma unroll 4
          for (int q = 0; q < HID; ++q) {
            const float dq = sD2[q];
#pragma unroll
            for (int r = 0; r < HID; ++r) d1[r] = fmaf(smem[L::W1 + r * HID + q], dq, d1[r]);
          }
#pragma unroll
          for (int k = 0; k < HID; ++k) d1[k] = ((mask1 >> k) & 1) ? d1[k] : 0.f;
#pragma unroll
          for (int k = 0; k < HID; k += 4)
            *reinterpret_cast<float4*>(sD1 + k) =
                make_float4(d1[k], d1[k + 1], d1[k + 2], d1[k + 3]);
        }
      }
      // feature gradient dx = W0 d1, computed per level and scattered into the
      // tables (ntc.py:278-288)
      scatter_rows<IN>(g, smem + L::W0, d1, xn, g_tables);
    } else {
      for (int k = 0; k < S::SX; ++k) sX[k] = 0.f;
      for (int k = 0; k < S::SH; ++k) {
        sH1[k] = 0.f;
        sD1[k] = 0.f;
        if (NL == 2) sH2[k] = 0.f, sD2[k] = 0.f;
      }
      for (int k = 0; k < S::SG; ++k) sG[k] = 0.f;
    }
    __syncthreads();
    // ---- CTA-level weight-gradient GEMM over the chunk (ntc.py:271-273),
    // register-blocked 4x4 tiles, flushed with vector reductions
#pragma unroll 1
    for (int s = 0; s < S::PER_THREAD; ++s) {
      const int t = tid + s * kChunk;
      if (t >= S::TASKS) break;
      TaskDesc<IN, NL> d = decode_task<IN, NL>(t);
      const float* pd = smem + d.d_off;
      float acc[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = 0.f;
      if (d.a_off < 0) {
#pragma unroll 4
        for (int r = 0; r < kChunk; ++r) {
          float4 v = *reinterpret_cast<const float4*>(pd + r * d.d_stride);
          acc[0] += v.x;
          acc[1] += v.y;
          acc[2] += v.z;
          acc[3] += v.w;
        }
        red_add_v4(g_params + d.dst, acc[0], acc[1], acc[2], acc[3]);
      } else {
        const float* pa = smem + d.a_off;
#pragma unroll 4
        for (int r = 0; r < kChunk; ++r) {
          float4 a = *reinterpret_cast<const float4*>(pa + r * d.a_stride);
          float4 v = *reinterpret_cast<const float4*>(pd + r * d.d_stride);
          const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            acc[4 * p + 0] = fmaf(av[p], v.x, acc[4 * p + 0]);
            acc[4 * p + 1] = fmaf(av[p], v.y, acc[4 * p + 1]);
            acc[4 * p + 2] = fmaf(av[p], v.z, acc[4 * p + 2]);
            acc[4 * p + 3] = fmaf(av[p], v.w, acc[4 * p + 3]);
          }
        }
#pragma unroll
        for (int p = 0; p < 4; ++p)
          red_add_v4(g_params + d.dst + p * d.dst_cols, acc[4 * p], acc[4 * p + 1],
                     acc[4 * p + 2], acc[4 * p + 3]);
      }
    }
    __syncthreads();
  }
}

// lazy Adam over tables (row mask) + dense MLP (optim.py:33-66)
__global__ void adam_kernel(int64_t n_table, float* __restrict__ tables,
                            float* __restrict__ g_tables, double* __restrict__ m_t,
                            double* __restrict__ v_t, const uint8_t* __restrict__ row_mask,
                            int row_width, int64_t n_params, float* __restrict__ params,
                            float* __restrict__ g_params, double* __restrict__ m_p,
                            double* __restrict__ v_p, const int32_t* __restrict__ step_dev,
                            double lr, double b1, double b2, double eps, int zero_grads) {
  const int step = *step_dev + 1;
  const double bc1 = 1.0 - pow(b1, (double)step);
  const double bc2 = 1.0 - pow(b2, (double)step);
  const int64_t total = n_table + n_params;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float *p, *gp;
    double *m, *v;
    int64_t j;
    if (i < n_table) {
      j = i;
      p = tables, gp = g_tables, m = m_t, v = v_t;
      if (row_mask && !row_mask[j / row_width]) {
        if (zero_grads) gp[j] = 0.f;
        continue;
      }
    } else {
      j = i - n_table;
      p = params, gp = g_params, m = m_p, v = v_p;
    }
    const double g = gp[j];
    const double mm = b1 * m[j] + (1.0 - b1) * g;
    const double vv = b2 * v[j] + (1.0 - b2) * (g * g);
    m[j] = mm;
    v[j] = vv;
    p[j] = (float)((double)p[j] - lr * (mm / bc1) / (sqrt(vv / bc2) + eps));
    if (zero_grads) gp[j] = 0.f;
  }
}

__global__ void increment_kernel(int32_t* step) { *step += 1; }

// ------------------------------------------------------------------ dispatch
template <class Fn>
int dispatch_mlp(const ss_mlp* mlp, Fn&& fn) {
  ss_mlp_layout L;
  if (ss_mlp_get_layout(mlp, &L) != SS_OK) return SS_ERR_DATA;
  if (L.in_pad == 16) return L.n_hidden == 2 ? fn.template run<16, 2>() : fn.template run<16, 1>();
  if (L.in_pad == 32) return L.n_hidden == 2 ? fn.template run<32, 2>() : fn.template run<32, 1>();
  return L.n_hidden == 2 ? fn.template run<64, 2>() : fn.template run<64, 1>();
}

static int check_grid(const ss_grid* g, const ss_mlp* mlp) {
  if (!g || g->n_levels < 1 || g->n_levels > SS_MAX_LEVELS || g->n_features < 1 ||
      g->log2_table < 1 || g->log2_table > 30) {
    set_error("invalid hash-grid configuration");
    return SS_ERR_DATA;
  }
  if (mlp && g->n_levels * g->n_features != mlp->in_dim) {
    set_error("decoder in_dim must equal n_levels * n_features");
    return SS_ERR_DATA;
  }
  return SS_OK;
}

struct FwdLaunch {
  const ss_grid* g;
  int64_t n;
  const float* means;
  const int32_t* rows;
  const float *tables, *params;
  float *out7, *feats;
  ss_cloud src;
  int rotate_sh;
  float *tm, *tr, *ts;
  uint32_t* status;
  cudaStream_t st;
  template <int IN, int NL>
  int run() {
    if (n == 0) return SS_OK;
    const size_t smem = Lay<IN, NL>::TOTAL * sizeof(float);
    auto k = ntc_forward_kernel<IN, NL>;
    SS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    prof_begin(PH_NTC_FWD, st);
    k<<<(unsigned)cdiv(n, 128), 128, smem, st>>>(*g, n, means, rows, tables, params, out7, feats,
                                                  src, rotate_sh, tm, tr, ts, status);
    SS_CHECK_LAUNCH("ntc_forward_kernel");
    prof_end(PH_NTC_FWD, st);
    return SS_OK;
  }
};

struct BwdLaunch {
  const ss_grid* g;
  int64_t n;
  const float* means;
  const int32_t* rows;
  const float *tables, *params, *g_out7;
  float *g_tables, *g_params;
  cudaStream_t st;
  template <int IN, int NL>
  int run() {
    if (n == 0) return SS_OK;
    const size_t smem = BwdSmem<IN, NL>::FLOATS * sizeof(float);
    auto k = ntc_backward_kernel<IN, NL>;
    SS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t chunks = cdiv(n, kChunk);
    const unsigned grid = (unsigned)std::min<int64_t>(chunks, sms);
    prof_begin(PH_NTC_BWD, st);
    k<<<grid, kChunk, smem, st>>>(*g, n, means, rows, tables, params, g_out7, g_tables,
                                  g_params);
    SS_CHECK_LAUNCH("ntc_backward_kernel");
    prof_end(PH_NTC_BWD, st);
    return SS_OK;
  }
};

}  // namespace ss

using namespace ss;

extern "C" {

int ss_ntc_encode(const ss_grid* grid, int64_t n, const float* means, int32_t* corner_idx,
                  float* corner_w, uint32_t* status, void* stream) {
  SS_TRY(check_grid(grid, nullptr));
  if (n == 0) return SS_OK;
  encode_kernel<<<(unsigned)cdiv(n, 128), 128, 0, as_stream(stream)>>>(*grid, n, means,
                                                                        corner_idx, corner_w,
                                                                        status);
  SS_CHECK_LAUNCH("encode_kernel");
  return SS_OK;
}

int ss_ntc_touched(const ss_grid* grid, int64_t n, const float* means, const int32_t* rows,
                   uint8_t* mask, void* stream) {
  SS_TRY(check_grid(grid, nullptr));
  if (n == 0) return SS_OK;
  touched_kernel<<<(unsigned)cdiv(n, 128), 128, 0, as_stream(stream)>>>(*grid, n, means, rows,
                                                                         mask);
  SS_CHECK_LAUNCH("touched_kernel");
  return SS_OK;
}

int ss_ntc_forward(const ss_grid* grid, const ss_mlp* mlp, int64_t n, const float* means,
                   const int32_t* rows, const float* tables, const float* params, float* out7,
                   float* feats, void* stream) {
  SS_TRY(check_grid(grid, mlp));
  FwdLaunch L{grid, n, means, rows, tables, params, out7, feats, ss_cloud{}, 0, nullptr,
              nullptr, nullptr, nullptr, as_stream(stream)};
  return dispatch_mlp(mlp, L);
}

size_t ss_ntc_backward_bytes(const ss_mlp* mlp) {
  (void)mlp;
  return 0;
}

int ss_ntc_backward(const ss_grid* grid, const ss_mlp* mlp, int64_t n, const float* means,
                    const int32_t* rows, const float* tables, const float* params,
                    const float* g_out7, float* g_tables, float* g_params, void* scratch,
                    void* stream) {
  (void)scratch;
  SS_TRY(check_grid(grid, mlp));
  if (!g_out7) {
    set_error("ss_ntc_backward: g_out7 required");
    return SS_ERR_DATA;
  }
  BwdLaunch L{grid, n, means, rows, tables, params, g_out7, g_tables, g_params,
              as_stream(stream)};
  return dispatch_mlp(mlp, L);
}

int ss_apply_ntc(const ss_grid* grid, const ss_mlp* mlp, const ss_cloud* src, int64_t n_in,
                 const int32_t* rows, const float* tables, const float* params,
                 int32_t rotate_sh, float* out_means, float* out_rotations, float* out_sh,
                 float* out7, uint32_t* status, void* stream) {
  SS_TRY(check_grid(grid, mlp));
  if (!src || !out_means || !out_rotations || (rotate_sh && src->sh_coeffs > 1 && !out_sh)) {
    set_error("ss_apply_ntc: missing cloud buffers");
    return SS_ERR_DATA;
  }
  if (src->sh_coeffs > 16) {
    set_error("SH degree > 3 unsupported");
    return SS_ERR_DATA;
  }
  SS_TRY(ensure_shrot_const());
  FwdLaunch L{grid, n_in, src->means, rows, tables, params, out7, nullptr, *src, rotate_sh,
              out_means, out_rotations, out_sh, status, as_stream(stream)};
  return dispatch_mlp(mlp, L);
}

size_t ss_apply_ntc_backward_bytes(int64_t n_in) {
  return align_up((size_t)(n_in > 0 ? n_in : 1) * 7 * sizeof(float)) * 2;
}

int ss_apply_ntc_backward(const ss_grid* grid, const ss_mlp* mlp, const ss_cloud* src,
                          int64_t n_in, const int32_t* rows, const float* tables,
                          const float* params, int32_t rotate_sh, const float* d_means,
                          const float* d_rotations, const float* d_sh, float* g_tables,
                          float* g_params, void* scratch, void* stream) {
  SS_TRY(check_grid(grid, mlp));
  if (!src || !d_means || !d_rotations || (rotate_sh && src->sh_coeffs > 1 && !d_sh) ||
      !scratch) {
    set_error("ss_apply_ntc_backward: missing gradient or scratch buffers");
    return SS_ERR_DATA;
  }
  if (n_in == 0) return SS_OK;
  // the decoder output is recomputed (K2f), then the transform VJP (K3b) and the
  // decoder/table backward (K2b/K1b) run as separate kernels
  float* out7 = static_cast<float*>(scratch);
  float* g7 = reinterpret_cast<float*>(static_cast<char*>(scratch) +
                                       ss_apply_ntc_backward_bytes(n_in) / 2);
  SS_TRY(ss_ntc_forward(grid, mlp, n_in, src->means, rows, tables, params, out7, nullptr,
                        stream));
  return ss_apply_ntc_backward_stored(grid, mlp, src, n_in, rows, tables, params, rotate_sh,
                                      out7, d_means, d_rotations, d_sh, g7, g_tables, g_params,
                                      stream);
}

int ss_apply_ntc_backward_stored(const ss_grid* grid, const ss_mlp* mlp, const ss_cloud* src,
                                 int64_t n_in, const int32_t* rows, const float* tables,
                                 const float* params, int32_t rotate_sh, const float* out7,
                                 const float* d_means, const float* d_rotations,
                                 const float* d_sh, float* g_out7, float* g_tables,
                                 float* g_params, void* stream) {
  SS_TRY(ss_transform_vjp(src, n_in, rows, out7, rotate_sh, d_means, d_rotations, d_sh, g_out7,
                          stream));
  return ss_ntc_backward(grid, mlp, n_in, src->means, rows, tables, params, g_out7, g_tables,
                         g_params, nullptr, stream);
}

int ss_transform_apply(const ss_cloud* src, int64_t n_in, const int32_t* rows, const float* out7,
                       int32_t rotate_sh, float* out_means, float* out_rotations, float* out_sh,
                       uint32_t* status, void* stream) {
  if (!src || src->sh_coeffs < 1 || src->sh_coeffs > 16) {
    set_error("ss_transform_apply: bad cloud");
    return SS_ERR_DATA;
  }
  if (n_in == 0) return SS_OK;
  SS_TRY(ensure_shrot_const());
  transform_apply_kernel<<<(unsigned)cdiv(n_in, 128), 128, 0, as_stream(stream)>>>(
      *src, n_in, rows, out7, rotate_sh, out_means, out_rotations, out_sh, status);
  SS_CHECK_LAUNCH("transform_apply_kernel");
  return SS_OK;
}

int ss_transform_vjp(const ss_cloud* src, int64_t n_in, const int32_t* rows, const float* out7,
                     int32_t rotate_sh, const float* d_means, const float* d_rotations,
                     const float* d_sh, float* g_out7, void* stream) {
  if (!src || src->sh_coeffs < 1 || src->sh_coeffs > 16) {
    set_error("ss_transform_vjp: bad cloud");
    return SS_ERR_DATA;
  }
  if (n_in == 0) return SS_OK;
  SS_TRY(ensure_shrot_const());
  transform_vjp_kernel<<<(unsigned)cdiv(n_in, 128), 128, 0, as_stream(stream)>>>(
      *src, n_in, rows, out7, rotate_sh, d_means, d_rotations, d_sh, g_out7);
  SS_CHECK_LAUNCH("transform_vjp_kernel");
  return SS_OK;
}

int ss_adam_step(int64_t n_table, float* tables, float* g_tables, double* m_tables,
                 double* v_tables, const uint8_t* row_mask, int32_t row_width,
                 int64_t n_params, float* params, float* g_params, double* m_params,
                 double* v_params, int32_t* step_dev, double lr, double beta1, double beta2,
                 double eps, int32_t zero_grads, void* stream) {
  if (!step_dev || row_width < 1) {
    set_error("ss_adam_step: bad arguments");
    return SS_ERR_DATA;
  }
  cudaStream_t st = as_stream(stream);
  const int64_t total = n_table + n_params;
  if (total > 0) {
    const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(total, 256), 148 * 8);
    prof_begin(PH_ADAM, st);
    adam_kernel<<<blocks, 256, 0, st>>>(n_table, tables, g_tables, m_tables, v_tables, row_mask,
                                        row_width, n_params, params, g_params, m_params,
                                        v_params, step_dev, lr, beta1, beta2, eps, zero_grads);
    SS_CHECK_LAUNCH("adam_kernel");
    prof_end(PH_ADAM, st);
  }
  increment_kernel<<<1, 1, 0, st>>>(step_dev);
  SS_CHECK_LAUNCH("increment_kernel");
  return SS_OK;
}

}  // extern "C"
