// Neural Transformation Cache on sm_100a: hash-grid encode/gather (K1f),
// decoder (K2f), transform (K3f), transform VJP (K3b), decoder backward (K2b),
// hash-table scatter (K1b) and the lazy Adam step (KA).  Features X and their
// gradient dX live in HBM between the kernels so each stage runs at its own
// occupancy (thread per Gaussian x level for the gather/scatter).
//
// Reference: ntc.py:161-293, transform.py:53-135, optim.py:33-66
// (/root/reference/pkg/src/splatstream/).
#include <mutex>

#include "common.cuh"
#include "hashgrid.cuh"

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
// (y, z, x) basis order of band 1, sh.py:30-32; constexpr so the unrolled
// loops index R / g_R with constants (a __constant__ table made every access
// a select chain over the nine registers)
__device__ __forceinline__ constexpr int c_perm(int a) { return a == 0 ? 1 : (a == 1 ? 2 : 0); }

// One colour channel of bands l >= 2 (4 lanes per Gaussian, see
// transform_kernel): out = S^{-1} y with y_k = f(R^T d_k), f the band-l SH
// function whose coefficients are `in` -- the same M = S^{-1} E(R) as
// band_matrix without forming M.
template <int B>
__device__ inline void rotate_band_channel(const float R[3][3], const float* in, float* out) {
  const float(*dirs)[3] = B == 5 ? c_shrot.dirs2 : c_shrot.dirs3;
  const float* sinv = B == 5 ? &c_shrot.binvT2[0][0] : &c_shrot.binvT3[0][0];
  float y[B];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    float e[3], v[B];
#pragma unroll
    for (int i = 0; i < 3; ++i)
      e[i] = R[0][i] * dirs[k][0] + R[1][i] * dirs[k][1] + R[2][i] * dirs[k][2];
    band_vals<B>(e[0], e[1], e[2], v);
    float sum = 0.f;
#pragma unroll
    for (int b = 0; b < B; ++b) sum = fmaf(v[b], in[b], sum);
    y[k] = sum;
  }
#pragma unroll
  for (int a = 0; a < B; ++a) {
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < B; ++k) sum = fmaf(sinv[a * B + k], y[k], sum);
    out[a] = sum;
  }
}

// Gradient at e of the band-l function f(e) = sum_b c_b Y_{l,b}(e): the band-l
// terms of sh_basis_vjp (the same polynomial derivatives), without the lower
// bands' zero-weighted work.
__device__ __forceinline__ void band_grad(const float* c, float x, float y, float z, float g[3],
                                          int B) {
  if (B == 5) {
    const float a = kShC2a, b = kShC2b, cc = kShC2c;
    g[0] = a * y * c[0] + a * z * c[3] - 2.f * b * x * c[2] + 2.f * cc * x * c[4];
    g[1] = a * x * c[0] + a * z * c[1] - 2.f * b * y * c[2] - 2.f * cc * y * c[4];
    g[2] = a * y * c[1] + 4.f * b * z * c[2] + a * x * c[3];
  } else {
    const float c3 = kShC3a, c2 = kShC3b, c1 = kShC3c, c0 = kShC3d, ch = kShC3e;
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
    g[0] = 6.f * c3 * xy * c[0] + c2 * yz * c[1] - 2.f * c1 * xy * c[2] - 6.f * c0 * xz * c[3] +
           c1 * (4.f * zz - 3.f * xx - yy) * c[4] + 2.f * ch * xz * c[5] +
           c3 * (3.f * xx - 3.f * yy) * c[6];
    g[1] = c3 * (3.f * xx - 3.f * yy) * c[0] + c2 * xz * c[1] +
           c1 * (4.f * zz - xx - 3.f * yy) * c[2] - 6.f * c0 * yz * c[3] - 2.f * c1 * xy * c[4] -
           2.f * ch * yz * c[5] - 6.f * c3 * xy * c[6];
    g[2] = c2 * xy * c[1] + 8.f * c1 * yz * c[2] + c0 * (6.f * zz - 3.f * xx - 3.f * yy) * c[3] +
           8.f * c1 * xz * c[4] + ch * (xx - yy) * c[5];
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

// K1f: interpolated features (ntc.py:176-216), one thread per inside row:
// the fp64 normalisation is done once and the L levels are walked in turn
// (8 float2 gathers each from the L2-resident tables).  Stage 1 orders the
// inside rows along a Morton curve, so neighbouring threads gather
// neighbouring cells.  X is (n, xs) row-major, padding columns zeroed.
__global__ void __launch_bounds__(256) gather_kernel(ss_grid g, int64_t n,
                                                     const float* __restrict__ means,
                                                     const int32_t* __restrict__ rows,
                                                     const float* __restrict__ tables,
                                                     float* __restrict__ X, int xs,
                                                     uint32_t* status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int L = g.n_levels, F = g.n_features;
  const int64_t gid = rows ? rows[i] : i;
  double xn[3];
  if (!normalise(g, means + 3 * gid, xn) && status) atomicOr(status, SS_FLAG_OUTSIDE);
  const size_t T = (size_t)1 << g.log2_table;
  float* xr = X + i * xs;
  if (F == 2 && (L & 1) == 0) {
    // two levels per step: 16 corner gathers in flight, one 16-byte store
    for (int l = 0; l < L; l += 2) {
      uint32_t ia[8], ib[8];
      float wa[8], wb[8];
      level_corners(g, l, xn, ia, wa);
      level_corners(g, l + 1, xn, ib, wb);
      const float2* ta = reinterpret_cast<const float2*>(tables + (size_t)l * T * 2);
      const float2* tb = reinterpret_cast<const float2*>(tables + (size_t)(l + 1) * T * 2);
      float2 va[8], vb[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        va[k] = __ldg(ta + ia[k]);
        vb[k] = __ldg(tb + ib[k]);
      }
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        acc.x = fmaf(wa[k], va[k].x, acc.x);
        acc.y = fmaf(wa[k], va[k].y, acc.y);
        acc.z = fmaf(wb[k], vb[k].x, acc.z);
        acc.w = fmaf(wb[k], vb[k].y, acc.w);
      }
      *reinterpret_cast<float4*>(xr + 2 * l) = acc;
    }
    for (int k = L * F; k < xs; ++k) xr[k] = 0.f;
    return;
  }
  for (int l = 0; l < L; ++l) {
    uint32_t idx[8];
    float w[8];
    level_corners(g, l, xn, idx, w);
    const float* tl = tables + (size_t)l * T * F;
    if (F == 2) {
      float2 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldg(reinterpret_cast<const float2*>(tl) + idx[k]);
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        a0 = fmaf(w[k], v[k].x, a0);
        a1 = fmaf(w[k], v[k].y, a1);
      }
      *reinterpret_cast<float2*>(xr + 2 * l) = make_float2(a0, a1);
    } else {
      for (int f = 0; f < F; ++f) {
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) a = fmaf(w[k], __ldg(tl + (size_t)idx[k] * F + f), a);
        xr[l * F + f] = a;
      }
    }
  }
  for (int k = L * F; k < xs; ++k) xr[k] = 0.f;
}

// K1b: table scatter of the feature gradient (ntc.py:278-288), one thread per
// inside row walking the levels, warp-aggregated vector reductions into the
// L2-resident gradient tables: lanes whose corner equals their left
// neighbour's form a run (rows are Morton-ordered, so equal corners are
// adjacent at the coarse levels), a segmented suffix sum gives each run head
// the run total and only heads issue red.global.add.v2.f32.  Non-adjacent
// duplicates are separate runs (still correct).
__global__ void __launch_bounds__(256) scatter_kernel(ss_grid g, int64_t n,
                                                      const float* __restrict__ means,
                                                      const int32_t* __restrict__ rows,
                                                      const float* __restrict__ dX, int xs,
                                                      float* __restrict__ g_tables) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int L = g.n_levels, F = g.n_features;
  const float* dr = dX + (i < n ? i : 0) * xs;
  // rows with an all-zero feature gradient (Gaussians no pixel saw in this
  // view) add nothing (np.add.at of zeros): skip them, whole warps at a time
  bool ok = i < n;
  if (ok) {
    bool nz = false;
    for (int k = 0; k < L * F; k += 4) {
      const float4 v = *reinterpret_cast<const float4*>(dr + k);
      nz |= (v.x != 0.f) | (v.y != 0.f) | (v.z != 0.f) | (v.w != 0.f);
    }
    ok = nz;
  }
  if (__all_sync(0xffffffffu, !ok)) return;  // warp-uniform exit keeps the shuffles full
  const int64_t gid = ok ? (rows ? rows[i] : i) : 0;
  double xn[3];
  normalise(g, means + 3 * gid, xn);
  const size_t T = (size_t)1 << g.log2_table;
  for (int l = 0; l < L; ++l) {
    uint32_t idx[8];
    float w[8];
    level_corners(g, l, xn, idx, w);
    float* gl = g_tables + (size_t)l * T * F;
    if (F == 2) {
      const float2 d = ok ? *reinterpret_cast<const float2*>(dr + 2 * l) : make_float2(0.f, 0.f);
      const bool live = ok && (d.x != 0.f || d.y != 0.f);
      // the 8 corners' warp aggregations side by side (independent shuffle
      // chains overlap): runs of equal keys in adjacent lanes, segmented
      // suffix sums over only as many steps as the longest run needs
      const int lane = threadIdx.x & 31;
      uint32_t key[8], seg_end[8];
      float vx[8], vy[8];
      bool head[8];
      uint32_t all_heads = 0xffffffffu;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        key[k] = live ? idx[k] : 0xffffffffu;
        vx[k] = w[k] * d.x;
        vy[k] = w[k] * d.y;
        const uint32_t prev = __shfl_up_sync(0xffffffffu, key[k], 1);
        head[k] = lane == 0 || prev != key[k];
        const uint32_t heads = __ballot_sync(0xffffffffu, head[k]);
        all_heads &= heads;
        const uint32_t after = heads & ~(0xffffffffu >> (31 - lane));  // heads above lane
        seg_end[k] = after ? __ffs(after) - 1 : 32;
      }
      if (all_heads != 0xffffffffu) {
        uint32_t run = 1;
#pragma unroll
        for (int k = 0; k < 8; ++k) run = max(run, head[k] ? seg_end[k] - lane : 1u);
        run = __reduce_max_sync(0xffffffffu, run);
        for (int off = 1; off < (int)run; off <<= 1) {  // warp-uniform
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float ox = __shfl_down_sync(0xffffffffu, vx[k], off);
            const float oy = __shfl_down_sync(0xffffffffu, vy[k], off);
            if (lane + off < (int)seg_end[k]) vx[k] += ox, vy[k] += oy;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (head[k] && key[k] != 0xffffffffu) red_add_v2(gl + 2 * (size_t)key[k], vx[k], vy[k]);
    } else if (ok) {
      for (int f = 0; f < F; ++f) {
        const float d = dr[l * F + f];
#pragma unroll
        for (int k = 0; k < 8; ++k) atomicAdd(gl + (size_t)idx[k] * F + f, w[k] * d);
      }
    }
  }
}

// K2f: decoder, one thread per row, weights broadcast from smem (ntc.py:241-248).
template <int IN, int NL>
__global__ void __launch_bounds__(128) mlp_fwd_kernel(int64_t n, const float* __restrict__ X,
                                                      int xs, const float* __restrict__ params,
                                                      float* __restrict__ out, int os) {
  extern __shared__ __align__(16) float smem[];
  load_params<Lay<IN, NL>::TOTAL>(smem, params);
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x[IN], h1[HID], h2[HID], o[OUTP];
#pragma unroll
  for (int k = 0; k < IN; k += 4) {
    const float4 v = *reinterpret_cast<const float4*>(X + i * xs + k);
    x[k] = v.x, x[k + 1] = v.y, x[k + 2] = v.z, x[k + 3] = v.w;
  }
  mlp_forward<IN, NL>(smem, x, h1, h2, o);
  if (os == 8) {
    *reinterpret_cast<float4*>(out + i * 8) = make_float4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<float4*>(out + i * 8 + 4) = make_float4(o[4], o[5], o[6], 0.f);
  } else {
#pragma unroll
    for (int k = 0; k < 7; ++k) out[i * os + k] = o[k];
  }
}

// K3f: transform (transform.py:70-84): mu' = mu + d_mu, q' = norm(d_q) (x) q_src,
// SH bands >= 1 rotated by R(norm(d_q)).  Three lanes per inside row (rows in
// index order, so a warp reads ~11 consecutive cloud rows): lane c rotates
// colour channel c; lane 0 also writes the mean and the rotation.
template <int DEG>
__global__ void __launch_bounds__(128) transform_kernel(ss_cloud src, int64_t n,
                                                        const int32_t* __restrict__ rows,
                                                        const int32_t* __restrict__ pos,
                                                        const float* __restrict__ out7, int os,
                                                        int rotate_sh, float* __restrict__ t_means,
                                                        float* __restrict__ t_rot,
                                                        float* __restrict__ t_sh,
                                                        uint32_t* status) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  // three lanes per row (no idle fourth lane): lane c rotates colour channel c,
  // lane 0 also writes the mean and the rotation
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j = t / 3;
  const int c = (int)(t - 3 * j);
  if (j >= n) return;
  // rows in index order (coalesced cloud rows); pos = the row's slot in out7
  const int64_t gid = rows ? rows[j] : j;
  const int64_t i = pos ? pos[j] : j;
  float o[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) o[k] = out7[i * os + k];
  float nq = sqrtf(o[3] * o[3] + o[4] * o[4] + o[5] * o[5] + o[6] * o[6]);
  if (nq < 1e-12f) {  // gaussians.py:46-47
    if (status && c == 0) atomicOr(status, SS_FLAG_ZERO_QUAT);
    nq = 1.f;
  }
  const float u[4] = {o[3] / nq, o[4] / nq, o[5] / nq, o[6] / nq};
  if (c == 0) {
    const float* m = src.means + 3 * gid;
    t_means[3 * gid + 0] = m[0] + o[0];
    t_means[3 * gid + 1] = m[1] + o[1];
    t_means[3 * gid + 2] = m[2] + o[2];
    const float4 q = *reinterpret_cast<const float4*>(src.rotations + 4 * gid);
    const float qs[4] = {q.x, q.y, q.z, q.w};
    float qo[4];
    quat_mul(u, qs, qo);
    *reinterpret_cast<float4*>(t_rot + 4 * gid) = make_float4(qo[0], qo[1], qo[2], qo[3]);
  }
  if (DEG < 1 || !rotate_sh) return;
  float R[3][3];
  quat_to_rot(u[0], u[1], u[2], u[3], R);
  const float* sh = src.sh + gid * 3 * K + c;
  float* tsh = t_sh + gid * 3 * K + c;
  {  // band 1: P R P^T
    float in[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) in[b] = sh[(1 + b) * 3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float sum = 0.f;
#pragma unroll
      for (int b = 0; b < 3; ++b) sum = fmaf(R[c_perm(a)][c_perm(b)], in[b], sum);
      tsh[(1 + a) * 3] = sum;
    }
  }
  if (DEG >= 2) {
    float in[5], out[5];
#pragma unroll
    for (int b = 0; b < 5; ++b) in[b] = sh[(4 + b) * 3];
    rotate_band_channel<5>(R, in, out);
#pragma unroll
    for (int a = 0; a < 5; ++a) tsh[(4 + a) * 3] = out[a];
  }
  if (DEG >= 3) {
    float in[7], out[7];
#pragma unroll
    for (int b = 0; b < 7; ++b) in[b] = sh[(9 + b) * 3];
    rotate_band_channel<7>(R, in, out);
#pragma unroll
    for (int a = 0; a < 7; ++a) tsh[(9 + a) * 3] = out[a];
  }
}

// K3b: dL/d[d_mu | d_q] from transformed-cloud gradients (transform.py:111-134).
// One thread per inside row.  The SH part of g_R is linear in the per-channel
// band gradients, so each band direction k is evaluated once for the three
// channels: with h_kc = (S^{-T} g_c)_k and w = sum_c h_kc in_c, direction k
// contributes d_k (x) grad f_w(R^T d_k) (band_channel_vjp summed over c).
// Then A(q_src)^T g_rot, the rotation and normalisation Jacobians -> g7.
template <int B>
__device__ __forceinline__ void band_vjp_rows(const float R[3][3], const float (*gc)[B],
                                              const float (*ic)[B], float gR[3][3]) {
  const float(*dirs)[3] = B == 5 ? c_shrot.dirs2 : c_shrot.dirs3;
  const float* sinv = B == 5 ? &c_shrot.binvT2[0][0] : &c_shrot.binvT3[0][0];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    float h[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < B; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) h[c] = fmaf(sinv[a * B + k], gc[c][a], h[c]);
    float w[B];
#pragma unroll
    for (int b = 0; b < B; ++b) w[b] = h[0] * ic[0][b] + h[1] * ic[1][b] + h[2] * ic[2][b];
    float e[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
      e[i] = R[0][i] * dirs[k][0] + R[1][i] * dirs[k][1] + R[2][i] * dirs[k][2];
    float ge[3];
    band_grad(w, e[0], e[1], e[2], ge, B);
#pragma unroll
    for (int jj = 0; jj < 3; ++jj)
#pragma unroll
      for (int ii = 0; ii < 3; ++ii) gR[jj][ii] = fmaf(dirs[k][jj], ge[ii], gR[jj][ii]);
  }
}

// coefficients [first, first + B) of the 3 channels of one SH row (3K floats,
// coefficient-major): out[c][b] = row[3 (first + b) + c]
template <int B>
__device__ __forceinline__ void load_band(const float* __restrict__ row, int first, float (*out)[B]) {
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int c = 0; c < 3; ++c) out[c][b] = __ldg(row + 3 * (first + b) + c);
}

template <int DEG>
__global__ void __launch_bounds__(128) transform_vjp_kernel(
    ss_cloud src, int64_t n, const int32_t* __restrict__ rows, const int32_t* __restrict__ pos,
    const float* __restrict__ out7, int os, int rotate_sh, const float* __restrict__ d_means,
    const float* __restrict__ d_rot, const float* __restrict__ d_sh, float* __restrict__ g7,
    int gs, const uint8_t* __restrict__ live) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t gid = rows ? rows[j] : j;
  const int64_t i = pos ? pos[j] : j;
  // a Gaussian no pixel of this view used has all-zero gradients: g7 row = 0
  if (live && !live[gid]) {
    if (gs == 8) {
      *reinterpret_cast<float4*>(g7 + i * 8) = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(g7 + i * 8 + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      for (int k = 0; k < gs; ++k) g7[i * gs + k] = 0.f;
    }
    return;
  }
  float o[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) o[k] = out7[i * os + k];
  float nq = sqrtf(o[3] * o[3] + o[4] * o[4] + o[5] * o[5] + o[6] * o[6]);
  nq = nq < 1e-12f ? 1.f : nq;
  const float u[4] = {o[3] / nq, o[4] / nq, o[5] / nq, o[6] / nq};
  float gR[3][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
  const bool rot = DEG >= 1 && rotate_sh;
  if (rot) {
    float R[3][3];
    quat_to_rot(u[0], u[1], u[2], u[3], R);
    const float* sh = src.sh + gid * 3 * K;
    const float* gsh = d_sh + gid * 3 * K;
    {  // band 1: g_R += P^T (sum_c g_c in_c^T) P
      float in[3][3], g[3][3];
      load_band<3>(sh, 1, in);
      load_band<3>(gsh, 1, g);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            gR[c_perm(a)][c_perm(b)] = fmaf(g[c][a], in[c][b], gR[c_perm(a)][c_perm(b)]);
    }
    if (DEG >= 2) {
      float in[3][5], g[3][5];
      load_band<5>(sh, 4, in);
      load_band<5>(gsh, 4, g);
      band_vjp_rows<5>(R, g, in, gR);
    }
    if (DEG >= 3) {
      float in[3][7], g[3][7];
      load_band<7>(sh, 9, in);
      load_band<7>(gsh, 9, g);
      band_vjp_rows<7>(R, g, in, gR);
    }
  }
  const float4 q = *reinterpret_cast<const float4*>(src.rotations + 4 * gid);
  const float4 gr = *reinterpret_cast<const float4*>(d_rot + 4 * gid);
  // g_u = A(q_src)^T g_rot, A rows: [w,-x,-y,-z],[x,w,z,-y],[y,-z,w,x],[z,y,-x,w]
  float gu[4];
  gu[0] = q.x * gr.x + q.y * gr.y + q.z * gr.z + q.w * gr.w;
  gu[1] = -q.y * gr.x + q.x * gr.y - q.w * gr.z + q.z * gr.w;
  gu[2] = -q.z * gr.x + q.w * gr.y + q.x * gr.z - q.y * gr.w;
  gu[3] = -q.w * gr.x - q.z * gr.y + q.y * gr.z + q.x * gr.w;
  if (rot) {
    float gq[4];
    quat_to_rot_vjp(u[0], u[1], u[2], u[3], gR, gq);
#pragma unroll
    for (int k = 0; k < 4; ++k) gu[k] += gq[k];
  }
  // (I - u u^T)/|q| (gaussians.py:109-117)
  const float dot = u[0] * gu[0] + u[1] * gu[1] + u[2] * gu[2] + u[3] * gu[3];
  float r[8] = {d_means[3 * gid], d_means[3 * gid + 1], d_means[3 * gid + 2], 0.f, 0.f, 0.f, 0.f,
                0.f};
#pragma unroll
  for (int k = 0; k < 4; ++k) r[3 + k] = (gu[k] - u[k] * dot) / nq;
  if (gs == 8) {
    *reinterpret_cast<float4*>(g7 + i * 8) = make_float4(r[0], r[1], r[2], r[3]);
    *reinterpret_cast<float4*>(g7 + i * 8 + 4) = make_float4(r[4], r[5], r[6], 0.f);
  } else {
#pragma unroll
    for (int k = 0; k < 7; ++k) g7[i * gs + k] = r[k];
  }
}

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

// K2b: decoder backward.  Persistent CTAs walk 128-row chunks: each thread
// recomputes its row's hidden layers from X (staged through its shared-memory
// rows), back-propagates g7 to dX (written to HBM for the scatter kernel), and
// the CTA reduces the weight gradient over the chunk with register-blocked
// 4x4 tiles flushed by vector reductions (ntc.py:258-276).
template <int IN, int NL>
__global__ void __launch_bounds__(kChunk, 1) mlp_bwd_kernel(
    int64_t n, const float* __restrict__ X, int xs, const float* __restrict__ g_out, int gs,
    const float* __restrict__ params, float* __restrict__ dX, float* __restrict__ g_params) {
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
      uint64_t mask1 = 0, mask2 = 0;
#pragma unroll
      for (int k = 0; k < IN; k += 4)
        *reinterpret_cast<float4*>(sX + k) = *reinterpret_cast<const float4*>(X + i * xs + k);
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
      for (int k = 0; k < 7; ++k) g7[k] = g_out[i * gs + k];
      g7[7] = 0.f;
      *reinterpret_cast<float4*>(sG) = make_float4(g7[0], g7[1], g7[2], g7[3]);
      *reinterpret_cast<float4*>(sG + 4) = make_float4(g7[4], g7[5], g7[6], g7[7]);
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
      // feature gradient dX = W0 d1 -> HBM for the scatter kernel
#pragma unroll
      for (int r0 = 0; r0 < IN; r0 += 4) {
        float dv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4* w4 = reinterpret_cast<const float4*>(smem + L::W0 + (r0 + u) * HID);
          float s = 0.f;
#pragma unroll
          for (int q = 0; q < HID / 4; ++q) {
            const float4 w = w4[q];
            s = fmaf(w.x, d1[4 * q], s);
            s = fmaf(w.y, d1[4 * q + 1], s);
            s = fmaf(w.z, d1[4 * q + 2], s);
            s = fmaf(w.w, d1[4 * q + 3], s);
          }
          dv[u] = s;
        }
        *reinterpret_cast<float4*>(dX + i * xs + r0) = make_float4(dv[0], dv[1], dv[2], dv[3]);
      }
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
    // ---- CTA-level weight-gradient GEMM over the chunk (ntc.py:271-273)
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
          const float4 v = *reinterpret_cast<const float4*>(pd + r * d.d_stride);
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
          const float4 a = *reinterpret_cast<const float4*>(pa + r * d.a_stride);
          const float4 v = *reinterpret_cast<const float4*>(pd + r * d.d_stride);
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
__global__ void __launch_bounds__(256) adam_kernel(
    int64_t n_table, float* __restrict__ tables, float* __restrict__ g_tables,
    double* __restrict__ m_t, double* __restrict__ v_t, const uint8_t* __restrict__ row_mask,
    int row_width, int64_t n_params, float* __restrict__ params, float* __restrict__ g_params,
    double* __restrict__ m_p, double* __restrict__ v_p, const int32_t* __restrict__ step_dev,
    double lr, double b1, double b2, double eps, int zero_grads) {
  __shared__ double s_bc[2];
  if (threadIdx.x == 0) {  // bias corrections once per block (optim.py:52-53), as reciprocals
    const int step = *step_dev + 1;
    s_bc[0] = 1.0 / (1.0 - pow(b1, (double)step));
    s_bc[1] = 1.0 / (1.0 - pow(b2, (double)step));
  }
  __syncthreads();
  const double ibc1 = s_bc[0], ibc2 = s_bc[1];
  const int shift = (row_width & (row_width - 1)) == 0 ? __ffs(row_width) - 1 : -1;
  const int64_t total = n_table + n_params;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float *p, *gp;
    double *m, *v;
    int64_t j;
    if (i < n_table) {
      j = i;
      p = tables, gp = g_tables, m = m_t, v = v_t;
      // untouched rows: no Adam update, and their gradient is never written
      if (row_mask && !row_mask[shift >= 0 ? (j >> shift) : (j / row_width)]) continue;
    } else {
      j = i - n_table;
      p = params, gp = g_params, m = m_p, v = v_p;
    }
    const double g = gp[j];
    const double mm = b1 * m[j] + (1.0 - b1) * g;
    const double vv = b2 * v[j] + (1.0 - b2) * (g * g);
    m[j] = mm;
    v[j] = vv;
    p[j] = (float)((double)p[j] - lr * (mm * ibc1) / (sqrt(vv * ibc2) + eps));
    if (zero_grads) gp[j] = 0.f;
  }
}

// Two-feature tables (the common F = 2): one row per thread iteration with
// 8/16-byte vector accesses and one mask read per row; the MLP part is scalar.
__global__ void __launch_bounds__(256) adam_rows2_kernel(
    int64_t n_rows, float2* __restrict__ tables, float2* __restrict__ g_tables,
    double2* __restrict__ m_t, double2* __restrict__ v_t, const uint8_t* __restrict__ row_mask,
    int64_t n_params, float* __restrict__ params, float* __restrict__ g_params,
    double* __restrict__ m_p, double* __restrict__ v_p, const int32_t* __restrict__ step_dev,
    double lr, double b1, double b2, double eps, int zero_grads) {
  __shared__ double s_bc[2];
  if (threadIdx.x == 0) {  // bias corrections once per block (optim.py:52-53), as reciprocals
    const int step = *step_dev + 1;
    s_bc[0] = 1.0 / (1.0 - pow(b1, (double)step));
    s_bc[1] = 1.0 / (1.0 - pow(b2, (double)step));
  }
  __syncthreads();
  const double ibc1 = s_bc[0], ibc2 = s_bc[1];
  auto upd = [&](double g, double& m, double& v, float& p) {
    m = b1 * m + (1.0 - b1) * g;
    v = b2 * v + (1.0 - b2) * (g * g);
    p = (float)((double)p - lr * (m * ibc1) / (sqrt(v * ibc2) + eps));
  };
  const int64_t total = n_rows + n_params;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n_rows) {
      // untouched rows: no Adam update, and their gradient is never written
      if (row_mask && !row_mask[i]) continue;
      const float2 g = g_tables[i];
      double2 m = m_t[i], v = v_t[i];
      float2 p = tables[i];
      upd(g.x, m.x, v.x, p.x);
      upd(g.y, m.y, v.y, p.y);
      m_t[i] = m;
      v_t[i] = v;
      tables[i] = p;
      if (zero_grads) g_tables[i] = make_float2(0.f, 0.f);
    } else {
      const int64_t j = i - n_rows;
      double m = m_p[j], v = v_p[j];
      float p = params[j];
      upd(g_params[j], m, v, p);
      m_p[j] = m;
      v_p[j] = v;
      params[j] = p;
      if (zero_grads) g_params[j] = 0.f;
    }
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
  if (mlp) {
    // the decoder shape decides the scratch layout: reject it before any carving
    ss_mlp_layout L{};
    if (ss_mlp_get_layout(mlp, &L) != SS_OK) return SS_ERR_DATA;
    if (g->n_levels * g->n_features != mlp->in_dim) {
      set_error("decoder in_dim must equal n_levels * n_features");
      return SS_ERR_DATA;
    }
  }
  return SS_OK;
}

static int in_pad_of(const ss_mlp* mlp) {
  ss_mlp_layout L{};
  ss_mlp_get_layout(mlp, &L);
  return L.in_pad;
}

static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

struct MlpFwd {
  int64_t n;
  const float* X;
  int xs;
  const float* params;
  float* out;
  int os;
  cudaStream_t st;
  template <int IN, int NL>
  int run() {
    const size_t smem = Lay<IN, NL>::TOTAL * sizeof(float);
    auto k = mlp_fwd_kernel<IN, NL>;
    SS_CUDA(smem_attr_once(k, (int)smem));
    k<<<(unsigned)cdiv(n, 128), 128, smem, st>>>(n, X, xs, params, out, os);
    SS_CHECK_LAUNCH("mlp_fwd_kernel");
    return SS_OK;
  }
};

struct MlpBwd {
  int64_t n;
  const float* X;
  int xs;
  const float* g;
  int gs;
  const float* params;
  float *dX, *g_params;
  cudaStream_t st;
  template <int IN, int NL>
  int run() {
    const size_t smem = BwdSmem<IN, NL>::FLOATS * sizeof(float);
    auto k = mlp_bwd_kernel<IN, NL>;
    SS_CUDA(smem_attr_once(k, (int)smem));
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv(n, kChunk), num_sms());
    k<<<grid, kChunk, smem, st>>>(n, X, xs, g, gs, params, dX, g_params);
    SS_CHECK_LAUNCH("mlp_bwd_kernel");
    return SS_OK;
  }
};

size_t ntc_scratch_bytes(const ss_mlp* mlp, int64_t n) {
  const int xs = mlp ? in_pad_of(mlp) : 64;
  const size_t nn = (size_t)(n > 0 ? n : 1);
  return 2 * align_up(nn * xs * sizeof(float)) + 2 * align_up(nn * 8 * sizeof(float)) +
         align_up(nn * 2 * sizeof(uint64_t));
}

NtcScratch ntc_scratch(void* base, const ss_mlp* mlp, int64_t n) {
  NtcScratch s{};
  s.xs = mlp ? in_pad_of(mlp) : 64;
  Carve c(base);
  const size_t nn = (size_t)(n > 0 ? n : 1);
  s.X = c.take<float>(nn * s.xs);
  s.dX = c.take<float>(nn * s.xs);
  s.out7 = c.take<float>(nn * 8);
  s.g7 = c.take<float>(nn * 8);
  s.relu = c.take<uint64_t>(nn * 2);
  return s;
}

int ntc_forward_run(const ss_grid* g, const ss_mlp* mlp, int64_t n, const float* means,
                    const int32_t* rows, const float* tables, const float* params, float* X, int xs,
                    float* out, int os, uint64_t* relu, uint32_t* status, cudaStream_t st) {
  SS_TRY(check_grid(g, mlp));
  if (n == 0) return SS_OK;
  prof_begin(PH_GATHER, st);
  gather_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(*g, n, means, rows, tables, X, xs, status);
  SS_CHECK_LAUNCH("gather_kernel");
  prof_end(PH_GATHER, st);
  prof_begin(PH_DECODER_FWD, st);
  const int f16 = mlp->precision == SS_MLP_F16;  // tensor cores only
  if (f16 || mlp_mode() != 0)
    SS_TRY(mlp_fwd_tc(xs, mlp->n_hidden, f16, n, X, xs, params, out, os, relu, st));  // tcgen05
  else
    SS_TRY(dispatch_mlp(mlp, MlpFwd{n, X, xs, params, out, os, st}));
  prof_end(PH_DECODER_FWD, st);
  return SS_OK;
}

int ntc_backward_run(const ss_grid* g, const ss_mlp* mlp, int64_t n, const float* means,
                     const int32_t* rows, const float* params, const float* X, int xs,
                     const float* g_out, int gs, const uint64_t* relu, float* dX,
                     float* g_tables, float* g_params, cudaStream_t st) {
  SS_TRY(check_grid(g, mlp));
  if (n == 0) return SS_OK;
  prof_begin(PH_DECODER_BWD, st);
  const int f16 = mlp->precision == SS_MLP_F16;
  if (f16 || mlp_mode() != 0)
    SS_TRY(mlp_bwd_tc(xs, mlp->n_hidden, f16, n, X, xs, g_out, gs, relu, params, dX, g_params, st));
  else
    SS_TRY(dispatch_mlp(mlp, MlpBwd{n, X, xs, g_out, gs, params, dX, g_params, st}));
  prof_end(PH_DECODER_BWD, st);
  // g_tables == nullptr: the caller runs the scatter later (ntc_scatter_run)
  return g_tables ? ntc_scatter_run(g, n, means, rows, dX, xs, g_tables, st) : SS_OK;
}

int ntc_scatter_run(const ss_grid* g, int64_t n, const float* means, const int32_t* rows,
                    const float* dX, int xs, float* g_tables, cudaStream_t st) {
  SS_TRY(check_grid(g, nullptr));
  if (n == 0) return SS_OK;
  prof_begin(PH_SCATTER, st);
  scatter_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(*g, n, means, rows, dX, xs, g_tables);
  SS_CHECK_LAUNCH("scatter_kernel");
  prof_end(PH_SCATTER, st);
  return SS_OK;
}

int transform_run(const ss_cloud* src, int64_t n, const int32_t* rows, const int32_t* pos,
                  const float* out7, int os, int rotate_sh, float* tm, float* tr, float* ts,
                  uint32_t* status, cudaStream_t st) {
  if (!src || src->sh_coeffs < 1 || src->sh_coeffs > 16) {
    set_error("transform: bad cloud");
    return SS_ERR_DATA;
  }
  if (n == 0) return SS_OK;
  SS_TRY(ensure_shrot_const());
  prof_begin(PH_TRANSFORM, st);
  const unsigned grid = (unsigned)cdiv(3 * n, 128);  // 3 lanes per row
  switch (sh_degree_of(src->sh_coeffs)) {
    case 0: transform_kernel<0><<<grid, 128, 0, st>>>(*src, n, rows, pos, out7, os, rotate_sh, tm, tr, ts, status); break;
    case 1: transform_kernel<1><<<grid, 128, 0, st>>>(*src, n, rows, pos, out7, os, rotate_sh, tm, tr, ts, status); break;
    case 2: transform_kernel<2><<<grid, 128, 0, st>>>(*src, n, rows, pos, out7, os, rotate_sh, tm, tr, ts, status); break;
    default: transform_kernel<3><<<grid, 128, 0, st>>>(*src, n, rows, pos, out7, os, rotate_sh, tm, tr, ts, status); break;
  }
  SS_CHECK_LAUNCH("transform_kernel");
  prof_end(PH_TRANSFORM, st);
  return SS_OK;
}

int transform_vjp_run(const ss_cloud* src, int64_t n, const int32_t* rows, const int32_t* pos,
                      const float* out7, int os, int rotate_sh, const float* dm, const float* dr,
                      const float* ds, float* g7, int gs, cudaStream_t st, const uint8_t* live) {
  if (!src || src->sh_coeffs < 1 || src->sh_coeffs > 16) {
    set_error("transform vjp: bad cloud");
    return SS_ERR_DATA;
  }
  if (n == 0) return SS_OK;
  SS_TRY(ensure_shrot_const());
  prof_begin(PH_TRANSFORM_BWD, st);
  const unsigned grid = (unsigned)cdiv(n, 128);  // one thread per row
  switch (sh_degree_of(src->sh_coeffs)) {
    case 0: transform_vjp_kernel<0><<<grid, 128, 0, st>>>(*src, n, rows, pos, out7, os, rotate_sh, dm, dr, ds, g7, gs, live); break;
    case 1: transform_vjp_kernel<1><<<grid, 128, 0, st>>>(*src, n, rows, pos, out7, os, rotate_sh, dm, dr, ds, g7, gs, live); break;
    case 2: transform_vjp_kernel<2><<<grid, 128, 0, st>>>(*src, n, rows, pos, out7, os, rotate_sh, dm, dr, ds, g7, gs, live); break;
    default: transform_vjp_kernel<3><<<grid, 128, 0, st>>>(*src, n, rows, pos, out7, os, rotate_sh, dm, dr, ds, g7, gs, live); break;
  }
  SS_CHECK_LAUNCH("transform_vjp_kernel");
  prof_end(PH_TRANSFORM_BWD, st);
  return SS_OK;
}

// F2 warm-up loss (losses.py:151-180): per row |d_mu|_1 - w^2 / |d_q|^2, summed
// in fp64; gradients of the batch mean written to g7 (n, 8)
__global__ void __launch_bounds__(256) warmup_loss_kernel(int64_t n, const float* __restrict__ out7,
                                                          float* __restrict__ g7,
                                                          double* __restrict__ loss_sum,
                                                          uint32_t* status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double term = 0.0;
  if (i < n) {
    const float4 a = *reinterpret_cast<const float4*>(out7 + 8 * i);
    const float4 b = *reinterpret_cast<const float4*>(out7 + 8 * i + 4);
    const double mu[3] = {a.x, a.y, a.z}, q[4] = {a.w, b.x, b.y, b.z};
    const double n2 = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
    if (n2 < 1e-24 && status) atomicOr(status, SS_FLAG_ZERO_QUAT);
    const double w = q[0], inv_b = 1.0 / (double)n, in4 = 1.0 / (n2 * n2);
    term = fabs(mu[0]) + fabs(mu[1]) + fabs(mu[2]) - w * w / n2;
    auto sgn = [](double v) { return (double)((v > 0.0) - (v < 0.0)); };
    float4 ga, gb;
    ga.x = (float)(sgn(mu[0]) * inv_b);
    ga.y = (float)(sgn(mu[1]) * inv_b);
    ga.z = (float)(sgn(mu[2]) * inv_b);
    ga.w = (float)(-2.0 * w * (n2 - w * w) * in4 * inv_b);
    gb.x = (float)(2.0 * w * w * q[1] * in4 * inv_b);
    gb.y = (float)(2.0 * w * w * q[2] * in4 * inv_b);
    gb.z = (float)(2.0 * w * w * q[3] * in4 * inv_b);
    gb.w = 0.f;
    *reinterpret_cast<float4*>(g7 + 8 * i) = ga;
    *reinterpret_cast<float4*>(g7 + 8 * i + 4) = gb;
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = term;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
    atomicAdd(loss_sum, t);
  }
}

// stream-ordered temporary for the reference-shaped API entry points
struct Temp {
  void* p = nullptr;
  cudaStream_t st;
  explicit Temp(cudaStream_t s) : st(s) {}
  int alloc(size_t bytes) {
    SS_CUDA(cudaMallocAsync(&p, bytes, st));
    return SS_OK;
  }
  ~Temp() {
    if (p) cudaFreeAsync(p, st);
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

__global__ void copy_cols_kernel(int64_t n, const float* __restrict__ src, int ss, int cols,
                                 float* __restrict__ dst, int ds) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * cols) return;
  const int64_t i = t / cols;
  const int c = (int)(t - i * cols);
  dst[i * ds + c] = src[i * ss + c];
}

int ss_ntc_forward(const ss_grid* grid, const ss_mlp* mlp, int64_t n, const float* means,
                   const int32_t* rows, const float* tables, const float* params, float* out7,
                   float* feats, void* stream) {
  SS_TRY(check_grid(grid, mlp));
  if (n == 0) return SS_OK;
  cudaStream_t st = as_stream(stream);
  Temp tmp(st);
  SS_TRY(tmp.alloc(ntc_scratch_bytes(mlp, n)));
  NtcScratch s = ntc_scratch(tmp.p, mlp, n);
  SS_TRY(ntc_forward_run(grid, mlp, n, means, rows, tables, params, s.X, s.xs, out7, 7, s.relu,
                         nullptr, st));
  if (feats) {
    const int nf = grid->n_levels * grid->n_features;
    copy_cols_kernel<<<(unsigned)cdiv(n * nf, 256), 256, 0, st>>>(n, s.X, s.xs, nf, feats, nf);
    SS_CHECK_LAUNCH("copy_cols_kernel");
  }
  return SS_OK;
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
  if (n == 0) return SS_OK;
  cudaStream_t st = as_stream(stream);
  Temp tmp(st);
  SS_TRY(tmp.alloc(ntc_scratch_bytes(mlp, n)));
  NtcScratch s = ntc_scratch(tmp.p, mlp, n);
  // decoder forward recomputed: features and the ReLU masks the backward reuses
  SS_TRY(ntc_forward_run(grid, mlp, n, means, rows, tables, params, s.X, s.xs, s.out7, 8, s.relu,
                         nullptr, st));
  return ntc_backward_run(grid, mlp, n, means, rows, params, s.X, s.xs, g_out7, 7, s.relu, s.dX,
                          g_tables, g_params, st);
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
  if (n_in == 0) return SS_OK;
  cudaStream_t st = as_stream(stream);
  Temp tmp(st);
  SS_TRY(tmp.alloc(ntc_scratch_bytes(mlp, n_in)));
  NtcScratch s = ntc_scratch(tmp.p, mlp, n_in);
  float* o = out7 ? out7 : s.out7;
  const int os = out7 ? 7 : 8;
  SS_TRY(ntc_forward_run(grid, mlp, n_in, src->means, rows, tables, params, s.X, s.xs, o, os,
                         s.relu, status, st));
  return transform_run(src, n_in, rows, nullptr, o, os, rotate_sh, out_means, out_rotations,
                       out_sh, status, st);
}

size_t ss_apply_ntc_backward_bytes(int64_t n_in) { return ntc_scratch_bytes(nullptr, n_in); }

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
  cudaStream_t st = as_stream(stream);
  // decoder output recomputed (K1f/K2f), then K3b, K2b and K1b
  NtcScratch s = ntc_scratch(scratch, mlp, n_in);
  SS_TRY(ntc_forward_run(grid, mlp, n_in, src->means, rows, tables, params, s.X, s.xs, s.out7, 8,
                         s.relu, nullptr, st));
  SS_TRY(transform_vjp_run(src, n_in, rows, nullptr, s.out7, 8, rotate_sh, d_means, d_rotations,
                           d_sh, s.g7, 8, st));
  return ntc_backward_run(grid, mlp, n_in, src->means, rows, params, s.X, s.xs, s.g7, 8, s.relu,
                          s.dX,
                          g_tables, g_params, st);
}

int ss_transform_apply(const ss_cloud* src, int64_t n_in, const int32_t* rows, const float* out7,
                       int32_t rotate_sh, float* out_means, float* out_rotations, float* out_sh,
                       uint32_t* status, void* stream) {
  return transform_run(src, n_in, rows, nullptr, out7, 7, rotate_sh, out_means, out_rotations,
                       out_sh, status, as_stream(stream));
}

int ss_transform_vjp(const ss_cloud* src, int64_t n_in, const int32_t* rows, const float* out7,
                     int32_t rotate_sh, const float* d_means, const float* d_rotations,
                     const float* d_sh, float* g_out7, void* stream) {
  return transform_vjp_run(src, n_in, rows, nullptr, out7, 7, rotate_sh, d_means, d_rotations,
                           d_sh, g_out7, 7, as_stream(stream));
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
    const bool rows2 = row_width == 2 && n_table % 2 == 0 &&
                       ((reinterpret_cast<uintptr_t>(tables) | reinterpret_cast<uintptr_t>(g_tables) |
                         reinterpret_cast<uintptr_t>(m_tables) | reinterpret_cast<uintptr_t>(v_tables)) &
                        15) == 0;
    if (rows2) {
      const unsigned b2 = (unsigned)std::min<int64_t>(cdiv(n_table / 2 + n_params, 256), 148 * 8);
      adam_rows2_kernel<<<b2, 256, 0, st>>>(
          n_table / 2, reinterpret_cast<float2*>(tables), reinterpret_cast<float2*>(g_tables),
          reinterpret_cast<double2*>(m_tables), reinterpret_cast<double2*>(v_tables), row_mask,
          n_params, params, g_params, m_params, v_params, step_dev, lr, beta1, beta2, eps,
          zero_grads);
      SS_CHECK_LAUNCH("adam_rows2_kernel");
    } else {
      adam_kernel<<<blocks, 256, 0, st>>>(n_table, tables, g_tables, m_tables, v_tables, row_mask,
                                          row_width, n_params, params, g_params, m_params,
                                          v_params, step_dev, lr, beta1, beta2, eps, zero_grads);
      SS_CHECK_LAUNCH("adam_kernel");
    }
    prof_end(PH_ADAM, st);
  }
  increment_kernel<<<1, 1, 0, st>>>(step_dev);
  SS_CHECK_LAUNCH("increment_kernel");
  return SS_OK;
}

size_t ss_ntc_warmup_bytes(int64_t n) { return ntc_scratch_bytes(nullptr, n); }

int ss_ntc_warmup_step(const ss_grid* grid, const ss_mlp* mlp, int64_t n, const float* batch,
                       float* tables, float* params, float* g_tables, float* g_params,
                       double* m_tables, double* v_tables, double* m_params, double* v_params,
                       uint8_t* row_mask, int32_t* step_dev, double lr, void* scratch,
                       double* loss_sum, uint32_t* status, void* stream) {
  SS_TRY(check_grid(grid, mlp));
  if (n <= 0 || !batch || !scratch || !loss_sum || !row_mask || !step_dev) {
    set_error("ss_ntc_warmup_step: empty batch or missing buffers");  // losses.py:167-168
    return SS_ERR_DATA;
  }
  cudaStream_t st = as_stream(stream);
  const int64_t T = (int64_t)1 << grid->log2_table;
  // touched rows = the batch's corners (ntc.py:187, :330)
  SS_CUDA(cudaMemsetAsync(row_mask, 0, (size_t)grid->n_levels * T, st));
  SS_TRY(ss_ntc_touched(grid, n, batch, nullptr, row_mask, stream));
  NtcScratch s = ntc_scratch(scratch, mlp, n);
  SS_TRY(ntc_forward_run(grid, mlp, n, batch, nullptr, tables, params, s.X, s.xs, s.out7, 8,
                         s.relu, status, st));
  SS_CUDA(cudaMemsetAsync(loss_sum, 0, sizeof(double), st));
  warmup_loss_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(n, s.out7, s.g7, loss_sum, status);
  SS_CHECK_LAUNCH("warmup_loss_kernel");
  SS_TRY(ntc_backward_run(grid, mlp, n, batch, nullptr, params, s.X, s.xs, s.g7, 8, s.relu, s.dX,
                          g_tables, g_params, st));
  ss_mlp_layout L{};
  SS_TRY(ss_mlp_get_layout(mlp, &L));
  return ss_adam_step((int64_t)grid->n_levels * T * grid->n_features, tables, g_tables, m_tables,
                      v_tables, row_mask, grid->n_features, L.total, params, g_params, m_params,
                      v_params, step_dev, lr, 0.9, 0.999, 1e-15, 1, stream);
}

}  // extern "C"
