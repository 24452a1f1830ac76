// Tile rasterizer on sm_100a: EWA projection + SH colour (K4a, float64),
// stable depth order (K4b), tile-rect prefix sum and key duplication (K4c),
// stable tile sort (K4d), tile blend (K4e), reverse blend (K5a) and the
// per-Gaussian chain back to raw parameters (K5b).
//
// Reference: rasterizer.py:107-402, cameras.py:132-178, sh.py:51-81,
// gaussians.py:120-154 (/root/reference/pkg/src/splatstream/).
#include <vector>

#include "common.cuh"

namespace ss {

// ------------------------------------------------------------------ workspace
constexpr int kAccStride = 12;  // 48 B per rank: two aligned v4 reductions

struct Geom {
  double* key_in;              // per gid: fp64 depth (+inf when culled), tie-break of the sort
  uint32_t *key32, *key32_tmp;  // per gid / rank: fp32 depth bits (the radix-sort key)
  int32_t *idx_in, *order;
  int32_t* rank_of;  // per gid: its position in `order` (>= survivors when culled)
  double2* g_mean;   // per gid
  double4* g_conop;  // per gid (c00, c01+c10, c11, opacity)
  float4* g_color;   // per gid
  double2* g_cov;    // per gid (cov2d[0][0], cov2d[1][1]) for the tile rect
  double2* r_mean;   // per rank
  float4* r_conop;   // per rank, fp32 copy for the blend
  float4* r_q;       // per rank: log2 Gaussian form (A, B, C) and the reject bound log2(skip/op)
  double4* r_conop_d;
  float4* r_color;
  int4* r_rect;     // per rank (tx0, tx1, ty0, ty1)
  double4* r_cull;  // per rank: 2 ln(opacity / skip_alpha) (tile-cull threshold), -c01/c11, -c01/c00
  int64_t* offsets;  // per rank, exclusive prefix of tile counts (n+1)
  float* acc;        // per rank x kAccStride: colour 3, M0 | M1 2, M2 3 (anchor moments, K5a)
  uint8_t* touched;  // per rank
  float* t_final;    // per pixel
  int32_t* n_contrib;
  int2* ranges;      // per tile
  int32_t* tile_order;  // tiles by descending pair count: the blends' block -> tile map
  int64_t* dev_counts;  // [survivors, pairs, n, band pairs]
  int64_t* band_off;    // per rank, prefix of the pairs inside the current band of tile rows
  unsigned long long* row_pairs;  // per tile row: pairs of every visible rectangle
  BinSortWS dsort;      // depth sort workspace
  unsigned long long* scan_lb;  // single-pass offsets scan: look-back words per 256 ranks, then the ticket
  int64_t scan_blocks;
  size_t total;
};

struct Bins {
  uint32_t *keys_in, *keys_out, *vals_in, *vals_out;
  int64_t capacity;  // pairs the buffers hold; the count itself stays on the device
  BinSortWS sort;
  size_t total;
};

static inline int ntiles_x(const ss_camera* c, const ss_raster_settings* s) {
  return (c->width + s->tile_size - 1) / s->tile_size;
}
static inline int ntiles_y(const ss_camera* c, const ss_raster_settings* s) {
  return (c->height + s->tile_size - 1) / s->tile_size;
}
static inline int key_bits(int64_t ntiles) {
  int b = 1;
  while ((int64_t(1) << b) < ntiles) ++b;
  return b;
}

constexpr int kScanThreads = 256;  // threads per block of the fused offsets scans
constexpr int kScanRanks = 4;      // ranks per thread in rank_kernel

static Geom plan_geom(void* base, int64_t n, const ss_camera* cam, const ss_raster_settings* s) {
  Geom g{};
  Carve c(base);
  const int64_t P = (int64_t)cam->width * cam->height;
  const int64_t NT = (int64_t)ntiles_x(cam, s) * ntiles_y(cam, s);
  const int64_t nn = n > 0 ? n : 1;
  g.key_in = c.take<double>(nn);
  g.key32 = c.take<uint32_t>(nn);
  g.key32_tmp = c.take<uint32_t>(nn);
  g.idx_in = c.take<int32_t>(nn);
  g.order = c.take<int32_t>(nn);
  g.rank_of = c.take<int32_t>(nn);
  g.g_mean = c.take<double2>(nn);
  g.g_conop = c.take<double4>(nn);
  g.g_color = c.take<float4>(nn);
  g.g_cov = c.take<double2>(nn);
  g.r_mean = c.take<double2>(nn);
  g.r_conop = c.take<float4>(nn);
  g.r_q = c.take<float4>(nn);
  g.r_conop_d = c.take<double4>(nn);
  g.r_color = c.take<float4>(nn);
  g.r_rect = c.take<int4>(nn);
  g.r_cull = c.take<double4>(nn);
  g.offsets = c.take<int64_t>(nn + 1);
  g.acc = c.take<float>(nn * kAccStride);
  g.touched = c.take<uint8_t>(nn);
  g.t_final = c.take<float>(P);
  g.n_contrib = c.take<int32_t>(P);
  g.ranges = c.take<int2>(NT);
  g.tile_order = c.take<int32_t>(NT);
  g.dev_counts = c.take<int64_t>(4);
  g.band_off = c.take<int64_t>(nn + 1);
  g.row_pairs = c.take<unsigned long long>((size_t)ntiles_y(cam, s));
  g.dsort = binsort_plan(c, nn, 4);
  g.scan_blocks = (nn + kScanThreads - 1) / kScanThreads;  // band_counts: one rank per thread
  g.scan_lb = c.take<unsigned long long>(g.scan_blocks + 1);
  g.total = c.bytes();
  return g;
}

static Bins plan_bins(void* base, int64_t capacity) {
  Bins b{};
  Carve c(base);
  const int64_t pp = capacity > 0 ? capacity : 1;
  b.capacity = pp;
  b.keys_in = c.take<uint32_t>(pp);
  b.keys_out = c.take<uint32_t>(pp);
  b.vals_in = c.take<uint32_t>(pp);
  b.vals_out = c.take<uint32_t>(pp);
  b.sort = binsort_plan(c, pp, 2);
  b.total = c.bytes();
  return b;
}

static unsigned stride_grid(int64_t items) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(items, 256), 148 * 16));
}

// ------------------------------------------------------------------ projection
struct CamD {
  double R[3][3], t[3], pos[3];
  double fx, fy, cx, cy, near_clip;
  int W, H;
};

static CamD make_cam(const ss_camera* c) {
  CamD d{};
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) d.R[i][j] = c->w2c[4 * i + j];
    d.t[i] = c->w2c[4 * i + 3];
  }
  for (int i = 0; i < 3; ++i)  // position = -R^T t (cameras.py:73-76)
    d.pos[i] = -(d.R[0][i] * d.t[0] + d.R[1][i] * d.t[1] + d.R[2][i] * d.t[2]);
  d.fx = c->fx, d.fy = c->fy, d.cx = c->cx, d.cy = c->cy, d.near_clip = c->near_clip;
  d.W = c->width, d.H = c->height;
  return d;
}

// world covariance from raw quaternion + log scales (gaussians.py:120-124, :231-235)
__device__ inline void covariance3d(const float* q, const float* ls, double S[3][3],
                                    double Rq[3][3], double var[3], double u[4], double& qn) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  qn = sqrt(w * w + x * x + y * y + z * z);
  double inv = qn > 0 ? 1.0 / qn : 0.0;
  u[0] = w * inv, u[1] = x * inv, u[2] = y * inv, u[3] = z * inv;
  quat_to_rot(u[0], u[1], u[2], u[3], Rq);
  for (int i = 0; i < 3; ++i) var[i] = exp(2.0 * (double)ls[i]);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      S[i][j] = Rq[i][0] * var[0] * Rq[j][0] + Rq[i][1] * var[1] * Rq[j][1] +
                Rq[i][2] * var[2] * Rq[j][2];
}

struct Projected {
  double p[3], mean[2], M[2][3], cov2d[2][2], conic[2][2], dir[3], dist, op;
  double S[3][3], Rq[3][3], var[3], u[4], qn;
  double raw[3];
};

// geometry only (no SH colour): camera-space point, EWA covariance chain,
// conic, view direction, opacity
__device__ inline void project_geom(const CamD& cam, const ss_cloud& cl, int64_t i, Projected& P) {
  const float* m = cl.means + 3 * i;
  for (int r = 0; r < 3; ++r)
    P.p[r] = cam.R[r][0] * (double)m[0] + cam.R[r][1] * (double)m[1] +
             cam.R[r][2] * (double)m[2] + cam.t[r];
  const double x = P.p[0], y = P.p[1], z = P.p[2];
  P.mean[0] = cam.fx * x / z + cam.cx;  // cameras.py:141-145
  P.mean[1] = cam.fy * y / z + cam.cy;
  covariance3d(cl.rotations + 4 * i, cl.log_scales + 3 * i, P.S, P.Rq, P.var, P.u, P.qn);
  // J (cameras.py:148-160), M = J R_w, cov2d = M S M^T + 0.3 I (cameras.py:163-178)
  const double J[2][3] = {{cam.fx / z, 0.0, -cam.fx * x / (z * z)},
                          {0.0, cam.fy / z, -cam.fy * y / (z * z)}};
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b)
      P.M[a][b] = J[a][0] * cam.R[0][b] + J[a][1] * cam.R[1][b] + J[a][2] * cam.R[2][b];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      double s = 0;
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) s += P.M[a][j] * P.S[j][k] * P.M[b][k];
      P.cov2d[a][b] = s;
    }
  P.cov2d[0][0] += kLowpass;
  P.cov2d[1][1] += kLowpass;
  const double A = P.cov2d[0][0], B = P.cov2d[0][1], C = P.cov2d[1][0], D = P.cov2d[1][1];
  const double det = A * D - B * C;  // rasterizer.py:93-104
  P.conic[0][0] = D / det;
  P.conic[0][1] = -B / det;
  P.conic[1][0] = -C / det;
  P.conic[1][1] = A / det;
  double d[3];
  for (int r = 0; r < 3; ++r) d[r] = (double)m[r] - cam.pos[r];
  P.dist = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  const double dd = fmax(P.dist, 1e-12);
  for (int r = 0; r < 3; ++r) P.dir[r] = d[r] / dd;
  P.op = 1.0 / (1.0 + exp(-(double)cl.opacity_logits[i]));
}

template <int DEG>
__device__ inline void project_one(const CamD& cam, const ss_cloud& cl, int64_t i, Projected& P) {
  project_geom(cam, cl, i, P);
  constexpr int K = (DEG + 1) * (DEG + 1);
  double basis[K];
  sh_basis<double>(DEG, P.dir[0], P.dir[1], P.dir[2], basis);
  double raw[3] = {0.5, 0.5, 0.5};
  const float* sh = cl.sh + i * 3 * K;
  if (K % 4 == 0 && (reinterpret_cast<uintptr_t>(cl.sh) & 15) == 0) {  // 3K floats as float4 (K = 4, 16)
#pragma unroll
    for (int j = 0; j < 3 * K / 4; ++j) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(sh) + j);
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) raw[(4 * j + t) % 3] += basis[(4 * j + t) / 3] * (double)e[t];
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) raw[c] += basis[k] * (double)sh[3 * k + c];
  }
  for (int c = 0; c < 3; ++c) P.raw[c] = raw[c];
}

// K4a: per-Gaussian projection; depth key (+inf when culled)
#ifndef SS_PP_BLOCKS
#define SS_PP_BLOCKS 4  // 64 registers: 4 CTAs per SM (measured 36 -> 34 us)
#endif
#ifndef SS_GB_BLOCKS
#define SS_GB_BLOCKS 4
#endif
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}

// Degree 3: the block's 256 SH rows (48 KB, contiguous) are copied into shared
// memory with cp.async at the start, so their latency hides under the fp64
// projection instead of stalling the colour evaluation after it.
constexpr int kPpPrefetchBytes = 256 * 48 * 4;
template <int DEG>
__global__ void __launch_bounds__(256, SS_PP_BLOCKS) preprocess_kernel(CamD cam, ss_cloud cl, Geom g) {
  constexpr int K = (DEG + 1) * (DEG + 1), RW = 3 * K;
  constexpr bool PF = DEG == 3;
  extern __shared__ __align__(16) float s_pf[];  // PF: [256][RW]
  __shared__ uint32_t s_hist[4][256];  // the depth sort's digit histograms
  const int64_t row0 = blockIdx.x * (int64_t)blockDim.x;
  const bool pf = PF && (reinterpret_cast<uintptr_t>(cl.sh) & 15) == 0;  // grid-uniform
  if (pf) {
    const int nv = (int)(min((int64_t)blockDim.x, cl.n - row0) * RW / 4);
    const float4* src = reinterpret_cast<const float4*>(cl.sh + row0 * RW);
    for (int v = threadIdx.x; v < nv; v += blockDim.x) cp_async16(s_pf + 4 * v, src + v);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int k = threadIdx.x; k < 1024; k += blockDim.x) (&s_hist[0][0])[k] = 0;
  __syncthreads();
  const int64_t i = row0 + threadIdx.x;
  bool vis = false;
  Projected P;
  if (i < cl.n) {
    if (i == 0) g.dev_counts[2] = cl.n;
    g.order[i] = (int32_t)i;  // sort input (4 passes: the input sits in the output buffers)
    const float* m = cl.means + 3 * i;
    // depth key, every operation rounded (no FMA contraction) in a fixed order,
    // ((R20 m0 + R21 m1) + R22 m2) + t2, so it is reproducible on the host; the
    // reference's own depth is a BLAS DGEMM (cameras.py:80) whose FMA use
    // depends on the CPU, which only matters for ties at the last ulp
    const double z = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(cam.R[2][0], (double)m[0]),
                                                   __dmul_rn(cam.R[2][1], (double)m[1])),
                                         __dmul_rn(cam.R[2][2], (double)m[2])),
                               cam.t[2]);
    uint32_t key = 0x7f800000u;  // +inf: culled (rasterizer.py:228)
    if (!(z > cam.near_clip)) {
      g.key_in[i] = __longlong_as_double(0x7ff0000000000000ll);
    } else {
      g.key_in[i] = z;
      // fp32 rounding is monotone, so sorting by the fp32 bits orders the fp64
      // depths up to ties, which depth_tie_kernel resolves
      key = __float_as_uint((float)z);
      atomicAdd(reinterpret_cast<unsigned long long*>(&g.dev_counts[0]), 1ull);
      if (pf) project_geom(cam, cl, i, P);
      else project_one<DEG>(cam, cl, i, P);
      vis = true;
    }
    g.key32[i] = key;
    bs_hist_add(s_hist, key, 32);
  }
  if (pf) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (vis) {  // the colour from the staged row, the same operation order as project_one
      double basis[K];
      sh_basis<double>(DEG, P.dir[0], P.dir[1], P.dir[2], basis);
      double raw[3] = {0.5, 0.5, 0.5};
      const float4* row = reinterpret_cast<const float4*>(s_pf + threadIdx.x * RW);
#pragma unroll
      for (int j = 0; j < RW / 4; ++j) {
        const float4 v = row[j];
        const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) raw[(4 * j + t) % 3] += basis[(4 * j + t) / 3] * (double)e[t];
      }
      for (int c = 0; c < 3; ++c) P.raw[c] = raw[c];
    }
  }
  if (vis) {
    g.g_mean[i] = make_double2(P.mean[0], P.mean[1]);
    g.g_conop[i] =
        make_double4(P.conic[0][0], P.conic[0][1] + P.conic[1][0], P.conic[1][1], P.op);
    // w: the unclipped-channel mask of clip(0.5 + SH, 0, 1) (sh.py:51-59) for the backward
    const int clip_mask = (P.raw[0] > 0.0 && P.raw[0] < 1.0) |
                          (P.raw[1] > 0.0 && P.raw[1] < 1.0) << 1 |
                          (P.raw[2] > 0.0 && P.raw[2] < 1.0) << 2;
    g.g_color[i] = make_float4((float)fmin(fmax(P.raw[0], 0.0), 1.0),
                               (float)fmin(fmax(P.raw[1], 0.0), 1.0),
                               (float)fmin(fmax(P.raw[2], 0.0), 1.0), (float)clip_mask);
    g.g_cov[i] = make_double2(P.cov2d[0][0], P.cov2d[1][1]);
  }
  __syncthreads();
  bs_hist_flush(s_hist, g.dsort.hist, 32);
}

// floor(v) // ts with Python floor-division semantics, clipped (rasterizer.py:142-145)
__device__ inline int tile_of(double v, int ts, int nt) {
  double f = floor(v);
  f = fmin(fmax(f, -4.0e18), 4.0e18);
  long long q = (long long)f;
  long long t = q >= 0 ? q / ts : -((-q + ts - 1) / ts);
  t = t < 0 ? 0 : (t > nt - 1 ? nt - 1 : t);
  return (int)t;
}

// K4b tie-break: survivors are sorted by their fp32 depth bits (stable, so
// index order within equal keys); runs of equal fp32 keys are re-sorted by
// (fp64 depth, index) so the order equals the stable fp64 sort
// (rasterizer.py:228-230).  Runs of up to kTieShort ranks (the common case) are
// insertion-sorted by the thread at their head; a longer run (a plane facing
// the camera puts every splat in one) is queued in shared memory and sorted by
// the whole CTA with a stable LSD radix sort over the fp64 depth's offset from
// the run minimum, so the cost stays linear in the run length.
constexpr int kTieShort = 32;
constexpr int kTieThreads = 256, kTieSteps = 4, kTieChunk = kTieThreads * kTieSteps;

// stable 4 x 8-bit LSD sort of order[r, e) by (fp64 depth bits - minimum bits);
// the run is in index order on entry, so equal depths keep index order
__device__ void tie_sort_run_cta(const Geom& g, int64_t r, int64_t e, uint64_t minb,
                                 uint32_t (*wh)[256], uint32_t* s_base, uint32_t* s_scan) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  int32_t* src = g.order + r;
  int32_t* dst = g.idx_in + r;  // the depth sort's ping-pong buffer, free after it
  const int64_t k = e - r;
  for (int pass = 0; pass < 4; ++pass) {
    const int sh = 8 * pass;
    s_base[tid] = 0;
    __syncthreads();
    for (int64_t i = tid; i < k; i += kTieThreads) {
      const uint64_t b = (uint64_t)__double_as_longlong(g.key_in[src[i]]) - minb;
      atomicAdd(&s_base[(b >> sh) & 255], 1u);
    }
    __syncthreads();
    {  // exclusive scan over the 256 digits (thread = digit)
      const uint32_t h = s_base[tid];
      uint32_t x = h;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_scan[warp] = x;
      __syncthreads();
      uint32_t w = 0;
      for (int j = 0; j < warp; ++j) w += s_scan[j];
      __syncthreads();
      s_base[tid] = x - h + w;
    }
    for (int64_t c = 0; c < k; c += kTieChunk) {
      for (int j = 0; j < kTieThreads / 32; ++j) wh[j][tid] = 0;
      __syncthreads();
      int32_t v[kTieSteps];
      uint32_t d[kTieSteps], rk[kTieSteps];
#pragma unroll
      for (int s2 = 0; s2 < kTieSteps; ++s2) {  // warp w owns [w*128, w*128+128) of the chunk
        const int64_t i = c + warp * (kTieSteps * 32) + s2 * 32 + lane;
        v[s2] = i < k ? src[i] : 0;
        d[s2] = i < k ? (uint32_t)((((uint64_t)__double_as_longlong(g.key_in[v[s2]]) - minb) >> sh) & 255)
                      : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d[s2]);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (i < k && lane == leader) {
          old = wh[warp][d[s2]];
          wh[warp][d[s2]] = old + __popc(peers);
        }
        rk[s2] = __shfl_sync(0xffffffffu, old, leader) + __popc(peers & lt);
        __syncwarp();
      }
      __syncthreads();
      {  // per digit: exclusive prefix over warps, chunk total into the base
        uint32_t cnt = 0;
#pragma unroll
        for (int j = 0; j < kTieThreads / 32; ++j) {
          const uint32_t t = wh[j][tid];
          wh[j][tid] = cnt;
          cnt += t;
        }
        __syncthreads();
#pragma unroll
        for (int s2 = 0; s2 < kTieSteps; ++s2)
          if (d[s2] < 256u) dst[s_base[d[s2]] + wh[warp][d[s2]] + rk[s2]] = v[s2];
        __syncthreads();
        s_base[tid] += cnt;
      }
      __syncthreads();
    }
    int32_t* t = src;
    src = dst;
    dst = t;
  }
}

__global__ void __launch_bounds__(kTieThreads) depth_tie_kernel(Geom g) {
  __shared__ uint32_t wh[kTieThreads / 32][256];
  __shared__ uint32_t s_base[256], s_scan[64];
  __shared__ int64_t s_long[kTieThreads];
  __shared__ int s_nlong;
  __shared__ unsigned long long s_min;
  __shared__ long long s_end;
  const int64_t V = g.dev_counts[0];
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (threadIdx.x == 0) s_nlong = 0;
  __syncthreads();
  if (r < V) {
    const uint32_t k = g.key32[r];
    if (!(r > 0 && g.key32[r - 1] == k) && r + 1 < V && g.key32[r + 1] == k) {
      int64_t e = r + 1;
      while (e < V && e - r <= kTieShort && g.key32[e] == k) ++e;
      if (e < V && g.key32[e] == k) {
        s_long[atomicAdd(&s_nlong, 1)] = r;  // longer than kTieShort: the CTA sorts it
      } else {
        for (int64_t a = r + 1; a < e; ++a) {  // insertion sort by (fp64 depth, index)
          const int32_t v = g.order[a];
          const double dv = g.key_in[v];
          int64_t b = a - 1;
          while (b >= r) {
            const int32_t u = g.order[b];
            const double du = g.key_in[u];
            if (du < dv || (du == dv && u < v)) break;
            g.order[b + 1] = u;
            --b;
          }
          g.order[b + 1] = v;
        }
      }
    }
  }
  __syncthreads();
  const int nlong = s_nlong;
  for (int j = 0; j < nlong; ++j) {  // block-uniform
    const int64_t h = s_long[j];
    const uint32_t k = g.key32[h];
    if (threadIdx.x == 0) {
      s_end = V;
      s_min = ~0ull;
    }
    __syncthreads();
    // run end: the first mismatching rank, found a CTA-width window at a time
    for (int64_t base = h + 1;; base += kTieThreads) {
      const int64_t i = base + threadIdx.x;
      if (i < V && g.key32[i] != k) atomicMin(&s_end, (long long)i);
      __syncthreads();
      if (s_end < base + kTieThreads || base + kTieThreads >= V) break;
    }
    const int64_t e = s_end;
    for (int64_t i = h + threadIdx.x; i < e; i += kTieThreads)
      atomicMin(&s_min, (unsigned long long)__double_as_longlong(g.key_in[g.order[i]]));
    __syncthreads();
    tie_sort_run_cta(g, h, e, s_min, wh, s_base, s_scan);
    __syncthreads();
  }
}

// ---- single-pass inclusive scan of per-rank int64 counts (offsets, band
// offsets): the producer kernel's block takes a logical id from a ticket (its
// predecessors are then running or done), scans its 256 counts, publishes the
// aggregate and resolves its exclusive prefix by a warp-wide decoupled
// look-back (32 predecessors per round trip).  Replaces a library scan (two
// launches) after each producer.
constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbVal = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ int64_t scan_logical_block(unsigned long long* lb, int64_t nb) {
  __shared__ int64_t s_bid;
  if (threadIdx.x == 0) s_bid = (int64_t)atomicAdd(lb + nb, 1ull);
  __syncthreads();
  return s_bid;
}

// inclusive prefix of v over all ranks before and including this thread's
__device__ int64_t scan_inclusive(int64_t v, int64_t bid, unsigned long long* lb) {
  __shared__ int64_t s_w[kScanThreads / 32];
  __shared__ int64_t s_excl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t t = lane < kScanThreads / 32 ? s_w[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kScanThreads / 32) s_w[lane] = t;  // inclusive warp totals
    const int64_t total = __shfl_sync(0xffffffffu, t, kScanThreads / 32 - 1);
    int64_t excl = 0;
    if (bid == 0) {
      if (lane == 0) atomicExch(lb, kLbInc | (unsigned long long)total);
    } else {
      if (lane == 0) atomicExch(lb + bid, kLbAgg | (unsigned long long)total);
      int64_t p = bid - 1;
      while (true) {
        const int64_t j = p - lane;
        const unsigned long long w = j >= 0 ? ld_volatile_u64(lb + j) : kLbInc;
        const uint32_t not_ready = __ballot_sync(0xffffffffu, (w & ~kLbVal) == 0);
        const uint32_t inc = __ballot_sync(0xffffffffu, (w & kLbInc) != 0);
        const int nr = not_ready ? __ffs(not_ready) - 1 : 32;
        const int fi = inc ? __ffs(inc) - 1 : 32;
        const int upto = fi < nr ? fi + 1 : nr;  // lanes [0, upto) are summed
        int64_t val = lane < upto ? (int64_t)(w & kLbVal) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (fi < nr) break;
        p -= nr;  // re-poll from the first predecessor that has not published
      }
      if (lane == 0) atomicExch(lb + bid, kLbInc | (unsigned long long)(excl + total));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  return s_excl + (warp > 0 ? s_w[warp - 1] : 0) + x;
}

// K4b/K4c: gather per-rank records, tile rectangle and its count
// (rank_count), then the inclusive scan of the counts into offsets[1..n]
// The per-Gaussian inputs of a rank (gathered by id in depth order)
struct RankIn {
  int gid;
  double2 m, cv;
  double4 co;
  float4 gc;
};
__device__ __forceinline__ void rank_load(const Geom& g, int64_t r, int64_t n, int64_t V,
                                          RankIn& in) {
  in.gid = r < n ? g.order[r] : 0;
  if (r < V) {
    in.m = g.g_mean[in.gid];
    in.co = g.g_conop[in.gid];
    in.gc = g.g_color[in.gid];
    in.cv = g.g_cov[in.gid];
  }
}
__device__ __forceinline__ int64_t rank_count(const CamD& cam, const ss_raster_settings& s,
                                              int64_t r, int64_t V, Geom& g, const RankIn& in) {
  g.rank_of[in.gid] = (int32_t)r;
  if (r >= V) return 0;
  const int gid = in.gid;
  const double2 m = in.m;
  const double4 co = in.co;
  g.r_mean[r] = m;
  g.r_conop_d[r] = co;
  g.r_conop[r] = make_float4((float)co.x, (float)co.y, (float)co.z, (float)co.w);
  // log2 G = A dx^2 + B dx dy + C dy^2; a pixel with log2 G below log2(skip (1 - 2e-4) / op)
  // has alpha < skip_alpha beyond any fp32 rounding (blend fast reject)
  constexpr double kq = -0.72134752044448170368;  // -0.5 log2(e)
  const double qthr = s.skip_alpha > 0.0 ? log2(s.skip_alpha * (1.0 - 2e-4) / co.w) : -1e30;
  g.r_q[r] = make_float4((float)(kq * co.x), (float)(kq * co.y), (float)(kq * co.z), (float)qthr);
  const float4 gc = in.gc;
  g.r_color[r] = make_float4(gc.x, gc.y, gc.z, (float)co.w);  // w: opacity
  const int ts = s.tile_size;
  const int ntx = (cam.W + ts - 1) / ts, nty = (cam.H + ts - 1) / ts;
  int4 rect;
  bool vis;
  if (s.skip_alpha > 0.0) {  // rasterizer.py:132-148
    const double ratio = fmax(co.w / s.skip_alpha, 1.0);
    const double r2 = sqrt(fmax(9.0, 2.0 * log(ratio)));
    const double2 cv = in.cv;
    const double hx = r2 * sqrt(fmax(cv.x, 0.0));
    const double hy = r2 * sqrt(fmax(cv.y, 0.0));
    const double xl = m.x - hx, xh = m.x + hx, yl = m.y - hy, yh = m.y + hy;
    rect = make_int4(tile_of(xl, ts, ntx), tile_of(xh, ts, ntx), tile_of(yl, ts, nty),
                     tile_of(yh, ts, nty));
    vis = !((xh < 0) || (xl > cam.W - 1) || (yh < 0) || (yl > cam.H - 1));
    // co.y = c01 + c10: the minimiser of the form along x = const is dy = -co.y dx / (2 c11)
    g.r_cull[r] = make_double4(2.0 * log(co.w / s.skip_alpha), -co.y / (2.0 * co.z),
                               -co.y / (2.0 * co.x), 0.0);
  } else {  // skip = 0: every tile (rasterizer.py:149-154)
    rect = make_int4(0, ntx - 1, 0, nty - 1);
    vis = true;
  }
  g.r_rect[r] = rect;
  return vis ? (int64_t)(rect.y - rect.x + 1) * (rect.w - rect.z + 1) : 0;
}

__global__ void __launch_bounds__(kScanThreads) rank_kernel(CamD cam, ss_raster_settings s,
                                                             int64_t n, Geom g) {
  // kScanRanks ranks per thread for the gathers (coalesced: rank base + k * 256 + tid),
  // then each thread scans kScanRanks consecutive counts from shared memory
  __shared__ int64_t s_cnt[kScanThreads * kScanRanks];
  const int64_t bid = scan_logical_block(g.scan_lb, g.scan_blocks);
  const int64_t base = bid * (kScanThreads * kScanRanks);
  const int64_t V = g.dev_counts[0];
  // every rank's gathers in flight before any store (the Geom pointers may alias)
  RankIn in[kScanRanks];
#pragma unroll
  for (int k = 0; k < kScanRanks; ++k)
    rank_load(g, base + k * kScanThreads + threadIdx.x, n, V, in[k]);
#pragma unroll
  for (int k = 0; k < kScanRanks; ++k) {
    const int64_t r = base + k * kScanThreads + threadIdx.x;
    s_cnt[k * kScanThreads + threadIdx.x] = r < n ? rank_count(cam, s, r, V, g, in[k]) : 0;
  }
  __syncthreads();
  int64_t c[kScanRanks], sum = 0;
#pragma unroll
  for (int k = 0; k < kScanRanks; ++k) c[k] = (sum += s_cnt[threadIdx.x * kScanRanks + k]);
  const int64_t excl = scan_inclusive(sum, bid, g.scan_lb) - sum;
  const int64_t r0 = base + threadIdx.x * kScanRanks;
#pragma unroll
  for (int k = 0; k < kScanRanks; ++k) {
    if (r0 + k < n) g.offsets[r0 + k + 1] = excl + c[k];
    if (r0 + k == n - 1) g.dev_counts[1] = excl + c[k];
  }
  if (bid == 0 && threadIdx.x == 0) g.offsets[0] = 0;
}

__global__ void finish_counts_kernel(Geom g, int64_t n) {
  // inclusive scan was written to offsets[1..n]; offsets[0] = 0; pairs = offsets[n]
  g.offsets[0] = 0;
  g.dev_counts[1] = n > 0 ? g.offsets[n] : 0;
}

// ---- tile-row bands: a view whose pairs exceed the bin workspace is binned
// and blended one band of tile rows at a time (host-driven, synchronous)
__global__ void row_pairs_kernel(int64_t n, Geom g, int nty) {
  extern __shared__ unsigned long long s_rows[];
  for (int i = threadIdx.x; i < nty; i += blockDim.x) s_rows[i] = 0;
  __syncthreads();
  const int64_t V = g.dev_counts[0];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < min(n, V);
       r += (int64_t)gridDim.x * blockDim.x) {
    if (g.offsets[r + 1] == g.offsets[r]) continue;  // not visible
    const int4 rc = g.r_rect[r];
    const unsigned long long wx = (unsigned long long)(rc.y - rc.x + 1);
    for (int ty = rc.z; ty <= rc.w; ++ty) atomicAdd(&s_rows[ty], wx);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nty; i += blockDim.x)
    if (s_rows[i]) atomicAdd(&g.row_pairs[i], s_rows[i]);
}

// pairs of each rank inside tile rows [ty_lo, ty_hi) (band_off[r], scanned later)
// and their inclusive scan into band_off[1..n], the band's total in dev_counts[3]
__global__ void __launch_bounds__(kScanThreads) band_counts_kernel(int64_t n, Geom g, int ty_lo,
                                                                   int ty_hi) {
  const int64_t bid = scan_logical_block(g.scan_lb, g.scan_blocks);
  const int64_t r = bid * kScanThreads + threadIdx.x;
  int64_t c = 0;
  if (r < n && r < g.dev_counts[0] && g.offsets[r + 1] > g.offsets[r]) {
    const int4 rc = g.r_rect[r];
    const int rows = min(rc.w, ty_hi - 1) - max(rc.z, ty_lo) + 1;
    c = rows > 0 ? (int64_t)(rc.y - rc.x + 1) * rows : 0;
  }
  const int64_t incl = scan_inclusive(c, bid, g.scan_lb);
  if (r < n) g.band_off[r + 1] = incl;
  if (r == 0) g.band_off[0] = 0;
  if (r == n - 1) g.dev_counts[3] = incl;
}

// K4c (render path) tile cull:
// near-camera splats can cover thousands of tiles).  The owning rank is the last
// r with offsets[r] <= j (zero-count ranks are skipped by construction).
// Tile-level cull (render path only): a (splat, tile) pair whose alpha stays
// below skip_alpha at every pixel centre of the tile contributes nothing to
// the image, the loss or any gradient (rasterizer.py:198-199), so its key is
// replaced by the sentinel ntiles and it sorts past every tile list.  The test
// bounds alpha by the minimum of the fp64 Mahalanobis form over the tile's
// pixel-centre rectangle (a relaxation of the discrete minimum: conservative).
__device__ inline bool splat_misses_tile(const double2 m, const double4 co, const double4 cl,
                                         double xa, double xb, double ya, double yb) {
  const double lx = xa - m.x, hx = xb - m.x, ly = ya - m.y, hy = yb - m.y;
  if (lx <= 0.0 && hx >= 0.0 && ly <= 0.0 && hy >= 0.0) return cl.x < -2e-6;
  auto q = [&](double dx, double dy) { return co.x * dx * dx + co.y * dx * dy + co.z * dy * dy; };
  auto clampd = [](double v, double a, double b) { return fmin(fmax(v, a), b); };
  double qmin = 1e300;
  // edges x = const: minimise over dy (dy* = cl.y dx); edges y = const: dx* = cl.z dy
  qmin = fmin(qmin, q(lx, clampd(cl.y * lx, ly, hy)));
  qmin = fmin(qmin, q(hx, clampd(cl.y * hx, ly, hy)));
  qmin = fmin(qmin, q(clampd(cl.z * ly, lx, hx), ly));
  qmin = fmin(qmin, q(clampd(cl.z * hy, lx, hx), hy));
  // op exp(-qmin / 2) < skip (1 - 1e-6)  <=>  qmin > 2 ln(op / skip) + 2e-6
  return qmin > cl.x + 2e-6;
}

// K4c: emit (tile id, rank) in rank order, one thread per pair (load-balanced:
// near-camera splats can cover thousands of tiles).  The owning rank is the last
// r with offsets[r] <= j; a CTA narrows the search range once per 1024 pairs.
__device__ inline int64_t owner_rank(const int64_t* __restrict__ off, int64_t lo, int64_t hi,
                                     int64_t j) {  // offsets[lo] <= j < offsets[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (off[mid] <= j) lo = mid; else hi = mid;
  }
  return lo;
}

// Block-parallel form (all threads call it, block-uniform result): each round
// the threads test blockDim.x evenly spaced ranks and the bracket shrinks by
// that factor, so a search over 250k ranks takes 3 rounds of one load each
// instead of 18 dependent loads on one thread.
__device__ inline int64_t block_owner_rank(const int64_t* __restrict__ off, int64_t lo,
                                           int64_t hi, int64_t j) {  // off[lo] <= j < off[hi]
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + blockDim.x - 1) / blockDim.x;
    const int64_t r = lo + (int64_t)threadIdx.x * step;
    const int cnt = __syncthreads_count(r < hi && off[r] <= j);  // a prefix of the threads
    lo += (int64_t)(cnt - 1) * step;
    hi = min(lo + step, hi);
  }
  return lo;
}

// One thread per pair, chunks of 1024 pairs per CTA pass.  The owner of every
// pair of a chunk comes from a block max-scan instead of a per-pair binary
// search: each rank starting inside the chunk marks its first pair, the chunk's
// first pair is owned by the rank found once per chunk (block_owner_rank), and
// the inclusive max-scan carries the owners forward (zero-count ranks share
// their successor's start and lose the max).
__global__ void __launch_bounds__(256) duplicate_kernel(int ntx, int64_t n, Geom g, Bins b,
                                                        uint32_t* kdst, uint32_t* vdst,
                                                        uint32_t* status, int cull, int ts, int W,
                                                        int H, uint32_t sentinel, int key_bits,
                                                        const int64_t* __restrict__ offs,
                                                        const int64_t* __restrict__ d_count,
                                                        int ty_lo) {
  constexpr int CH = 1024, NTH = 256, PER = CH / NTH;
  __shared__ int s_owner[CH];
  __shared__ int s_wmax[NTH / 32];
  __shared__ uint32_t s_hist[2][256];  // binsort digit histograms of the emitted keys
  for (int i = threadIdx.x; i < 512; i += blockDim.x) (&s_hist[0][0])[i] = 0;
  const int64_t count = *d_count;
  if (count > b.capacity && blockIdx.x == 0 && threadIdx.x == 0 && status)
    atomicOr(status, SS_FLAG_OVERFLOW);
  const int64_t pairs = min(count, b.capacity);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t j0 = (int64_t)blockIdx.x * CH; j0 < pairs; j0 += (int64_t)gridDim.x * CH) {
    __syncthreads();  // the previous chunk is done with s_owner
    const int cn = (int)min((int64_t)CH, pairs - j0);
    const int64_t rlo = block_owner_rank(offs, 0, n, j0);
    const int64_t rhi = block_owner_rank(offs, rlo, n, j0 + cn - 1);
    for (int i = threadIdx.x; i < CH; i += NTH) s_owner[i] = i == 0 ? (int)rlo : -1;
    __syncthreads();
    for (int64_t r = rlo + 1 + threadIdx.x; r <= rhi; r += NTH)
      atomicMax(&s_owner[(int)(offs[r] - j0)], (int)r);
    __syncthreads();
    // inclusive max-scan: PER consecutive entries per thread, then the warps
    int v[PER], m = -1;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      m = max(m, s_owner[threadIdx.x * PER + q]);
      v[q] = m;
    }
    int x = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x = max(x, y);
    }
    if (lane == 31) s_wmax[warp] = x;
    const int prev_lane = __shfl_up_sync(0xffffffffu, x, 1);
    __syncthreads();
    int carry = lane == 0 ? -1 : prev_lane;
    for (int w = 0; w < warp; ++w) carry = max(carry, s_wmax[w]);
#pragma unroll
    for (int q = 0; q < PER; ++q) s_owner[threadIdx.x * PER + q] = max(carry, v[q]);
    __syncthreads();
    for (int i = threadIdx.x; i < cn; i += NTH) {
      const int64_t j = j0 + i;
      const int lo = s_owner[i];
      const int4 rc = g.r_rect[lo];
      const int wx = rc.y - rc.x + 1;
      const int local = (int)(j - offs[lo]);  // < tiles per view
      // local / wx and local % wx (local < 2^22: one float estimate, one fix-up)
      int qy = (int)__fdividef((float)local, (float)wx);
      int qx = local - qy * wx;
      if (qx < 0) qx += wx, --qy;
      else if (qx >= wx) qx -= wx, ++qy;
      const int ty = max(rc.z, ty_lo) + qy, tx = rc.x + qx;
      uint32_t key = (uint32_t)(ty * ntx + tx);
      // the cull test pays off for splats spanning several tiles; it never
      // changes a result (culled pairs have alpha < skip at every pixel)
      if (cull && wx * (rc.w - rc.z + 1) > 2) {
        const double xa = tx * ts, xb = min(tx * ts + ts, W) - 1, ya = ty * ts,
                     yb = min(ty * ts + ts, H) - 1;
        if (splat_misses_tile(g.r_mean[lo], g.r_conop_d[lo], g.r_cull[lo], xa, xb, ya, yb))
          key = sentinel;
      }
      kdst[j] = key;
      vdst[j] = (uint32_t)lo;
      bs_hist_add(s_hist, key, key_bits);
    }
  }
  __syncthreads();
  bs_hist_flush(s_hist, b.sort.hist, key_bits);
}

// Per-tile [start, end) of the sorted keys: four keys per thread (one 16-byte
// load), the neighbours across threads by warp shuffles (only the warp's end
// lanes read past their own keys)
__global__ void ranges_kernel(const int64_t* __restrict__ d_pairs, int64_t cap,
                              const uint32_t* __restrict__ keys, int2* ranges, uint32_t ntiles) {
  const int64_t pairs = min(*d_pairs, cap);
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane) * 4; i0 < pairs;
       i0 += stride) {  // warp-uniform: i0 = the warp's first key
    const int64_t i = i0 + 4 * lane;
    uint32_t k[4];
    if (i + 3 < pairs) {  // keys is 16-byte aligned (Carve), i a multiple of 4
      const uint4 v = *reinterpret_cast<const uint4*>(keys + i);
      k[0] = v.x, k[1] = v.y, k[2] = v.z, k[3] = v.w;
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) k[t] = i + t < pairs ? keys[i + t] : 0xffffffffu;
    }
    uint32_t prev = __shfl_up_sync(0xffffffffu, k[3], 1);
    uint32_t next = __shfl_down_sync(0xffffffffu, k[0], 1);
    if (lane == 0) prev = i > 0 && i - 1 < pairs ? keys[i - 1] : 0xffffffffu;
    if (lane == 31) next = i + 4 < pairs ? keys[i + 4] : 0xffffffffu;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t e = i + t;
      if (e >= pairs) break;
      const uint32_t kk = k[t];
      if (kk >= ntiles) continue;  // culled pairs (sentinel key) sort past the last tile
      const uint32_t kp = t == 0 ? prev : k[t - 1];
      const uint32_t kn = t == 3 ? next : k[t + 1];
      if (e == 0 || kp != kk) ranges[kk].x = (int)e;
      if (e == pairs - 1 || kn != kk) ranges[kk].y = (int)(e + 1);
    }
  }
}

struct ZeroRegions {
  static constexpr int kMax = 10;
  uint8_t* p[kMax];
  int64_t bytes[kMax];
  int n;
};
__global__ void __launch_bounds__(256) zero_regions_kernel(ZeroRegions z) {
  for (int r = 0; r < z.n; ++r) {
    uint8_t* p = z.p[r];
    const int64_t b = z.bytes[r];
    const int64_t n16 = (reinterpret_cast<uintptr_t>(p) & 15) == 0 ? b >> 4 : 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16;
         i += (int64_t)gridDim.x * blockDim.x)
      reinterpret_cast<uint4*>(p)[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int64_t i = n16 * 16 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < b;
         i += (int64_t)gridDim.x * blockDim.x)
      p[i] = 0;
  }
}

// Block -> tile map of the blends, heaviest tiles first (longest-processing-
// time order): the per-tile work ranges over orders of magnitude, and in
// index order the last wave's heavy tiles leave most SMs idle.  Tiles are
// bucketed by 4 log2(pairs) (one CTA: histogram, descending scan, scatter);
// the order inside a bucket is free (it changes no result).
__global__ void __launch_bounds__(1024) tile_order_kernel(int ntiles, const int2* __restrict__ ranges,
                                                          int32_t* __restrict__ order) {
  constexpr int NB = 64, PER = 8;  // up to 8192 tiles from registers, beyond that re-read
  __shared__ uint32_t s_hist[NB];
  auto bucket = [](int c) { return c <= 0 ? 0 : min(NB - 1, 1 + (int)(4.f * __log2f((float)c))); };
  if (threadIdx.x < NB) s_hist[threadIdx.x] = 0;
  int b[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int t = threadIdx.x + k * 1024;
    b[k] = -1;
    if (t < ntiles) {
      const int2 r = ranges[t];
      b[k] = bucket(r.y - r.x);
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PER; ++k)
    if (b[k] >= 0) atomicAdd(&s_hist[b[k]], 1u);
  for (int t = threadIdx.x + PER * 1024; t < ntiles; t += blockDim.x) {
    const int2 r = ranges[t];
    atomicAdd(&s_hist[bucket(r.y - r.x)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // descending exclusive scan of the 64 buckets
    const int l = threadIdx.x;
    const uint32_t hi = s_hist[NB - 1 - l], lo = s_hist[NB / 2 - 1 - l];  // bucket 63 - l, 31 - l
    uint32_t x = hi;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (l >= o) x += y;
    }
    const uint32_t tot_hi = __shfl_sync(0xffffffffu, x, 31);
    uint32_t z = lo;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (l >= o) z += y;
    }
    s_hist[NB - 1 - l] = x - hi;
    s_hist[NB / 2 - 1 - l] = tot_hi + z - lo;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PER; ++k)
    if (b[k] >= 0) order[atomicAdd(&s_hist[b[k]], 1u)] = threadIdx.x + k * 1024;
  for (int t = threadIdx.x + PER * 1024; t < ntiles; t += blockDim.x) {
    const int2 r = ranges[t];
    order[atomicAdd(&s_hist[bucket(r.y - r.x)], 1u)] = t;
  }
}

// duplicate -> stable tile sort -> per-tile ranges, all driven by the device
// count *d_count of the pairs listed by `offs` (the whole view, or one band of
// tile rows starting at ty_lo)
static int bin_pairs(const ss_camera* cam, const ss_raster_settings* s, int64_t n, Geom& g,
                     Bins& b, uint32_t* status, int cull, cudaStream_t st,
                     const int64_t* offs = nullptr, const int64_t* d_count = nullptr,
                     int ty_lo = 0) {
  const int ntx = ntiles_x(cam, s), nty = ntiles_y(cam, s);
  const int64_t ntiles = (int64_t)ntx * nty;
  const bool whole = !offs;  // the whole view (not one band of tile rows)
  if (!offs) offs = g.offsets, d_count = g.dev_counts + 1;
  cull = cull && s->skip_alpha > 0.0;
  const int kb = key_bits(cull ? ntiles + 1 : ntiles);
  const bool two = binsort_passes(kb) == 2;
  // the bin workspace can be replaced between raster_begin and here (the host
  // sizes it from the pair count), and bands reuse it: its clears always run
  PrezeroScope scope(false);
  {  // ranges, the sort's histograms (duplicate_kernel fills them) and look-back
     // words: one kernel instead of three memset nodes
    ZeroRegions z{};
    z.p[0] = reinterpret_cast<uint8_t*>(g.ranges), z.bytes[0] = ntiles * (int64_t)sizeof(int2);
    z.p[1] = reinterpret_cast<uint8_t*>(b.sort.hist), z.bytes[1] = (4 * 256 + 64) * sizeof(uint32_t);
    z.p[2] = reinterpret_cast<uint8_t*>(b.sort.status);
    z.bytes[2] = (int64_t)binsort_passes(kb) * b.sort.max_blocks * 256 * sizeof(uint32_t);
    z.n = 3;
    zero_regions_kernel<<<148 * 4, 256, 0, st>>>(z);
    SS_CHECK_LAUNCH("zero_regions_kernel");
  }
  prof_begin(PH_DUPLICATE, st);
  const unsigned dgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(b.capacity, 1024),
                                                                         148 * 8));
  duplicate_kernel<<<dgrid, 256, 0, st>>>(ntx, n, g, b, two ? b.keys_out : b.keys_in,
                                          two ? b.vals_out : b.vals_in, status, cull, s->tile_size,
                                          cam->width, cam->height, (uint32_t)ntiles, kb, offs,
                                          d_count, ty_lo);
  SS_CHECK_LAUNCH("duplicate_kernel");
  prof_end(PH_DUPLICATE, st);
  prof_begin(PH_TILE_SORT, st);
  SS_TRY(binsort_run(b.sort, b.keys_in, b.vals_in, b.keys_out, b.vals_out, d_count, b.capacity, kb,
                     st, /*hist_ready=*/true));
  g_launches.fetch_add(two ? 2 : 1);
  prof_end(PH_TILE_SORT, st);
  prof_begin(PH_RANGES, st);
  ranges_kernel<<<stride_grid(b.capacity), 256, 0, st>>>(d_count, b.capacity, b.keys_out,
                                                         g.ranges, (uint32_t)ntiles);
  SS_CHECK_LAUNCH("ranges_kernel");
  if (whole) {
    tile_order_kernel<<<1, 1024, 0, st>>>((int)ntiles, g.ranges, g.tile_order);
    SS_CHECK_LAUNCH("tile_order_kernel");
  }
  prof_end(PH_RANGES, st);
  return SS_OK;
}

// Bands of tile rows whose pairs fit `cap` (host side, after raster_begin):
// per-row pair totals, then a greedy split.  Synchronises the stream.
static int plan_bands(const ss_camera* cam, const ss_raster_settings* s, int64_t n, Geom& g,
                      int64_t cap, std::vector<int2>& bands, cudaStream_t st) {
  const int nty = ntiles_y(cam, s);
  SS_CUDA(cudaMemsetAsync(g.row_pairs, 0, nty * sizeof(unsigned long long), st));
  row_pairs_kernel<<<stride_grid(n), 256, nty * sizeof(unsigned long long), st>>>(n, g, nty);
  SS_CHECK_LAUNCH("row_pairs_kernel");
  std::vector<unsigned long long> rows(nty);
  SS_CUDA(cudaMemcpyAsync(rows.data(), g.row_pairs, nty * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaStreamSynchronize(st));
  bands.clear();
  int lo = 0;
  unsigned long long acc = 0;
  for (int ty = 0; ty < nty; ++ty) {
    if (rows[ty] > (unsigned long long)cap) {
      set_error("one tile row holds more pairs than the bin workspace");
      return SS_ERR_CAPACITY;
    }
    if (acc + rows[ty] > (unsigned long long)cap) {
      bands.push_back(make_int2(lo, ty));
      lo = ty;
      acc = 0;
    }
    acc += rows[ty];
  }
  bands.push_back(make_int2(lo, nty));
  return SS_OK;
}

// list the pairs of band [ty_lo, ty_hi) (band_off, dev_counts[3]) and bin them
static int bin_band(const ss_camera* cam, const ss_raster_settings* s, int64_t n, Geom& g, Bins& b,
                    uint32_t* status, int cull, int2 band, cudaStream_t st) {
  SS_CUDA(cudaMemsetAsync(g.scan_lb, 0, (g.scan_blocks + 1) * sizeof(unsigned long long), st));
  SS_CUDA(cudaMemsetAsync(g.dev_counts + 3, 0, sizeof(int64_t), st));
  if (n > 0) {
    band_counts_kernel<<<(unsigned)g.scan_blocks, kScanThreads, 0, st>>>(n, g, band.x, band.y);
    SS_CHECK_LAUNCH("band_counts_kernel");
  }
  return bin_pairs(cam, s, n, g, b, status, cull, st, g.band_off, g.dev_counts + 3, band.x);
}

// ------------------------------------------------------------------ blend
struct BlendParams {
  int W, H, ntx;
  float clamp, skip, stop;
  double clamp_d, skip_d, stop_d;
  float bg[3];
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- the tile-centred log2 form
// For a splat staged in a tile, with D = (tile centre) - mean (float64) and a
// pixel at offset d from the tile centre, the log2 Gaussian is exactly
//   lg(d) = lg0 + gx dx + gy dy + A dx^2 + B dx dy + C dy^2,
// lg0 = k D^T Q D, (gx, gy) = 2 k Q D, (A, B, C) = k (c00, c01 + c10, c11),
// k = -0.5 log2(e): the large mean offset lives in lg0 and g, evaluated in
// float64 once per (splat, tile) at staging, so the per-pixel fp32 evaluation
// (five FMAs on per-thread constants d, d^2) carries no cancellation even for
// splats whose mean lies 1e5 pixels away (a Gaussian at the near plane).
//
// Alpha decisions: rank_kernel sets the reject threshold
// thr = log2(skip (1 - 2e-4) / op); with the exact lg, a pair with lg < thr has
// alpha below skip and a pair with lg >= thr + kNearBand (= log2(skip (1 + 1e-4)
// / op)) alpha above it, beyond the ex2.approx error.  The fp32 lg is off by at
// most `band` (below), so pairs with lg in [thr - band, thr + kNearBand + band)
// take the float64 decision (a rare, per-thread branch) and every include /
// skip decision equals the float64 reference's (rasterizer.py:198-199).
constexpr float kNearBand = 4.3284e-4f;  // log2(1 + 1e-4) - log2(1 - 2e-4), rounded up

// One staged splat of a blend batch: everything the inner loop reads (64 B:
// three vector loads per splat, the rank only on rare paths)
struct __align__(16) SplatRec {
  float4 L;    // lg0, gx, gy, lo: reject below lo = thr - band
  float4 Q;    // A, B, C, hi: float64 decision below hi = thr + kNearBand + band
  float4 col;  // rgb, opacity
  int rank, pad0, pad1, pad2;
};

#ifndef SS_FWD_PPT16
#define SS_FWD_PPT16 2
#endif
#ifndef SS_BWD_PPT16
#define SS_BWD_PPT16 4
#endif
template <int TS, bool BWD = false>
struct BlendShape {
  // 16x16 tiles: several pixels per thread (whole rows per warp), which divides
  // the per-splat shared-memory loads, loop overhead and (backward) warp
  // reductions per pixel
  static constexpr int P16 = BWD ? SS_BWD_PPT16 : SS_FWD_PPT16;
  static constexpr int NT = TS == 16 ? 256 / P16 : (TS * TS <= 256 ? TS * TS : 256);
  static constexpr int PPT = TS * TS / NT;
};

template <int TS>
__device__ __forceinline__ void stage_splat(const Geom& g, int r, int x0, int y0, SplatRec& rec) {
  constexpr double c0 = 0.5 * (TS - 1);
  constexpr double kq = -0.72134752044448170368;  // -0.5 log2(e)
  const double2 m = g.r_mean[r];
  const double4 c = g.r_conop_d[r];  // c00, c01 + c10, c11, opacity
  const float4 q = g.r_q[r];         // (float) k (c00, c01 + c10, c11), thr
  const double dx = ((double)x0 + c0) - m.x, dy = ((double)y0 + c0) - m.y;
  const float lg0 = (float)(kq * (c.x * dx * dx + c.y * dx * dy + c.z * dy * dy));
  const float gx = (float)(kq * (2.0 * c.x * dx + c.y * dy));
  const float gy = (float)(kq * (c.y * dx + 2.0 * c.z * dy));
  // band = bound of |lg_fp32 - lg| over the tile: coefficient rounding (1 eps)
  // + five rounded FMAs whose partial sums are all bounded by S (5 eps), with
  // headroom: 8 eps
  constexpr float h = (float)c0;
  const float S = fabsf(lg0) + (fabsf(gx) + fabsf(gy)) * h +
                  (fabsf(q.x) + fabsf(q.y) + fabsf(q.z)) * h * h;
  const float band = 4.8e-7f * S + 1e-30f;
  rec.L = make_float4(lg0, gx, gy, q.w - band);
  rec.Q = make_float4(q.x, q.y, q.z, q.w + (kNearBand + band));
  rec.col = g.r_color[r];
  rec.rank = r;
}

// per-thread pixel constants: offsets from the tile centre (k + 1/2, exact)
template <int TS, int PPT>
struct PixelOffsets {
  float dx[PPT], dy[PPT];
  __device__ __forceinline__ void init(int t);
  // lg = (A dx + B dy + gx) dx + (C dy + gy) dy + lg0: five FMAs
  __device__ __forceinline__ float lg(const float4& L, const float4& Q, int p) const {
    const float t1 = fmaf(Q.y, dy[p], fmaf(Q.x, dx[p], L.y));
    const float t2 = fmaf(Q.z, dy[p], L.z);
    return fmaf(t2, dy[p], fmaf(t1, dx[p], L.x));
  }
  // every pixel's lg, two pixels per packed FMA (FFMA2 with the splat's
  // coefficients as broadcast scalars): the same five roundings per pixel
  __device__ __forceinline__ void lg_all(const float4& L, const float4& Q, float (&out)[PPT]) const {
    if constexpr (PPT % 2 == 0) {
      const float2 qx = make_float2(Q.x, Q.x), qy = make_float2(Q.y, Q.y), qz = make_float2(Q.z, Q.z);
      const float2 lx = make_float2(L.x, L.x), ly = make_float2(L.y, L.y), lz = make_float2(L.z, L.z);
#pragma unroll
      for (int p = 0; p < PPT; p += 2) {
        const float2 ddx = make_float2(dx[p], dx[p + 1]), ddy = make_float2(dy[p], dy[p + 1]);
        const float2 t1 = __ffma2_rn(qy, ddy, __ffma2_rn(qx, ddx, ly));
        const float2 t2 = __ffma2_rn(qz, ddy, lz);
        const float2 r = __ffma2_rn(t2, ddy, __ffma2_rn(t1, ddx, lx));
        out[p] = r.x;
        out[p + 1] = r.y;
      }
    } else {
#pragma unroll
      for (int p = 0; p < PPT; ++p) out[p] = lg(L, Q, p);
    }
  }
};

__device__ __noinline__ float alpha_f64(const BlendParams& bp, const Geom& g, int rank, float px,
                                        float py) {
  const double2 m = g.r_mean[rank];
  const double4 c = g.r_conop_d[rank];
  const double ddx = (double)px - m.x, ddy = (double)py - m.y;
  const double mh = c.x * ddx * ddx + c.y * ddx * ddy + c.z * ddy * ddy;
  const double ad = fmin(bp.clamp_d, c.w * exp(-0.5 * mh));
  return ad < bp.skip_d ? 0.f : fmaxf((float)ad, bp.skip);
}


// Pixel p of thread t: each warp owns a contiguous run of 32 * PPT pixels of
// the tile (whole rows), or with two pixels per thread on 16x16 tiles an 8x8
// quadrant (fewer splats touch a quadrant than a 16x4 strip, so more
// warp-uniform skips; SS_QUAD=0 restores the strips).
#ifndef SS_QUAD
#define SS_QUAD 1
#endif
template <int TS, int PPT>
__device__ __forceinline__ int tile_pixel(int t, int p) {
  if (SS_QUAD && TS == 16 && PPT == 2) {  // warp w: the 8x8 quadrant w
    const int w = t >> 5, l = t & 31;
    return ((w >> 1) * 8 + p * 4 + (l >> 3)) * 16 + (w & 1) * 8 + (l & 7);
  }
  return (t >> 5) * (32 * PPT) + p * 32 + (t & 31);
}

template <int TS, int PPT>
__device__ __forceinline__ void PixelOffsets<TS, PPT>::init(int t) {
  constexpr float c0 = 0.5f * (TS - 1);
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int li = tile_pixel<TS, PPT>(t, p);
    dx[p] = (float)(li % TS) - c0;
    dy[p] = (float)(li / TS) - c0;
  }
}

// TOUCH = false: the Stage-1 path, fp32 with the float64 decision band above.
// TOUCH = true (the public rasterize_forward, which also returns the per-
// Gaussian touch counts, rasterizer.py:279): every pair in float64 exactly as
// the reference evaluates it (maha, exp, alpha, T_before and the stop test), so
// the counts of weight = alpha T_before > 0 are the reference's.
template <int TS, bool TOUCH>
__global__ void __launch_bounds__(BlendShape<TS>::NT) blend_fwd_kernel(
    BlendParams bp, Geom g, const uint32_t* __restrict__ vals, float* __restrict__ image,
    float* __restrict__ alpha_map, int32_t* __restrict__ touch, int tile0) {
  constexpr int NT = BlendShape<TS>::NT, PPT = BlendShape<TS>::PPT;
  __shared__ SplatRec s_sp[NT];
  __shared__ double2 s_md[TOUCH ? NT : 1];  // float64 mean (TOUCH)
  __shared__ double4 s_cd[TOUCH ? NT : 1];  // float64 conic (c00, c01 + c10, c11) + opacity
  __shared__ int s_touch[TOUCH ? NT : 1];
  // tile0 < 0: the whole view in tile_order (heaviest first); else a band
  const int tile = tile0 >= 0 ? tile0 + (int)blockIdx.x : g.tile_order[blockIdx.x];
  const int x0 = (tile % bp.ntx) * TS, y0 = (tile / bp.ntx) * TS;
  const int2 range = g.ranges[tile];
  PixelOffsets<TS, PPT> po;
  po.init(threadIdx.x);
  // per-pixel transmittance and colour as register pairs (pixels 2q, 2q + 1),
  // so the update below runs two pixels per packed FMA
  float2 TT[(PPT + 1) / 2], CC[3][(PPT + 1) / 2];
  auto Tr = [&](int p) -> float& { return (p & 1) ? TT[p >> 1].y : TT[p >> 1].x; };
  auto Cr = [&](int p, int c) -> float& { return (p & 1) ? CC[c][p >> 1].y : CC[c][p >> 1].x; };
  double Td[TOUCH ? PPT : 1], Cd[TOUCH ? PPT : 1][3];
  int last[PPT];
  bool done[PPT];
  float px[PPT], py[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int li = tile_pixel<TS, PPT>(threadIdx.x, p);
    px[p] = (float)(x0 + li % TS);
    py[p] = (float)(y0 + li / TS);
    Tr(p) = 1.f;
    Cr(p, 0) = 0.f;
    Cr(p, 1) = 0.f;
    Cr(p, 2) = 0.f;
    if (TOUCH) {
      Td[p] = 1.0;
      Cd[p][0] = Cd[p][1] = Cd[p][2] = 0.0;
    }
    last[p] = 0;
    done[p] = (x0 + li % TS >= bp.W) || (y0 + li / TS >= bp.H);
    // fast path: "done" is T < stop itself (later splats fail T_before >= stop);
    // pixels outside the image start at T = 0 and are never written
    if (!TOUCH && done[p]) Tr(p) = 0.f;
  }
  for (int b = range.x; b < range.y; b += NT) {
    bool all_done = true;
#pragma unroll
    for (int p = 0; p < PPT; ++p) all_done &= TOUCH ? done[p] : !(Tr(p) >= bp.stop);
    if (__syncthreads_count(all_done) == NT) break;
    const int j = b + threadIdx.x;
    if (j < range.y) {
      const int r = (int)vals[j];
      stage_splat<TS>(g, r, x0, y0, s_sp[threadIdx.x]);
      if (TOUCH) {
        s_md[threadIdx.x] = g.r_mean[r];
        s_cd[threadIdx.x] = g.r_conop_d[r];
      }
    }
    if (TOUCH) s_touch[threadIdx.x] = 0;
    __syncthreads();
    const int cnt = min(NT, range.y - b);
    for (int k = 0; k < cnt; ++k) {
      if (!TOUCH) {  // fast path: reject on the log2 form before the exponential
        // (the vote makes the branch provably warp-uniform: the loop keeps its
        // uniform-register addressing)
        const float4 L = s_sp[k].L, Q = s_sp[k].Q;
        const float qlo = L.w, qhi = Q.w;
        float lgs[PPT];
        bool live[PPT], any_live = false, any_near = false;
        po.lg_all(L, Q, lgs);
#pragma unroll
        for (int p = 0; p < PPT; ++p) {
          live[p] = Tr(p) >= bp.stop && !(lgs[p] < qlo);
          any_live |= live[p];
          any_near |= live[p] && lgs[p] < qhi;
        }
        if (!__any_sync(0xffffffffu, any_live)) {  // warp-uniform skip
          bool alive = false;
#pragma unroll
          for (int p = 0; p < PPT; ++p) alive |= Tr(p) >= bp.stop;
          if (!__any_sync(0xffffffffu, alive)) break;  // this warp's pixels are all finished
          continue;
        }
        const float4 col = s_sp[k].col;
        float av[PPT];
#pragma unroll
        for (int p = 0; p < PPT; ++p) av[p] = live[p] ? fminf(bp.clamp, col.w * ex2_approx(lgs[p])) : 0.f;
        if (any_near) {  // rare: decide in float64
#pragma unroll
          for (int p = 0; p < PPT; ++p)
            if (live[p] && lgs[p] < qhi) av[p] = alpha_f64(bp, g, s_sp[k].rank, px[p], py[p]);
        }
        if constexpr (PPT % 2 == 0) {  // two pixels per packed FMA, the same roundings
#pragma unroll
          for (int q = 0; q < PPT / 2; ++q) {
            const float2 a = make_float2(av[2 * q], av[2 * q + 1]);
            const float2 wgt = __fmul2_rn(a, TT[q]);
            CC[0][q] = __ffma2_rn(wgt, make_float2(col.x, col.x), CC[0][q]);
            CC[1][q] = __ffma2_rn(wgt, make_float2(col.y, col.y), CC[1][q]);
            CC[2][q] = __ffma2_rn(wgt, make_float2(col.z, col.z), CC[2][q]);
            TT[q] = __ffma2_rn(make_float2(-a.x, -a.y), TT[q], TT[q]);  // T (1 - a) in one rounding
            last[2 * q] = a.x > 0.f ? b - range.x + k + 1 : last[2 * q];
            last[2 * q + 1] = a.y > 0.f ? b - range.x + k + 1 : last[2 * q + 1];
          }
        } else {
#pragma unroll
        for (int p = 0; p < PPT; ++p) {  // predicated: a = 0 leaves the pixel unchanged
          const float a = av[p];
          const float wgt = a * Tr(p);
          Cr(p, 0) = fmaf(wgt, col.x, Cr(p, 0));
          Cr(p, 1) = fmaf(wgt, col.y, Cr(p, 1));
          Cr(p, 2) = fmaf(wgt, col.z, Cr(p, 2));
          Tr(p) = fmaf(-a, Tr(p), Tr(p));  // T (1 - a) in one rounding
          last[p] = a > 0.f ? b - range.x + k + 1 : last[p];
        }
        }
        continue;
      }
      // ---- TOUCH: float64 per pair (rasterizer.py:187-211, :279)
      const double2 md = s_md[k];
      const double4 cd = s_cd[k];
      const float4 col = s_sp[k].col;
      int contrib = 0;
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        if (done[p]) continue;
        const double ddx = (double)px[p] - md.x, ddy = (double)py[p] - md.y;
        const double mh = cd.x * ddx * ddx + cd.y * ddx * ddy + cd.z * ddy * ddy;
        double a = fmin(bp.clamp_d, cd.w * exp(-0.5 * mh));
        if (a < bp.skip_d) a = 0.0;
        const double w = a * Td[p];
        if (w > 0.0) ++contrib;
        if (a == 0.0) continue;
        Cd[p][0] += w * (double)col.x;
        Cd[p][1] += w * (double)col.y;
        Cd[p][2] += w * (double)col.z;
        Td[p] *= 1.0 - a;
        last[p] = b - range.x + k + 1;
        if (Td[p] < bp.stop_d) done[p] = true;  // later splats fail T_before >= stop
      }
      const unsigned bal = __ballot_sync(0xffffffffu, contrib > 0);
      int tot = contrib;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      if (bal && (threadIdx.x & 31) == 0) atomicAdd(&s_touch[k], tot);
    }
    if (TOUCH) {
      __syncthreads();
      if (threadIdx.x < cnt && s_touch[threadIdx.x] > 0)
        atomicAdd(&touch[g.order[s_sp[threadIdx.x].rank]], s_touch[threadIdx.x]);
    }
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int pxi = (int)px[p], pyi = (int)py[p];
    if (pxi >= bp.W || pyi >= bp.H) continue;
    const int64_t pix = (int64_t)pyi * bp.W + pxi;
    if (TOUCH) {
      Tr(p) = (float)Td[p];
      image[3 * pix + 0] = (float)(Cd[p][0] + Td[p] * (double)bp.bg[0]);
      image[3 * pix + 1] = (float)(Cd[p][1] + Td[p] * (double)bp.bg[1]);
      image[3 * pix + 2] = (float)(Cd[p][2] + Td[p] * (double)bp.bg[2]);
      if (alpha_map) alpha_map[pix] = (float)(1.0 - Td[p]);
    } else {
      image[3 * pix + 0] = Cr(p, 0) + Tr(p) * bp.bg[0];
      image[3 * pix + 1] = Cr(p, 1) + Tr(p) * bp.bg[1];
      image[3 * pix + 2] = Cr(p, 2) + Tr(p) * bp.bg[2];
      if (alpha_map) alpha_map[pix] = 1.f - Tr(p);
    }
    g.t_final[pix] = Tr(p);
    g.n_contrib[pix] = last[p];
  }
}

// K5a: reverse blend (rasterizer.py:306-349).  Per pixel, walk the tile list
// back to front from the last contributor reconstructing T_before by
// division, keeping the suffix sum incl. the background term.  Per splat the
// geometric gradient is kept as moments about the tile centre d:
//   M0 = sum dm, M1 = sum dm d, M2 = sum dm d d^T   (dm = op G dalpha),
// which carry no large offsets; the flush shifts them to the splat's anchor
// (the centre of its rectangle's first tile, integer multiples of the tile
// size away) and K5b applies the anchor-to-mean offset in float64:
//   sum dm (x - mu) = Delta M0 + M1, sum dm (x - mu)(x - mu)^T = ... .
// Without that, fp32 sums of dm (x - mu)^2 over a splat near the camera plane
// (|x - mu| ~ 1e5 px) lose the gradient entirely.  Per splat the 8 terms
// colour 3, M1 2, M2 3 are reduced across the warp with a reduce-scatter
// butterfly (9 shuffles) so lane 4i ends up holding term i, M0 with a warp
// sum; those lanes add into shared-memory per-splat accumulators, flushed to
// the per-rank global accumulators once per batch.
template <int TS>
__global__ void __launch_bounds__(BlendShape<TS, true>::NT) blend_bwd_kernel(
    BlendParams bp, Geom g, const uint32_t* __restrict__ vals, const float* __restrict__ d_image,
    int tile0) {
  constexpr int NT = BlendShape<TS, true>::NT, PPT = BlendShape<TS, true>::PPT;
  constexpr int NA = 9;  // colour 3, M1 2, M2 3, M0
  // a thread's pixels share their column when the tile width divides the
  // warp's 32-pixel rows (tile_pixel): the dx moments then follow from M0, M1y
  constexpr bool DXC = TS <= 32;
#ifndef SS_BWD_PAIRS
#define SS_BWD_PAIRS 1
#endif
  constexpr bool PAIRS = SS_BWD_PAIRS && DXC && PPT % 2 == 0;
  __shared__ SplatRec s_sp[NT];
  // each warp owns a slot per splat (plain stores, summed at the flush);
  // larger tiles share one slot through shared-memory atomics
  constexpr bool PRIV = NT / 32 <= 4;
  constexpr int NW = PRIV ? NT / 32 : 1;
  __shared__ float s_acc[NW * NT * NA];  // [warp][splat][term]
  __shared__ int s_any[NT];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tile = tile0 >= 0 ? tile0 + (int)blockIdx.x : g.tile_order[blockIdx.x];
  const int tx = tile % bp.ntx, ty = tile / bp.ntx;
  const int x0 = tx * TS, y0 = ty * TS;
  const int2 range = g.ranges[tile];
  PixelOffsets<TS, PPT> po;
  po.init(threadIdx.x);
  float T[PPT], S[PPT], gp[PPT][3], px[PPT], py[PPT];
  int last[PPT];
  int max_last = 0;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int li = tile_pixel<TS, PPT>(threadIdx.x, p);
    const int pxi = x0 + li % TS, pyi = y0 + li / TS;
    px[p] = (float)pxi;
    py[p] = (float)pyi;
    if (pxi < bp.W && pyi < bp.H) {
      const int64_t pix = (int64_t)pyi * bp.W + pxi;
      T[p] = g.t_final[pix];
      last[p] = g.n_contrib[pix];
      gp[p][0] = d_image[3 * pix];
      gp[p][1] = d_image[3 * pix + 1];
      gp[p][2] = d_image[3 * pix + 2];
    } else {
      T[p] = 0.f;
      last[p] = 0;
      gp[p][0] = gp[p][1] = gp[p][2] = 0.f;
    }
    const float gb = gp[p][0] * bp.bg[0] + gp[p][1] * bp.bg[1] + gp[p][2] * bp.bg[2];
    S[p] = gb * T[p];
    max_last = max(max_last, last[p]);
  }
  if (threadIdx.x == 0) s_last = 0;
  for (int i = threadIdx.x; i < NW * NT * NA; i += NT) s_acc[i] = 0.f;
  s_any[threadIdx.x] = 0;
  __syncthreads();
  atomicMax(&s_last, max_last);
  __syncthreads();
  const int end0 = range.x + s_last;  // positions past every pixel's last contributor are dead
  // pixel pairs as packed registers for the FFMA2 path
  float2 T2[PAIRS ? PPT / 2 : 1], S2[PAIRS ? PPT / 2 : 1], G0[PAIRS ? PPT / 2 : 1],
      G1[PAIRS ? PPT / 2 : 1], G2[PAIRS ? PPT / 2 : 1], DY[PAIRS ? PPT / 2 : 1];
  if constexpr (PAIRS) {
#pragma unroll
    for (int q = 0; q < PPT / 2; ++q) {
      T2[q] = make_float2(T[2 * q], T[2 * q + 1]);
      S2[q] = make_float2(S[2 * q], S[2 * q + 1]);
      G0[q] = make_float2(gp[2 * q][0], gp[2 * q + 1][0]);
      G1[q] = make_float2(gp[2 * q][1], gp[2 * q + 1][1]);
      G2[q] = make_float2(gp[2 * q][2], gp[2 * q + 1][2]);
      DY[q] = make_float2(po.dy[2 * q], po.dy[2 * q + 1]);
    }
  }
  for (int end = end0; end > range.x; end -= NT) {
    const int start = max(range.x, end - NT);
    const int cnt = end - start;
    if (threadIdx.x < cnt) stage_splat<TS>(g, (int)vals[end - 1 - threadIdx.x], x0, y0,
                                           s_sp[threadIdx.x]);
    __syncthreads();
    for (int k = 0; k < cnt; ++k) {
      const int pos_rel = end - 1 - k - range.x;
      const float4 L = s_sp[k].L, Q = s_sp[k].Q;
      const float qlo = L.w, qhi = Q.w;
      // cheap part for every pixel, then a warp-uniform skip; the rest is
      // predicated (a = 0 makes every update a no-op) instead of branching
      float lgs[PPT];
      bool live[PPT], any_live = false, any_near = false;
      po.lg_all(L, Q, lgs);  // same decisions as the forward
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        live[p] = pos_rel < last[p] && !(lgs[p] < qlo);
        any_live |= live[p];
        any_near |= live[p] && lgs[p] < qhi;
      }
      if (!__any_sync(0xffffffffu, any_live)) continue;
      const float4 col = s_sp[k].col;
      // og = opacity G for live pixels, 0 otherwise: a = min(clamp, og) is then
      // 0 for dead pixels without a separate select
      float og[PPT], av[PPT];
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        og[p] = live[p] ? col.w * ex2_approx(lgs[p]) : 0.f;
        av[p] = fminf(bp.clamp, og[p]);
      }
      if (any_near) {  // rare: decide in float64
#pragma unroll
        for (int p = 0; p < PPT; ++p)
          if (live[p] && lgs[p] < qhi) {
            av[p] = alpha_f64(bp, g, s_sp[k].rank, px[p], py[p]);
            if (!(av[p] > 0.f)) og[p] = 0.f;
          }
      }
      float v[NA] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      bool any = false;
      if constexpr (PAIRS) {
        // the same per-pixel roundings, two pixels per packed instruction
        // (FFMA2 / FMUL2, the splat's values as broadcast scalars); the
        // accumulators keep one partial per pixel of a pair
        const float2 cx = make_float2(col.x, col.x), cy = make_float2(col.y, col.y),
                     cz = make_float2(col.z, col.z);
        const float2 one = make_float2(1.f, 1.f), mone = make_float2(-1.f, -1.f);
        float2 c0 = make_float2(0.f, 0.f), c1 = c0, c2 = c0, m1 = c0, m2 = c0, m0 = c0;
#pragma unroll
        for (int q = 0; q < PPT / 2; ++q) {
          const float2 a = make_float2(av[2 * q], av[2 * q + 1]);
          const float2 om = __ffma2_rn(a, mone, one);  // 1 - a, one rounding
          const float2 ioma = make_float2(rcp_approx(om.x), rcp_approx(om.y));
          const float2 tb = __fmul2_rn(T2[q], ioma);
          const float2 w = __fmul2_rn(a, tb);
          c0 = __ffma2_rn(w, G0[q], c0);
          c1 = __ffma2_rn(w, G1[q], c1);
          c2 = __ffma2_rn(w, G2[q], c2);
          const float2 u = __ffma2_rn(G2[q], cz, __ffma2_rn(G1[q], cy, __fmul2_rn(G0[q], cx)));
          const float2 da = __fmul2_rn(__ffma2_rn(u, T2[q], make_float2(-S2[q].x, -S2[q].y)), ioma);
          S2[q] = __ffma2_rn(u, w, S2[q]);
          T2[q] = tb;
          const float2 dmr = __fmul2_rn(make_float2(og[2 * q], og[2 * q + 1]), da);
          const float2 dm = make_float2(og[2 * q] < bp.clamp ? dmr.x : 0.f,
                                        og[2 * q + 1] < bp.clamp ? dmr.y : 0.f);
          const float2 f = __fmul2_rn(dm, DY[q]);
          m1 = __fadd2_rn(m1, f);
          m2 = __ffma2_rn(f, DY[q], m2);
          m0 = __fadd2_rn(m0, dm);
          any |= a.x > 0.f || a.y > 0.f;
        }
        v[0] = c0.x + c0.y;
        v[1] = c1.x + c1.y;
        v[2] = c2.x + c2.y;
        v[4] = m1.x + m1.y;
        v[7] = m2.x + m2.y;
        v[8] = m0.x + m0.y;
      } else {
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        const float a = av[p];
        // one approximate reciprocal serves T_before = T / (1 - a) and
        // dL/dalpha = (u T - S) / (1 - a)  (T after this splat, S the suffix)
        const float ioma = rcp_approx(1.f - a);  // a <= alpha_clamp < 1
        const float tb = T[p] * ioma;
        const float w = a * tb;
        v[0] = fmaf(w, gp[p][0], v[0]);
        v[1] = fmaf(w, gp[p][1], v[1]);
        v[2] = fmaf(w, gp[p][2], v[2]);
        const float u = gp[p][0] * col.x + gp[p][1] * col.y + gp[p][2] * col.z;
        const float da = fmaf(u, T[p], -S[p]) * ioma;
        S[p] = fmaf(u, w, S[p]);
        T[p] = tb;
        // dm = og da (the reference's -0.5 is applied in K5b), zero for dead
        // pixels (og = 0) and flat above the clamp (rasterizer.py:336-337);
        // moments about the tile centre
        const float dm = og[p] < bp.clamp ? og[p] * da : 0.f;
        if (DXC) {  // this thread's pixels share dx: sum dm, dm dy, dm dy^2 only
          const float f = dm * po.dy[p];
          v[4] += f;
          v[7] = fmaf(f, po.dy[p], v[7]);
        } else {
          const float e = dm * po.dx[p], f = dm * po.dy[p];
          v[3] += e;
          v[4] += f;
          v[5] = fmaf(e, po.dx[p], v[5]);
          v[6] = fmaf(e, po.dy[p], v[6]);
          v[7] = fmaf(f, po.dy[p], v[7]);
        }
        v[8] += dm;
        any |= a > 0.f;
      }
      }
      if (DXC) {  // M1x = dx M0, M2xx = dx M1x, M2xy = dx M1y
        const float dx = po.dx[0];
        v[3] = dx * v[8];
        v[5] = dx * v[3];
        v[6] = dx * v[4];
      }
      const unsigned bal = __ballot_sync(0xffffffffu, any);
      if (bal) {
        // reduce-scatter butterfly over terms 0..7: after it lane L holds the
        // warp total of term (L >> 2) (valid in lanes with L & 3 == 0)
        const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
        float h4[4], h2[2], h1;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float send = b4 ? v[i] : v[4 + i];
          h4[i] = (b4 ? v[4 + i] : v[i]) + __shfl_xor_sync(0xffffffffu, send, 16);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const float send = b3 ? h4[i] : h4[2 + i];
          h2[i] = (b3 ? h4[2 + i] : h4[i]) + __shfl_xor_sync(0xffffffffu, send, 8);
        }
        {
          const float send = b2 ? h2[0] : h2[1];
          h1 = (b2 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
        h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
        const float m0 = warp_sum(v[8]);
        float* slot = s_acc + ((PRIV ? warp : 0) * NT + k) * NA;
        if ((lane & 3) == 0) {
          if (PRIV) slot[lane >> 2] = h1;
          else atomicAdd(slot + (lane >> 2), h1);
        }
        if (lane == 0) {
          if (PRIV) slot[8] = m0;
          else atomicAdd(slot + 8, m0);
          s_any[k] = 1;
        }
      }
    }
    __syncthreads();
    // flush this batch's per-splat sums (one row per splat) and reset them
    if (threadIdx.x < cnt && s_any[threadIdx.x]) {
      const int r = s_sp[threadIdx.x].rank;
      float* a = g.acc + (int64_t)r * kAccStride;
      float t[NA];
#pragma unroll
      for (int q = 0; q < NA; ++q) t[q] = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        float* sa = s_acc + (w * NT + threadIdx.x) * NA;
#pragma unroll
        for (int q = 0; q < NA; ++q) {
          t[q] += sa[q];
          sa[q] = 0.f;
        }
      }
      // shift the moments from this tile's centre to the anchor (the centre
      // of the rectangle's first tile): d_anchor = d_tile + s, s multiples of TS
      const int4 rc = g.r_rect[r];
      const float sx = (float)((tx - rc.x) * TS), sy = (float)((ty - rc.z) * TS);
      const float M0 = t[8], M1x = t[3], M1y = t[4];
      red_add_v4(a, t[0], t[1], t[2], M0);
      red_add_v4(a + 4, fmaf(sx, M0, M1x), fmaf(sy, M0, M1y),
                 fmaf(sx * sx, M0, fmaf(2.f * sx, M1x, t[5])),
                 fmaf(sx * sy, M0, fmaf(sx, M1y, fmaf(sy, M1x, t[6]))));
      atomicAdd(a + 8, fmaf(sy * sy, M0, fmaf(2.f * sy, M1y, t[7])));
      g.touched[r] = 1;
      s_any[threadIdx.x] = 0;
    }
    __syncthreads();
  }
}

// K5b: per-Gaussian chain from the rank accumulators back to the raw parameters
// (rasterizer.py:351-402).  One thread per Gaussian in index order (coalesced
// parameter reads and gradient writes; the rank accumulators are gathered).
// The EWA / covariance / projection chain runs in fp64; the SH part (d_sh,
// the view-direction gradient) in fp32 with the forward's clip mask.
template <int DEG>
__global__ void __launch_bounds__(128, SS_GB_BLOCKS) gaussian_bwd_kernel(CamD cam, ss_cloud cl, Geom g,
                                                              int64_t n, ss_cloud_grads out,
                                                              int full, int ts, int acc) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= n) return;
  constexpr int K = (DEG + 1) * (DEG + 1);  // == cl.sh_coeffs
  const int r = g.rank_of[gid];
  // culled, or no pixel of this view took a weight from it (all accumulators
  // are exactly 0, so every gradient is): zero rows so callers need no memset
  // (acc != 0: the parameter gradients are sums over views, leave them)
  if (r >= g.dev_counts[0] || !g.touched[r]) {
    if (out.viewspace) out.viewspace[gid] = 0.f;
    if (out.contributed) out.contributed[gid] = 0;
    if (acc) return;
    if (out.d_means) for (int j = 0; j < 3; ++j) out.d_means[3 * gid + j] = 0.f;
    if (out.d_rotations)
      *reinterpret_cast<float4*>(out.d_rotations + 4 * gid) = make_float4(0.f, 0.f, 0.f, 0.f);
    if (out.d_sh) {
      if (K == 16 && (reinterpret_cast<uintptr_t>(out.d_sh) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 12; ++j)
          reinterpret_cast<float4*>(out.d_sh + gid * 48)[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        for (int j = 0; j < 3 * K; ++j) out.d_sh[gid * 3 * K + j] = 0.f;
      }
    }
    if (full && out.d_log_scales) for (int j = 0; j < 3; ++j) out.d_log_scales[3 * gid + j] = 0.f;
    if (full && out.d_opacity_logits) out.d_opacity_logits[gid] = 0.f;
    return;
  }
  // degree 3: this Gaussian's 48 SH coefficients copied into shared memory
  // now (cp.async, no registers), consumed after the accumulator loads and
  // the anchor algebra instead of stalling the colour backward
  __shared__ __align__(16) float s_sh[K == 16 ? 128 * 48 : 1];
  const bool pf = K == 16 && blockDim.x <= 128 &&
                  ((reinterpret_cast<uintptr_t>(cl.sh) | reinterpret_cast<uintptr_t>(out.d_sh)) &
                   15) == 0;
  float* my_sh = s_sh + (K == 16 ? threadIdx.x * 48 : 0);
  if (pf) {
#pragma unroll
    for (int j = 0; j < 12; ++j)
      cp_async16(my_sh + 4 * j, reinterpret_cast<const float4*>(cl.sh + gid * 48) + j);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const float4 a0 = *reinterpret_cast<const float4*>(g.acc + (int64_t)r * kAccStride);
  const float4 a1 = *reinterpret_cast<const float4*>(g.acc + (int64_t)r * kAccStride + 4);
  const float a8 = g.acc[(int64_t)r * kAccStride + 8];
  // moments about the anchor (K5a) -> sums over (x - mu): Delta = anchor - mu
  double am[2], A[2][2], aop;
  {
    const int4 rc = g.r_rect[r];
    const double2 m = g.r_mean[r];
    const double4 cd = g.r_conop_d[r];
    const double c0 = 0.5 * (ts - 1);
    const double Dx = ((double)rc.x * ts + c0) - m.x, Dy = ((double)rc.z * ts + c0) - m.y;
    const double M0 = a0.w, M1x = a1.x, M1y = a1.y, M2xx = a1.z, M2xy = a1.w, M2yy = a8;
    const double E = Dx * M0 + M1x, F = Dy * M0 + M1y;
    const double Exx = Dx * Dx * M0 + 2.0 * Dx * M1x + M2xx;
    const double Exy = Dx * Dy * M0 + Dx * M1y + Dy * M1x + M2xy;
    const double Fyy = Dy * Dy * M0 + 2.0 * Dy * M1y + M2yy;
    // acc_mean2d = C [E, F] (rasterizer.py:342-343 with dm_ref = -dm / 2),
    // acc_conic = -1/2 [E_xx E_xy; E_xy F_yy], acc_opacity = sum G da = M0 / op
    const double c01 = 0.5 * cd.y;
    am[0] = cd.x * E + c01 * F;
    am[1] = c01 * E + cd.z * F;
    A[0][0] = -0.5 * Exx;
    A[0][1] = A[1][0] = -0.5 * Exy;
    A[1][1] = -0.5 * Fyy;
    aop = M0 / cd.w;
  }
  if (out.viewspace) out.viewspace[gid] = (float)sqrt(am[0] * am[0] + am[1] * am[1]);
  if (out.contributed) out.contributed[gid] = g.touched[r];
  // ---- colour -> SH and view direction first (sh.py:62-81), fp32 with the
  // forward's clip mask; its registers are free before the fp64 chain below
  double gw[3];
  {
    const float* m = cl.means + 3 * gid;
    double d[3];
    for (int q = 0; q < 3; ++q) d[q] = (double)m[q] - cam.pos[q];
    const double dist = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    const double dd = fmax(dist, 1e-12);
    double dir[3];
    for (int q = 0; q < 3; ++q) dir[q] = d[q] / dd;
    const int cm = (int)g.g_color[gid].w;
    const float gc[3] = {(cm & 1) ? a0.x : 0.f, (cm & 2) ? a0.y : 0.f, (cm & 4) ? a0.z : 0.f};
    const float fdir[3] = {(float)dir[0], (float)dir[1], (float)dir[2]};
    float basis[K], gbasis[K];
    sh_basis<float>(DEG, fdir[0], fdir[1], fdir[2], basis);
    const float* sh = cl.sh + gid * 3 * K;
    float* dsh = out.d_sh ? out.d_sh + gid * 3 * K : nullptr;
    if (pf) {  // degree 3: the 48 staged coefficients as 12 float4 / 12 float4 stores
      asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
      for (int k = 0; k < K; ++k) gbasis[k] = 0.f;
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        const float4 v = reinterpret_cast<const float4*>(my_sh)[j];
        const float e[4] = {v.x, v.y, v.z, v.w};
        float o[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int k = (4 * j + t) / 3, c = (4 * j + t) % 3;
          gbasis[k] = fmaf(e[t], gc[c], gbasis[k]);
          o[t] = basis[k] * gc[c];
        }
        if (dsh) {
          float4 w4 = make_float4(o[0], o[1], o[2], o[3]);
          if (acc) {
            const float4 p4 = reinterpret_cast<const float4*>(dsh)[j];
            w4.x += p4.x, w4.y += p4.y, w4.z += p4.z, w4.w += p4.w;
          }
          reinterpret_cast<float4*>(dsh)[j] = w4;
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        gbasis[k] = sh[3 * k] * gc[0] + sh[3 * k + 1] * gc[1] + sh[3 * k + 2] * gc[2];
        if (dsh) {
          dsh[3 * k] = basis[k] * gc[0] + (acc ? dsh[3 * k] : 0.f);
          dsh[3 * k + 1] = basis[k] * gc[1] + (acc ? dsh[3 * k + 1] : 0.f);
          dsh[3 * k + 2] = basis[k] * gc[2] + (acc ? dsh[3 * k + 2] : 0.f);
        }
      }
    }
    float gdirf[3] = {0.f, 0.f, 0.f};
    sh_basis_vjp<float>(DEG, fdir[0], fdir[1], fdir[2], gbasis, gdirf);
    const double gdir[3] = {gdirf[0], gdirf[1], gdirf[2]};
    const double dg = dir[0] * gdir[0] + dir[1] * gdir[1] + dir[2] * gdir[2];
    for (int i = 0; i < 3; ++i) gw[i] = (gdir[i] - dir[i] * dg) / dd;
  }
  Projected P;
  project_geom(cam, cl, gid, P);
  // conic -> cov2d: -C A C
  double CA[2][2], gcov2[2][2];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) CA[i][j] = P.conic[i][0] * A[0][j] + P.conic[i][1] * A[1][j];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) gcov2[i][j] = -(CA[i][0] * P.conic[0][j] + CA[i][1] * P.conic[1][j]);
  // cov2d = M S M^T: g_S = M^T G M, g_M = (G + G^T) M S
  double gS[3][3], GM[2][3], gM[2][3];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)
      GM[i][j] = (gcov2[i][0] + gcov2[0][i]) * P.M[0][j] + (gcov2[i][1] + gcov2[1][i]) * P.M[1][j];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)
      gM[i][j] = GM[i][0] * P.S[0][j] + GM[i][1] * P.S[1][j] + GM[i][2] * P.S[2][j];
  double GMt[2][3];  // gcov2 M, rows p
  for (int p = 0; p < 2; ++p)
    for (int j = 0; j < 3; ++j) GMt[p][j] = gcov2[p][0] * P.M[0][j] + gcov2[p][1] * P.M[1][j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) gS[i][j] = P.M[0][i] * GMt[0][j] + P.M[1][i] * GMt[1][j];
  // g_J = g_M R_w^T
  double gJ[2][3];
  for (int i = 0; i < 2; ++i)
    for (int k = 0; k < 3; ++k)
      gJ[i][k] = gM[i][0] * cam.R[k][0] + gM[i][1] * cam.R[k][1] + gM[i][2] * cam.R[k][2];
  const double x = P.p[0], y = P.p[1], z = P.p[2];
  const double fx = cam.fx, fy = cam.fy;
  const double iz = 1.0 / z, iz2 = iz * iz;
  double gp[3];
  gp[0] = gJ[0][2] * (-fx * iz2);
  gp[1] = gJ[1][2] * (-fy * iz2);
  gp[2] = gJ[0][0] * (-fx * iz2) + gJ[1][1] * (-fy * iz2) + gJ[0][2] * (2.0 * fx * x * iz2 * iz) +
          gJ[1][2] * (2.0 * fy * y * iz2 * iz);
  // + J^T acc_mean2d
  gp[0] += (fx * iz) * am[0];
  gp[1] += (fy * iz) * am[1];
  gp[2] += (-fx * x * iz2) * am[0] + (-fy * y * iz2) * am[1];
  for (int j = 0; j < 3; ++j)
    gw[j] += gp[0] * cam.R[0][j] + gp[1] * cam.R[1][j] + gp[2] * cam.R[2][j];
  if (out.d_means)
    for (int j = 0; j < 3; ++j)
      out.d_means[3 * gid + j] = (float)gw[j] + (acc ? out.d_means[3 * gid + j] : 0.f);
  // covariance -> quaternion / log scales (gaussians.py:127-154)
  double gsym[3][3], gR[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) gsym[i][j] = gS[i][j] + gS[j][i];
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k)
      gR[i][k] = (gsym[i][0] * P.Rq[0][k] + gsym[i][1] * P.Rq[1][k] + gsym[i][2] * P.Rq[2][k]) *
                 P.var[k];
  if (out.d_rotations) {
    double gu[4];
    quat_to_rot_vjp(P.u[0], P.u[1], P.u[2], P.u[3], gR, gu);
    const double dot = P.u[0] * gu[0] + P.u[1] * gu[1] + P.u[2] * gu[2] + P.u[3] * gu[3];
    float4 q4 = make_float4((float)((gu[0] - P.u[0] * dot) / P.qn),
                            (float)((gu[1] - P.u[1] * dot) / P.qn),
                            (float)((gu[2] - P.u[2] * dot) / P.qn),
                            (float)((gu[3] - P.u[3] * dot) / P.qn));
    if (acc) {
      const float4 p4 = *reinterpret_cast<const float4*>(out.d_rotations + 4 * gid);
      q4.x += p4.x, q4.y += p4.y, q4.z += p4.z, q4.w += p4.w;
    }
    *reinterpret_cast<float4*>(out.d_rotations + 4 * gid) = q4;
  }
  if (full) {
    if (out.d_log_scales)
      for (int i = 0; i < 3; ++i) {
        double s = 0;
        for (int j = 0; j < 3; ++j)
          for (int k = 0; k < 3; ++k) s += P.Rq[j][i] * gS[j][k] * P.Rq[k][i];
        out.d_log_scales[3 * gid + i] =
            (float)(s * 2.0 * P.var[i]) + (acc ? out.d_log_scales[3 * gid + i] : 0.f);
      }
    if (out.d_opacity_logits)
      out.d_opacity_logits[gid] =
          (float)(aop * P.op * (1.0 - P.op)) + (acc ? out.d_opacity_logits[gid] : 0.f);
  }
}

// ------------------------------------------------------------------ host glue
static BlendParams blend_params(const ss_camera* cam, const ss_raster_settings* s) {
  BlendParams bp{};
  bp.W = cam->width;
  bp.H = cam->height;
  bp.ntx = ntiles_x(cam, s);
  bp.clamp = (float)s->alpha_clamp;
  bp.skip = (float)s->skip_alpha;
  bp.stop = (float)s->stop_transmittance;
  bp.clamp_d = s->alpha_clamp;
  bp.skip_d = s->skip_alpha;
  bp.stop_d = s->stop_transmittance;
  for (int i = 0; i < 3; ++i) bp.bg[i] = (float)s->background[i];
  return bp;
}

static int check_raster(const ss_cloud* cl, const ss_camera* cam, const ss_raster_settings* s) {
  if (!cam || !s || cam->width <= 0 || cam->height <= 0) {
    set_error("invalid camera");
    return SS_ERR_DATA;
  }
  if (s->tile_size != 8 && s->tile_size != 16 && s->tile_size != 32 && s->tile_size != 64) {
    set_error("tile_size must be 8, 16, 32 or 64");
    return SS_ERR_DATA;
  }
  if (cl && (cl->sh_coeffs < 1 || cl->sh_coeffs > 16 ||
             sh_degree_of(cl->sh_coeffs) != (int)std::sqrt((double)cl->sh_coeffs) - 1)) {
    set_error("sh_coeffs must be 1, 4, 9 or 16");
    return SS_ERR_DATA;
  }
  return SS_OK;
}

template <bool TOUCH>
static int launch_blend_fwd(int ts, int64_t ntiles, cudaStream_t st, const BlendParams& bp,
                            const Geom& g, const uint32_t* vals, float* image, float* alpha,
                            int32_t* touch, int tile0 = 0) {
  const unsigned grid = (unsigned)ntiles;
  switch (ts) {
    case 8: blend_fwd_kernel<8, TOUCH><<<grid, BlendShape<8>::NT, 0, st>>>(bp, g, vals, image, alpha, touch, tile0); break;
    case 16: blend_fwd_kernel<16, TOUCH><<<grid, BlendShape<16>::NT, 0, st>>>(bp, g, vals, image, alpha, touch, tile0); break;
    case 32: blend_fwd_kernel<32, TOUCH><<<grid, BlendShape<32>::NT, 0, st>>>(bp, g, vals, image, alpha, touch, tile0); break;
    default: blend_fwd_kernel<64, TOUCH><<<grid, BlendShape<64>::NT, 0, st>>>(bp, g, vals, image, alpha, touch, tile0); break;
  }
  SS_CHECK_LAUNCH("blend_fwd_kernel");
  return SS_OK;
}

static int launch_blend_bwd(int ts, int64_t ntiles, cudaStream_t st, const BlendParams& bp,
                            const Geom& g, const uint32_t* vals, const float* d_image,
                            int tile0 = 0) {
  const unsigned grid = (unsigned)ntiles;
  switch (ts) {
    case 8: blend_bwd_kernel<8><<<grid, BlendShape<8, true>::NT, 0, st>>>(bp, g, vals, d_image, tile0); break;
    case 16: blend_bwd_kernel<16><<<grid, BlendShape<16, true>::NT, 0, st>>>(bp, g, vals, d_image, tile0); break;
    case 32: blend_bwd_kernel<32><<<grid, BlendShape<32, true>::NT, 0, st>>>(bp, g, vals, d_image, tile0); break;
    default: blend_bwd_kernel<64><<<grid, BlendShape<64, true>::NT, 0, st>>>(bp, g, vals, d_image, tile0); break;
  }
  SS_CHECK_LAUNCH("blend_bwd_kernel");
  return SS_OK;
}

int raster_zero_iteration(void* geom, int64_t n, const ss_camera* cam, const ss_raster_settings* s,
                          void* bins, int64_t cap, void* extra, size_t extra_bytes,
                          cudaStream_t st) {
  const Geom g = plan_geom(geom, n, cam, s);
  (void)bins, (void)cap;  // the bins are cleared by bin_pairs (see there)
  ZeroRegions z{};
  auto add = [&](void* p, int64_t bytes) {
    if (p && bytes > 0) z.p[z.n] = static_cast<uint8_t*>(p), z.bytes[z.n++] = bytes;
  };
  const int64_t hist_bytes = (4 * 256 + 64) * sizeof(uint32_t);  // binsort_clear_bytes
  add(g.dev_counts, 3 * sizeof(int64_t));
  add(g.dsort.hist, hist_bytes);
  add(g.dsort.status, (int64_t)g.dsort.max_passes * g.dsort.max_blocks * 256 * sizeof(uint32_t));
  add(g.scan_lb, (g.scan_blocks + 1) * (int64_t)sizeof(unsigned long long));
  add(g.acc, n * kAccStride * (int64_t)sizeof(float));
  add(g.touched, n);
  add(extra, (int64_t)extra_bytes);
  zero_regions_kernel<<<148 * 4, 256, 0, st>>>(z);
  SS_CHECK_LAUNCH("zero_regions_kernel");
  return SS_OK;
}

int raster_begin(const ss_cloud* cl, const ss_camera* cam, const ss_raster_settings* s,
                 void* geom, int64_t* counts_host, cudaStream_t st) {
  SS_TRY(check_raster(cl, cam, s));
  const int64_t n = cl->n;
  Geom g = plan_geom(geom, n, cam, s);
  const CamD cd = make_cam(cam);
  if (!t_prezeroed) SS_CUDA(cudaMemsetAsync(g.dev_counts, 0, 3 * sizeof(int64_t), st));
  if (n > 0) {
    SS_TRY(binsort_clear(g.dsort, 32, st));  // preprocess_kernel builds the histograms
    prof_begin(PH_PROJECT, st);
    {
      const unsigned grid = (unsigned)cdiv(n, 256);
      switch (cl->sh_coeffs) {
        case 1: preprocess_kernel<0><<<grid, 256, 0, st>>>(cd, *cl, g); break;
        case 4: preprocess_kernel<1><<<grid, 256, 0, st>>>(cd, *cl, g); break;
        case 9: preprocess_kernel<2><<<grid, 256, 0, st>>>(cd, *cl, g); break;
        default: {
          static bool attr = false;  // 48 KB dynamic + the static histograms
          if (!attr) {
            SS_CUDA(cudaFuncSetAttribute(preprocess_kernel<3>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kPpPrefetchBytes));
            attr = true;
          }
          preprocess_kernel<3><<<grid, 256, kPpPrefetchBytes, st>>>(cd, *cl, g);
          break;
        }
      }
    }
    SS_CHECK_LAUNCH("preprocess_kernel");
    prof_end(PH_PROJECT, st);
    prof_begin(PH_DEPTH_SORT, st);
    SS_TRY(binsort_run(g.dsort, g.key32_tmp, reinterpret_cast<uint32_t*>(g.idx_in), g.key32,
                       reinterpret_cast<uint32_t*>(g.order), g.dev_counts + 2, n, 32, st,
                       /*hist_ready=*/true));
    g_launches.fetch_add(4);
    depth_tie_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(g);
    SS_CHECK_LAUNCH("depth_tie_kernel");
    prof_end(PH_DEPTH_SORT, st);
    prof_begin(PH_RANK_SCAN, st);
    if (!t_prezeroed)
      SS_CUDA(cudaMemsetAsync(g.scan_lb, 0, (g.scan_blocks + 1) * sizeof(unsigned long long), st));
    rank_kernel<<<(unsigned)cdiv(n, kScanThreads * kScanRanks), kScanThreads, 0, st>>>(cd, *s, n, g);
    SS_CHECK_LAUNCH("rank_kernel");
    prof_end(PH_RANK_SCAN, st);
  } else {
    finish_counts_kernel<<<1, 1, 0, st>>>(g, n);
    SS_CHECK_LAUNCH("finish_counts_kernel");
  }
  if (counts_host)
    SS_CUDA(cudaMemcpyAsync(counts_host, g.dev_counts, 2 * sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
  return SS_OK;
}

// cap: pairs the `bins` workspace holds; total: the view's pair count when the
// host knows it (-1: only on the device, single band, overflow flagged).  A
// known total above cap is binned and blended in bands of tile rows.
int raster_finish(const ss_cloud* cl, const ss_camera* cam, const ss_raster_settings* s,
                  void* geom, void* bins, int64_t cap, float* image, float* alpha,
                  int32_t* touch, uint32_t* status, int cull, cudaStream_t st, int64_t total) {
  SS_TRY(check_raster(cl, cam, s));
  const int64_t n = cl->n;
  Geom g = plan_geom(geom, n, cam, s);
  Bins b = plan_bins(bins, cap);
  const int ntx = ntiles_x(cam, s), nty = ntiles_y(cam, s);
  const int64_t ntiles = (int64_t)ntx * nty;
  if (cap > (int64_t)0x7fffffff) {
    set_error("bin workspace above 2^31 pairs: bin in bands of tile rows instead");
    return SS_ERR_CAPACITY;
  }
  const BlendParams bp = blend_params(cam, s);
  if (total <= cap) {
    SS_TRY(bin_pairs(cam, s, n, g, b, status, cull, st));
    prof_begin(PH_BLEND_FWD, st);
    const int rc = touch ? launch_blend_fwd<true>(s->tile_size, ntiles, st, bp, g, b.vals_out,
                                                  image, alpha, touch, -1)
                         : launch_blend_fwd<false>(s->tile_size, ntiles, st, bp, g, b.vals_out,
                                                   image, alpha, nullptr, -1);
    prof_end(PH_BLEND_FWD, st);
    return rc;
  }
  std::vector<int2> bands;
  SS_TRY(plan_bands(cam, s, n, g, cap, bands, st));
  for (const int2 band : bands) {
    SS_TRY(bin_band(cam, s, n, g, b, status, cull, band, st));
    const int64_t nt = (int64_t)(band.y - band.x) * ntx;
    if (touch) SS_TRY(launch_blend_fwd<true>(s->tile_size, nt, st, bp, g, b.vals_out, image, alpha,
                                             touch, band.x * ntx));
    else SS_TRY(launch_blend_fwd<false>(s->tile_size, nt, st, bp, g, b.vals_out, image, alpha,
                                        nullptr, band.x * ntx));
  }
  return SS_OK;
}

const int64_t* raster_counts(void* geom, int64_t n, const ss_camera* cam,
                             const ss_raster_settings* s) {
  return plan_geom(geom, n, cam, s).dev_counts;
}

int raster_backward(const ss_cloud* cl, const ss_camera* cam, const ss_raster_settings* s,
                    void* geom, void* bins, int64_t cap, const float* d_image,
                    const ss_cloud_grads* grads, int full, cudaStream_t st, int64_t total,
                    int cull, uint32_t* status, int accumulate) {
  SS_TRY(check_raster(cl, cam, s));
  const int64_t n = cl->n;
  if (n == 0) return SS_OK;
  Geom g = plan_geom(geom, n, cam, s);
  Bins b = plan_bins(bins, cap);
  const int ntx = ntiles_x(cam, s);
  const int64_t ntiles = (int64_t)ntx * ntiles_y(cam, s);
  if (!t_prezeroed) {
    SS_CUDA(cudaMemsetAsync(g.acc, 0, n * kAccStride * sizeof(float), st));
    SS_CUDA(cudaMemsetAsync(g.touched, 0, n, st));
  }
  const BlendParams bp = blend_params(cam, s);
  if (total <= cap) {  // the forward's bins are still in the workspace
    prof_begin(PH_BLEND_BWD, st);
    SS_TRY(launch_blend_bwd(s->tile_size, ntiles, st, bp, g, b.vals_out, d_image, -1));
    prof_end(PH_BLEND_BWD, st);
  } else {  // bin every band again (the workspace holds one band)
    std::vector<int2> bands;
    SS_TRY(plan_bands(cam, s, n, g, cap, bands, st));
    for (const int2 band : bands) {
      SS_TRY(bin_band(cam, s, n, g, b, status, cull, band, st));
      SS_TRY(launch_blend_bwd(s->tile_size, (int64_t)(band.y - band.x) * ntx, st, bp, g,
                              b.vals_out, d_image, band.x * ntx));
    }
  }
  prof_begin(PH_GAUSS_BWD, st);
  {
    const unsigned grid = (unsigned)cdiv(n, 128);
    const CamD cd = make_cam(cam);
    switch (cl->sh_coeffs) {
      case 1: gaussian_bwd_kernel<0><<<grid, 128, 0, st>>>(cd, *cl, g, n, *grads, full, s->tile_size, accumulate); break;
      case 4: gaussian_bwd_kernel<1><<<grid, 128, 0, st>>>(cd, *cl, g, n, *grads, full, s->tile_size, accumulate); break;
      case 9: gaussian_bwd_kernel<2><<<grid, 128, 0, st>>>(cd, *cl, g, n, *grads, full, s->tile_size, accumulate); break;
      default: gaussian_bwd_kernel<3><<<grid, 128, 0, st>>>(cd, *cl, g, n, *grads, full, s->tile_size, accumulate); break;
    }
  }
  SS_CHECK_LAUNCH("gaussian_bwd_kernel");
  prof_end(PH_GAUSS_BWD, st);
  return SS_OK;
}

__global__ void tile_lists_kernel(int64_t ntiles, const int2* ranges, int32_t* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  out[2 * t] = ranges[t].x;
  out[2 * t + 1] = ranges[t].y;
}

// tile_bin on given projections (depth order = input order)
__global__ void tile_bin_setup_kernel(int64_t n, const double* __restrict__ mean2d,
                                      const double* __restrict__ cov2d,
                                      const double* __restrict__ opacity, Geom g) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i == 0) g.dev_counts[0] = n;
  if (i >= n) return;
  g.order[i] = (int32_t)i;
  g.g_mean[i] = make_double2(mean2d[2 * i], mean2d[2 * i + 1]);
  g.g_cov[i] = make_double2(cov2d[4 * i], cov2d[4 * i + 3]);
  g.g_conop[i] = make_double4(0.0, 0.0, 0.0, opacity[i]);
  g.g_color[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

int tile_bin_begin(int64_t n, const double* mean2d, const double* cov2d, const double* opacity,
                   const ss_camera* cam, const ss_raster_settings* s, void* geom,
                   int64_t* counts_host, cudaStream_t st) {
  SS_TRY(check_raster(nullptr, cam, s));
  Geom g = plan_geom(geom, n, cam, s);
  SS_CUDA(cudaMemsetAsync(g.dev_counts, 0, 3 * sizeof(int64_t), st));
  if (n > 0) {
    tile_bin_setup_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(n, mean2d, cov2d, opacity, g);
    SS_CHECK_LAUNCH("tile_bin_setup_kernel");
    SS_CUDA(cudaMemsetAsync(g.scan_lb, 0, (g.scan_blocks + 1) * sizeof(unsigned long long), st));
    rank_kernel<<<(unsigned)cdiv(n, kScanThreads * kScanRanks), kScanThreads, 0, st>>>(make_cam(cam),
                                                                                   *s, n, g);
    SS_CHECK_LAUNCH("rank_kernel");
  } else {
    finish_counts_kernel<<<1, 1, 0, st>>>(g, n);
    SS_CHECK_LAUNCH("finish_counts_kernel");
  }
  if (counts_host)
    SS_CUDA(cudaMemcpyAsync(counts_host, g.dev_counts, 2 * sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
  return SS_OK;
}

int tile_bin_finish(int64_t n, const ss_camera* cam, const ss_raster_settings* s, void* geom,
                    void* bins, int64_t pairs, cudaStream_t st) {
  Geom g = plan_geom(geom, n, cam, s);
  Bins b = plan_bins(bins, pairs);
  const int ntx = ntiles_x(cam, s), nty = ntiles_y(cam, s);
  const int64_t ntiles = (int64_t)ntx * nty;
  (void)ntiles;
  return bin_pairs(cam, s, n, g, b, nullptr, 0, st);
}

}  // namespace ss

using namespace ss;

extern "C" {

size_t ss_raster_geom_bytes(int64_t n, const ss_camera* cam, const ss_raster_settings* s) {
  if (check_raster(nullptr, cam, s) != SS_OK) return 0;
  return plan_geom(nullptr, n, cam, s).total;
}

size_t ss_raster_bin_bytes(int64_t n_pairs, int64_t n, const ss_camera* cam,
                           const ss_raster_settings* s) {
  (void)n, (void)cam, (void)s;
  return plan_bins(nullptr, n_pairs).total;
}

int ss_raster_forward_begin(const ss_cloud* cloud, const ss_camera* cam,
                            const ss_raster_settings* s, void* geom, int64_t* counts_host,
                            void* stream) {
  return raster_begin(cloud, cam, s, geom, counts_host, as_stream(stream));
}

int ss_raster_forward_finish(const ss_cloud* cloud, const ss_camera* cam,
                             const ss_raster_settings* s, void* geom, void* bins,
                             int64_t n_pairs, float* image, float* alpha_map, int32_t* touch,
                             void* stream) {
  return raster_finish(cloud, cam, s, geom, bins, n_pairs, image, alpha_map, touch, nullptr, 0,
                       as_stream(stream), n_pairs);
}

int ss_raster_backward(const ss_cloud* cloud, const ss_camera* cam, const ss_raster_settings* s,
                       void* geom, void* bins, int64_t n_pairs, const float* d_image,
                       const ss_cloud_grads* grads, void* stream) {
  return raster_backward(cloud, cam, s, geom, bins, n_pairs, d_image, grads, 1,
                         as_stream(stream), n_pairs, 0, nullptr, 0);
}

int ss_raster_forward_finish_banded(const ss_cloud* cloud, const ss_camera* cam,
                                    const ss_raster_settings* s, void* geom, void* bins,
                                    int64_t bin_capacity, int64_t n_pairs, float* image,
                                    float* alpha_map, int32_t* touch, void* stream) {
  return raster_finish(cloud, cam, s, geom, bins, bin_capacity, image, alpha_map, touch, nullptr,
                       0, as_stream(stream), n_pairs);
}

int ss_raster_backward_banded(const ss_cloud* cloud, const ss_camera* cam,
                              const ss_raster_settings* s, void* geom, void* bins,
                              int64_t bin_capacity, int64_t n_pairs, const float* d_image,
                              const ss_cloud_grads* grads, void* stream) {
  return raster_backward(cloud, cam, s, geom, bins, bin_capacity, d_image, grads, 1,
                         as_stream(stream), n_pairs, 0, nullptr, 0);
}

int ss_tile_bin_begin(int64_t n, const double* mean2d, const double* cov2d, const double* opacity,
                      const ss_camera* cam, const ss_raster_settings* s, void* geom,
                      int64_t* counts_host, void* stream) {
  return tile_bin_begin(n, mean2d, cov2d, opacity, cam, s, geom, counts_host, as_stream(stream));
}

int ss_tile_bin_finish(int64_t n, const ss_camera* cam, const ss_raster_settings* s, void* geom,
                       void* bins, int64_t n_pairs, int32_t* tile_ranges, int32_t* members,
                       void* stream) {
  SS_TRY(tile_bin_finish(n, cam, s, geom, bins, n_pairs, as_stream(stream)));
  return ss_raster_tile_lists(cam, s, geom, bins, n_pairs, n, tile_ranges, members, nullptr,
                              stream);
}

int ss_raster_tile_lists(const ss_camera* cam, const ss_raster_settings* s, const void* geom,
                         const void* bins, int64_t n_pairs, int64_t n, int32_t* tile_ranges,
                         int32_t* members, int32_t* indices, void* stream) {
  SS_TRY(check_raster(nullptr, cam, s));
  cudaStream_t st = as_stream(stream);
  Geom g = plan_geom(const_cast<void*>(geom), n, cam, s);
  Bins b = plan_bins(const_cast<void*>(bins), n_pairs);
  const int64_t ntiles = (int64_t)ntiles_x(cam, s) * ntiles_y(cam, s);
  if (tile_ranges && ntiles > 0) {
    tile_lists_kernel<<<(unsigned)cdiv(ntiles, 256), 256, 0, st>>>(ntiles, g.ranges, tile_ranges);
    SS_CHECK_LAUNCH("tile_lists_kernel");
  }
  if (members && n_pairs > 0)
    SS_CUDA(cudaMemcpyAsync(members, b.vals_out, n_pairs * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, st));
  if (indices && n > 0)
    SS_CUDA(cudaMemcpyAsync(indices, g.order, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  return SS_OK;
}

}  // extern "C"
