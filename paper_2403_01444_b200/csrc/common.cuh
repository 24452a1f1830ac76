// Shared device/host helpers for the sm_100a Stage-1 kernels.
// Math restates gaussians.py / sh.py / cameras.py of the reference
// (/root/reference/pkg/src/splatstream/), templated on float/double.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <string>

#include "ss_b200.h"

namespace ss {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
extern std::atomic<int64_t> g_launches;

#define SS_CHECK_LAUNCH(name)                                                    \
  do {                                                                           \
    ::ss::g_launches.fetch_add(1, std::memory_order_relaxed);                    \
    cudaError_t _e = cudaGetLastError();                                         \
    if (_e != cudaSuccess) {                                                     \
      ::ss::set_error(std::string(name) + ": " + cudaGetErrorString(_e));        \
      return SS_ERR_CUDA;                                                        \
    }                                                                            \
  } while (0)

#define SS_CUDA(call)                                                            \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::ss::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));       \
      return SS_ERR_CUDA;                                                        \
    }                                                                            \
  } while (0)

#define SS_TRY(call)                                                             \
  do {                                                                           \
    int _s = (call);                                                             \
    if (_s != SS_OK) return _s;                                                  \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// bump allocator over a caller-provided workspace
struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t count) {
    off = align_up(off);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
  size_t bytes() const { return align_up(off); }
};

// ------------------------------------------------------------ constants
constexpr double kShC0 = 0.28209479177387814;  // sh.py:26
constexpr double kShC1 = 0.4886025119029199;   // sh.py:27
// degree 2/3: orthonormal real SH without the Condon-Shortley phase (the
// convention of the reference's degree-1 +y,+z,+x basis); extension.
constexpr double kShC2a = 1.0925484305920792, kShC2b = 0.31539156525252005,
                 kShC2c = 0.5462742152960396;
constexpr double kShC3a = 0.5900435899266435, kShC3b = 2.890611442640554,
                 kShC3c = 0.4570457994644658, kShC3d = 0.3731763325901154,
                 kShC3e = 1.445305721320277;
constexpr double kLowpass = 0.3;  // cameras.py:27

// sample directions + B^{-T} for the band-2/3 SH rotation (M_l = BinvT Y(R^T D)^T)
struct ShRotConst {
  float dirs2[5][3];
  float binvT2[5][5];
  float dirs3[7][3];
  float binvT3[7][7];
};
void build_shrot_host(ShRotConst* h);  // lib.cu
int ensure_shrot_const();               // ntc.cu (owns the __constant__ copy)

// ------------------------------------------------------------ quaternions
template <class T>
struct Q4 {
  T w, x, y, z;
};

template <class T>
__host__ __device__ inline void quat_to_rot(T w, T x, T y, T z, T r[3][3]) {
  // gaussians.py:68-85 (polynomial map, q assumed unit)
  r[0][0] = T(1) - T(2) * (y * y + z * z);
  r[0][1] = T(2) * (x * y - w * z);
  r[0][2] = T(2) * (x * z + w * y);
  r[1][0] = T(2) * (x * y + w * z);
  r[1][1] = T(1) - T(2) * (x * x + z * z);
  r[1][2] = T(2) * (y * z - w * x);
  r[2][0] = T(2) * (x * z - w * y);
  r[2][1] = T(2) * (y * z + w * x);
  r[2][2] = T(1) - T(2) * (x * x + y * y);
}

// sum_ij g[i][j] dR_ij/dq  (gaussians.py:88-106)
template <class T>
__host__ __device__ inline void quat_to_rot_vjp(T w, T x, T y, T z, const T g[3][3], T out[4]) {
  out[0] = T(2) * (-z * g[0][1] + y * g[0][2] + z * g[1][0] - x * g[1][2] - y * g[2][0] +
                   x * g[2][1]);
  out[1] = T(2) * (y * g[0][1] + z * g[0][2] + y * g[1][0] - T(2) * x * g[1][1] - w * g[1][2] +
                   z * g[2][0] + w * g[2][1] - T(2) * x * g[2][2]);
  out[2] = T(2) * (-T(2) * y * g[0][0] + x * g[0][1] + w * g[0][2] + x * g[1][0] + z * g[1][2] -
                   w * g[2][0] + z * g[2][1] - T(2) * y * g[2][2]);
  out[3] = T(2) * (-T(2) * z * g[0][0] - w * g[0][1] + x * g[0][2] + w * g[1][0] -
                   T(2) * z * g[1][1] + y * g[1][2] + x * g[2][0] + y * g[2][1]);
}

// Hamilton product a*b, wxyz (gaussians.py:51-65)
template <class T>
__host__ __device__ inline void quat_mul(const T a[4], const T b[4], T o[4]) {
  o[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  o[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  o[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  o[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}

// ------------------------------------------------------------ SH basis
// basis values (K) at direction d (sh.py:35-42 for degree <= 1)
template <class T>
__host__ __device__ inline void sh_basis(int deg, T x, T y, T z, T* b) {
  b[0] = T(kShC0);
  if (deg < 1) return;
  b[1] = T(kShC1) * y;
  b[2] = T(kShC1) * z;
  b[3] = T(kShC1) * x;
  if (deg < 2) return;
  b[4] = T(kShC2a) * x * y;
  b[5] = T(kShC2a) * y * z;
  b[6] = T(kShC2b) * (T(2) * z * z - x * x - y * y);
  b[7] = T(kShC2a) * x * z;
  b[8] = T(kShC2c) * (x * x - y * y);
  if (deg < 3) return;
  b[9] = T(kShC3a) * y * (T(3) * x * x - y * y);
  b[10] = T(kShC3b) * x * y * z;
  b[11] = T(kShC3c) * y * (T(4) * z * z - x * x - y * y);
  b[12] = T(kShC3d) * z * (T(2) * z * z - T(3) * x * x - T(3) * y * y);
  b[13] = T(kShC3c) * x * (T(4) * z * z - x * x - y * y);
  b[14] = T(kShC3e) * z * (x * x - y * y);
  b[15] = T(kShC3a) * x * (x * x - T(3) * y * y);
}

// g_d += sum_k gb[k] * d basis_k / d d   (sh.py:62-81 for degree <= 1)
template <class T>
__host__ __device__ inline void sh_basis_vjp(int deg, T x, T y, T z, const T* gb, T g[3]) {
  if (deg < 1) return;
  g[1] += T(kShC1) * gb[1];
  g[2] += T(kShC1) * gb[2];
  g[0] += T(kShC1) * gb[3];
  if (deg < 2) return;
  const T a = T(kShC2a), b = T(kShC2b), c = T(kShC2c);
  g[0] += a * y * gb[4] + a * z * gb[7] - T(2) * b * x * gb[6] + T(2) * c * x * gb[8];
  g[1] += a * x * gb[4] + a * z * gb[5] - T(2) * b * y * gb[6] - T(2) * c * y * gb[8];
  g[2] += a * y * gb[5] + T(4) * b * z * gb[6] + a * x * gb[7];
  if (deg < 3) return;
  const T c3 = T(kShC3a), c2 = T(kShC3b), c1 = T(kShC3c), c0 = T(kShC3d), ch = T(kShC3e);
  g[0] += T(6) * c3 * x * y * gb[9] + c2 * y * z * gb[10] - T(2) * c1 * x * y * gb[11] -
          T(6) * c0 * x * z * gb[12] + c1 * (T(4) * z * z - T(3) * x * x - y * y) * gb[13] +
          T(2) * ch * x * z * gb[14] + c3 * (T(3) * x * x - T(3) * y * y) * gb[15];
  g[1] += c3 * (T(3) * x * x - T(3) * y * y) * gb[9] + c2 * x * z * gb[10] +
          c1 * (T(4) * z * z - x * x - T(3) * y * y) * gb[11] - T(6) * c0 * y * z * gb[12] -
          T(2) * c1 * x * y * gb[13] - T(2) * ch * y * z * gb[14] - T(6) * c3 * x * y * gb[15];
  g[2] += c2 * x * y * gb[10] + T(8) * c1 * y * z * gb[11] +
          c0 * (T(6) * z * z - T(3) * x * x - T(3) * y * y) * gb[12] +
          T(8) * c1 * x * z * gb[13] + ch * (x * x - y * y) * gb[14];
}

__host__ __device__ inline int sh_degree_of(int k) {
  return k >= 16 ? 3 : (k >= 9 ? 2 : (k >= 4 ? 1 : 0));
}

// ------------------------------------------------------------ small helpers
__device__ inline float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// vector reduction into global memory (sm_90+: red.global.add.v2.f32)
__device__ inline void red_add_v2(float* addr, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(a), "f"(b) : "memory");
}
__device__ inline void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

}  // namespace ss

// Opt a kernel into `bytes` of dynamic shared memory once per (kernel, device):
// the attribute persists, and re-setting it on every launch costs host time.
namespace ss {
cudaError_t smem_attr_once(const void* kernel, int bytes);
template <class K>
inline cudaError_t smem_attr_once(K* kernel, int bytes) {
  return smem_attr_once(reinterpret_cast<const void*>(kernel), bytes);
}
}  // namespace ss

// ---------------------------------------------------------------- internal API
namespace ss {
int raster_begin(const ss_cloud* cl, const ss_camera* cam, const ss_raster_settings* s,
                 void* geom, int64_t* counts_host, cudaStream_t st);
// cap: pairs the bins workspace holds; total: the view's pairs if known on the
// host (above cap: binned and blended in bands of tile rows), else <= cap
int raster_finish(const ss_cloud* cl, const ss_camera* cam, const ss_raster_settings* s,
                  void* geom, void* bins, int64_t cap, float* image, float* alpha,
                  int32_t* touch, uint32_t* status, int cull, cudaStream_t st, int64_t total);
// device pointer to [survivors, pairs] of the last raster_begin on `geom`
const int64_t* raster_counts(void* geom, int64_t n, const ss_camera* cam,
                             const ss_raster_settings* s);
int raster_backward(const ss_cloud* cl, const ss_camera* cam, const ss_raster_settings* s,
                    void* geom, void* bins, int64_t cap, const float* d_image,
                    const ss_cloud_grads* grads, int full, cudaStream_t st, int64_t total,
                    int cull, uint32_t* status, int accumulate = 0);
}  // namespace ss

// ---------------------------------------------------------------- phase timing
// CUDA events recorded on the launching stream around each hot-path phase when
// enabled with ss_profile_enable(1); read back with ss_profile_read().
namespace ss {
// One phase per kernel, except depth_sort / tile_sort (radix passes + tie fix-up)
// and rank_scan (rank kernel + scan).
enum Phase {
  PH_GATHER = 0, PH_DECODER_FWD, PH_TRANSFORM, PH_PROJECT, PH_DEPTH_SORT, PH_RANK_SCAN,
  PH_DUPLICATE, PH_TILE_SORT, PH_RANGES, PH_BLEND_FWD, PH_SSIM_MAP, PH_SSIM_GRAD,
  PH_BLEND_BWD, PH_GAUSS_BWD, PH_TRANSFORM_BWD, PH_DECODER_BWD, PH_SCATTER, PH_ADAM,
  PH_COUNT
};
void prof_begin(int phase, cudaStream_t s);
void prof_end(int phase, cudaStream_t s);

// Device-count stable radix sort of (tile key, rank) pairs (binsort.cu)
struct BinSortWS {
  uint32_t* hist;    // [4][256] digit histograms, then the pass tickets
  uint32_t* status;  // [passes][max_blocks][256] look-back words
  int64_t max_blocks;
  int max_passes;
  int steps;  // items per thread of a pass tile
};
BinSortWS binsort_plan(Carve& c, int64_t capacity, int max_passes);
// Stage-1 iterations zero the per-iteration scratch of the geometry workspace
// and the loss (depth-sort look-back words and histograms, counters, reverse-
// blend accumulators, loss sums) with ONE kernel (a memset node costs ~1.5 us
// in a replayed graph); inside such a scope those memsets are skipped.  The
// bin workspace keeps its own clears (the host may replace it mid-iteration).
extern thread_local bool t_prezeroed;
struct PrezeroScope {
  bool prev;
  explicit PrezeroScope(bool on) : prev(t_prezeroed) { t_prezeroed = on; }
  ~PrezeroScope() { t_prezeroed = prev; }
};
int raster_zero_iteration(void* geom, int64_t n, const ss_camera* cam, const ss_raster_settings* s,
                          void* bins, int64_t cap, void* extra, size_t extra_bytes,
                          cudaStream_t st);
int binsort_passes(int key_bits);
// zero the histograms, tickets and look-back words (before a producer that
// accumulates the histograms itself with bs_hist_add, then hist_ready = true)
int binsort_clear(const BinSortWS& w, int key_bits, cudaStream_t st);
int binsort_run(const BinSortWS& w, uint32_t* keys_tmp, uint32_t* vals_tmp, uint32_t* keys_out,
                uint32_t* vals_out, const int64_t* d_n, int64_t cap, int key_bits,
                cudaStream_t st, bool hist_ready = false);

// Producer-side histogram for binsort (8-bit digits, up to 4 passes): add a
// key into the block's shared histogram sh[pass][digit]; bs_hist_flush adds
// the block's counts to the global ones after a __syncthreads().
__device__ __forceinline__ void bs_hist_add(uint32_t (*sh)[256], uint32_t key, int key_bits) {
  for (int p = 0; 8 * p < key_bits; ++p) {
    const int bits = key_bits - 8 * p < 8 ? key_bits - 8 * p : 8;
    atomicAdd(&sh[p][(key >> (8 * p)) & ((1u << bits) - 1)], 1u);
  }
}
__device__ __forceinline__ void bs_hist_flush(const uint32_t (*sh)[256], uint32_t* hist,
                                              int key_bits) {
  const int passes = (key_bits + 7) / 8;
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
    const uint32_t v = sh[i >> 8][i & 255];
    if (v) atomicAdd(hist + i, v);
  }
}

// NTC pipeline pieces (ntc.cu): features X and their gradient dX are (n, xs)
// row-major in HBM between the gather / decoder / scatter kernels; out7 and g7
// are (n, 8) (or stride 7 on the reference-shaped API).
struct NtcScratch {
  float *X, *dX, *out7, *g7;
  uint64_t* relu;  // (n, 2) ReLU masks of the decoder forward, reused by its backward
  int xs;
};
size_t ntc_scratch_bytes(const ss_mlp* mlp, int64_t n);
NtcScratch ntc_scratch(void* base, const ss_mlp* mlp, int64_t n);
int ntc_forward_run(const ss_grid* g, const ss_mlp* mlp, int64_t n, const float* means,
                    const int32_t* rows, const float* tables, const float* params, float* X, int xs,
                    float* out, int os, uint64_t* relu, uint32_t* status, cudaStream_t st);
int ntc_backward_run(const ss_grid* g, const ss_mlp* mlp, int64_t n, const float* means,
                     const int32_t* rows, const float* params, const float* X, int xs,
                     const float* g_out, int gs, const uint64_t* relu, float* dX,
                     float* g_tables, float* g_params, cudaStream_t st);
// K1b alone: g_tables += corner-weighted dX (ntc.py:278-288)
int ntc_scatter_run(const ss_grid* g, int64_t n, const float* means, const int32_t* rows,
                    const float* dX, int xs, float* g_tables, cudaStream_t st);
// rows: cloud row of thread j; pos (nullable = identity): its slot in out7 / g7
int transform_run(const ss_cloud* src, int64_t n, const int32_t* rows, const int32_t* pos,
                  const float* out7, int os, int rotate_sh, float* tm, float* tr, float* ts,
                  uint32_t* status, cudaStream_t st);
// live (nullable): per-Gaussian flag of the raster backward's `contributed`;
// rows without it get a zero g7 row without reading their gradients
int transform_vjp_run(const ss_cloud* src, int64_t n, const int32_t* rows, const int32_t* pos,
                      const float* out7, int os, int rotate_sh, const float* dm, const float* dr,
                      const float* ds, float* g7, int gs, cudaStream_t st,
                      const uint8_t* live = nullptr);
}  // namespace ss

// decoder on tensor cores (mlp_tc.cu); mode 0 = FFMA fp32, 1 = 3xTF32, 2 = tf32
namespace ss {
int mlp_mode();
int mlp_fwd_tc(int in_pad, int n_hidden, int f16, int64_t n, const float* X, int xs, const float* params,
               float* out, int os, uint64_t* relu_masks, cudaStream_t st);
int mlp_bwd_tc(int in_pad, int n_hidden, int f16, int64_t n, const float* X, int xs, const float* g,
               int gs, const uint64_t* relu_masks, const float* params, float* dX,
               float* g_params, cudaStream_t st);
}  // namespace ss
