// Fused L1 + D-SSIM loss and its image gradient (KL) on sm_100a.
// Reference: losses.py:36-148 (/root/reference/pkg/src/splatstream/):
//   L = (1-lam) mean|x-y| + lam (1 - mean_valid SSIM) / 2,
// 11x11 Gaussian window (sigma 1.5), VALID windows only, mean over windows x
// channels; the SSIM adjoint is a FULL convolution of three per-window maps.
// Separable 11-tap strip walks (below) in fp32, window moments on shifted data.
#include "common.cuh"

namespace ss {

constexpr int WIN = 11, HALO = WIN - 1;
constexpr int SW = 64;   // strip width: a warp per (strip, row chunk, channel), two columns per lane
constexpr int RW = SW + HALO;  // input columns of a strip
constexpr int RWP = RW + 2;    // padded row (float2 loads)
constexpr int RCH = 32;        // output rows per chunk
constexpr int WPB = 4;         // warps per CTA (independent, warp-level sync only)

struct LossParams {
  int H, W, Hv, Wv, C;
  int Wp;          // row pitch of the maps (Wv rounded up to the strip width: aligned float2)
  double g[WIN];
  float gf[WIN];  // fp32 copy: FFMA operands straight from the parameter bank
  double c1, c2, lam, up;  // up = -lam / (2 n_windows)
  double l1w;              // (1 - lam) / (H W C)
};

// Both passes walk a 64-column strip down a chunk of rows, one warp per
// (strip, chunk, channel) and two adjacent output columns per lane.  Each input
// row is staged once in the warp's shared-memory row (double-buffered); a lane
// reads its 12 taps per quantity as six float2 loads (the two columns share 10)
// and filters it horizontally; the vertical pass keeps, per column and
// quantity, 11 rotating accumulators in registers: acc[j] = partial sum of
// output row yi - 10 + j, each input row completes acc[0] and shifts the rest
// down inside the FMAs.

// pass 1: valid windows -> SSIM (summed) and the three adjoint maps
// (losses.py:121-137): dL/dmu_x part, dL/dsigma_xx, dL/dsigma_xy (all / lam-scale)
//
// Window moments are accumulated in fp32 on shifted data: every warp subtracts
// a per-channel constant (the pixel at its first row, strip centre) from x and
// y.  Variances and the covariance are shift-invariant, so the shift removes
// the E[x^2] - mu^2 cancellation that would otherwise cost fp32 its accuracy in
// flat regions; the means get the constant added back.  The per-input-column
// quantities are x, y, x^2 + y^2 (SSIM needs only the sum of the variances) and
// xy.
__global__ void __launch_bounds__(32 * WPB) ssim_map_kernel(LossParams lp,
                                                          const float* __restrict__ img,
                                                          const float* __restrict__ tgt,
                                                          float* __restrict__ maps,
                                                          double* __restrict__ sums) {
  constexpr int NQ = 4;
  __shared__ __align__(16) float sv[WPB][2][NQ][RWP];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int c = blockIdx.z, C = lp.C;
  const int x0 = blockIdx.x * SW, oy0 = (blockIdx.y * WPB + wl) * RCH;
  if (oy0 >= lp.Hv) return;  // warp-uniform; warp-level synchronisation only
  const int oy1 = min(oy0 + RCH, lp.Hv), iy1 = oy1 + HALO;
  const int64_t cs = ((int64_t)oy0 * lp.W + min(x0 + SW / 2, lp.W - 1)) * C + c;
  const float shx = __ldg(img + cs), shy = __ldg(tgt + cs);
  float (*buf)[NQ][RWP] = sv[wl];
  float g[WIN];
#pragma unroll
  for (int k = 0; k < WIN; ++k) g[k] = lp.gf[k];
  // staging: lane covers input columns lane, lane + 32, lane + 64 (< RW); the
  // raw values of the row after next are fetched into registers one step
  // ahead, so their global latency overlaps the current row's filtering
  float rx[3], ry[3];
  auto fetch = [&](int yi) {
    const bool row_ok = yi < lp.H;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int e = lane + 32 * m;
      const bool ok = e < RW && row_ok && x0 + e < lp.W;
      const int64_t o = ((int64_t)yi * lp.W + x0 + e) * C + c;
      rx[m] = ok ? __ldg(img + o) : shx;
      ry[m] = ok ? __ldg(tgt + o) : shy;
    }
  };
  auto stage = [&](int b) {
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int e = lane + 32 * m;
      if (e < RW) {
        const float xv = rx[m] - shx, yv = ry[m] - shy;
        buf[b][0][e] = xv;
        buf[b][1][e] = yv;
        buf[b][2][e] = fmaf(xv, xv, yv * yv);
        buf[b][3][e] = xv * yv;
      }
    }
  };
  float acc[2][NQ][WIN];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int j = 0; j < WIN; ++j) acc[u][q][j] = 0.f;
  double ssum = 0.0;
  const float c1f = (float)lp.c1, c2f = (float)lp.c2;
  const int64_t plane = (int64_t)lp.Hv * lp.Wp;
  const int col = x0 + 2 * lane;  // this lane's first output column
  fetch(oy0);
  stage(0);
  fetch(oy0 + 1);
  __syncwarp();
  for (int yi = oy0; yi < iy1; ++yi) {
    const int cur = (yi - oy0) & 1;
    if (yi + 1 < iy1) {  // next row into the other buffer, then fetch the one after
      stage(cur ^ 1);
      fetch(yi + 2);
    }
    // horizontal sums of row yi at columns col, col + 1
    float h[2][NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float2* row = reinterpret_cast<const float2*>(&buf[cur][q][2 * lane]);
      float v[12];
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const float2 p2 = row[t];
        v[2 * t] = p2.x;
        v[2 * t + 1] = p2.y;
      }
      float h0 = 0.f, h1 = 0.f;
#pragma unroll
      for (int k = 0; k < WIN; ++k) {
        h0 = fmaf(g[k], v[k], h0);
        h1 = fmaf(g[k], v[k + 1], h1);
      }
      h[0][q] = h0;
      h[1][q] = h1;
    }
    // output row yi - 10 completes with tap 10; the others shift down one row
    float fin[2][NQ];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        fin[u][q] = fmaf(g[HALO], h[u][q], acc[u][q][0]);
#pragma unroll
        for (int j = 0; j < HALO; ++j) acc[u][q][j] = fmaf(g[HALO - 1 - j], h[u][q], acc[u][q][j + 1]);
        acc[u][q][HALO] = 0.f;
      }
    const int o = yi - HALO;
    if (o >= oy0) {
      float r[3][2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        // per-window algebra in fp32 (the maps are stored in fp32 anyway); the
        // shifted moments carry no cancellation, the SSIM sum is kept in fp64
        const float mx0 = fin[u][0], my0 = fin[u][1];
        const float vsum = fin[u][2] - mx0 * mx0 - my0 * my0, cxy = fin[u][3] - mx0 * my0;
        const float mx = mx0 + shx, my = my0 + shy;
        const float a1 = 2.f * mx * my + c1f, a2 = 2.f * cxy + c2f;
        const float b1 = mx * mx + my * my + c1f, b2 = vsum + c2f;
        const float inv = 1.f / (b1 * b2);
        const float sv_ = a1 * a2 * inv;
        if (col + u < lp.Wv) ssum += (double)sv_;
        // one division: sv / b1 = sv b2 inv, sv / b2 = sv b1 inv
        const float ga1 = a2 * inv, ga2 = a1 * inv, gb1 = -sv_ * b2 * inv, gb2 = -sv_ * b1 * inv;
        r[0][u] = 2.f * (my * (ga1 - ga2) + mx * (gb1 - gb2));
        r[1][u] = gb2;
        r[2][u] = 2.f * ga2;
      }
      if (col < lp.Wv) {  // col + 1 < Wp always: the pitch pads to the strip width
        const int64_t oo = (int64_t)o * lp.Wp + col;
#pragma unroll
        for (int m = 0; m < 3; ++m)
          *reinterpret_cast<float2*>(maps + (m * C + c) * plane + oo) = make_float2(r[m][0], r[m][1]);
      }
    }
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, off);
  if (lane == 0 && ssum != 0.0) atomicAdd(&sums[0], ssum);
}

// pass 2: full convolution of the maps + L1 term -> dL/dimage; sum |x - y|
// (losses.py:106-108, :138-145).  Same strip walk: map rows [oy0 - 10, oy1)
// feed output rows [oy0, oy1), map columns [x0 - 10, x0 + 64).
// acc[i] = partial sum of output row r + i; map row r completes acc[0].
__global__ void __launch_bounds__(32 * WPB) ssim_grad_kernel(LossParams lp,
                                                           const float* __restrict__ img,
                                                           const float* __restrict__ tgt,
                                                           const float* __restrict__ maps,
                                                           float* __restrict__ grad,
                                                           double* __restrict__ sums) {
  constexpr int NQ = 3;
  __shared__ __align__(16) float sm[WPB][2][NQ][RWP];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int c = blockIdx.z, C = lp.C;
  const int x0 = blockIdx.x * SW, oy0 = (blockIdx.y * WPB + wl) * RCH;
  if (oy0 >= lp.H) return;
  const int oy1 = min(oy0 + RCH, lp.H);
  const int ry0 = max(oy0 - HALO, 0), ry1 = min(oy1, lp.Hv);  // map rows that contribute
  const int64_t plane = (int64_t)lp.Hv * lp.Wp;
  float (*buf)[NQ][RWP] = sm[wl];
  float g[WIN];
#pragma unroll
  for (int k = 0; k < WIN; ++k) g[k] = lp.gf[k];
  // staging: lane covers map columns x0 - 10 + e, e = lane, lane + 32, lane + 64;
  // one row fetched into registers ahead of its staging
  float rm[3][NQ];
  auto fetch = [&](int r) {
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int e = lane + 32 * m, vx = x0 - HALO + e;
      const bool ok = e < RW && r < ry1 && vx >= 0 && vx < lp.Wv;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        rm[m][q] = ok ? __ldg(maps + (q * C + c) * plane + (int64_t)r * lp.Wp + vx) : 0.f;
    }
  };
  auto stage = [&](int b) {
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int e = lane + 32 * m;
      if (e < RW)
#pragma unroll
        for (int q = 0; q < NQ; ++q) buf[b][q][e] = rm[m][q];
    }
  };
  float acc[2][NQ][WIN];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int j = 0; j < WIN; ++j) acc[u][q][j] = 0.f;
  double l1 = 0.0;
  const int px = x0 + 2 * lane;  // this lane's first output column
  // output row r needs map rows r - 10 .. r; walk map rows from ry0 and emit
  // output row r once map row r (or the last map row) has been folded in
  const int rend = oy1;  // walk rows [ry0, rend): rows >= ry1 contribute zeros
  float xn[2] = {0.f, 0.f}, tn[2] = {0.f, 0.f};
  if (ry0 >= oy0)  // (ry0 == oy0 == 0): the first output row's pixels
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const bool ok = px + u < lp.W;
      const int64_t o = ((int64_t)ry0 * lp.W + px + u) * C + c;
      xn[u] = ok ? __ldg(img + o) : 0.f;
      tn[u] = ok ? __ldg(tgt + o) : 0.f;
    }
  fetch(ry0);
  stage(0);
  fetch(ry0 + 1);
  __syncwarp();
  for (int r = ry0; r < rend; ++r) {
    const int cur = (r - ry0) & 1;
    if (r + 1 < rend) {
      stage(cur ^ 1);
      fetch(r + 2);
    }
    // horizontal full convolution at output columns px, px + 1: map cols px - j
    float h[2][NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float2* row = reinterpret_cast<const float2*>(&buf[cur][q][2 * lane]);
      float v[12];
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const float2 p2 = row[t];
        v[2 * t] = p2.x;
        v[2 * t + 1] = p2.y;
      }
      // buffer index e = col - x0 + 10: output col px + u, tap j -> e = 2 lane + u + 10 - j
      float h0 = 0.f, h1 = 0.f;
#pragma unroll
      for (int j = 0; j < WIN; ++j) {
        h0 = fmaf(g[j], v[HALO - j], h0);
        h1 = fmaf(g[j], v[HALO + 1 - j], h1);
      }
      h[0][q] = h0;
      h[1][q] = h1;
    }
    // output row r completes with tap 0; rows r + 1 .. r + 10 shift down
    float fin[2][NQ];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        fin[u][q] = fmaf(g[0], h[u][q], acc[u][q][0]);
#pragma unroll
        for (int i = 0; i < HALO; ++i) acc[u][q][i] = fmaf(g[i + 1], h[u][q], acc[u][q][i + 1]);
        acc[u][q][HALO] = 0.f;
      }
    float xc[2], tc[2];  // this row's image / target (fetched a row ahead)
#pragma unroll
    for (int u = 0; u < 2; ++u) xc[u] = xn[u], tc[u] = tn[u];
    if (r + 1 >= oy0 && r + 1 < oy1)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const bool ok = px + u < lp.W;
        const int64_t o = ((int64_t)(r + 1) * lp.W + px + u) * C + c;
        xn[u] = ok ? __ldg(img + o) : 0.f;
        tn[u] = ok ? __ldg(tgt + o) : 0.f;
      }
    if (r >= oy0) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (px + u >= lp.W) continue;
        const int64_t o = ((int64_t)r * lp.W + px + u) * C + c;
        const float xr = xc[u], tr = tc[u];
        const float d = xr - tr;
        l1 += fabs((double)xr - (double)tr);
        const double sgn = d > 0.f ? 1.0 : (d < 0.f ? -1.0 : 0.0);
        const double back = (double)fin[u][0] + (double)fin[u][1] * 2.0 * xr + (double)fin[u][2] * tr;
        grad[o] = (float)(lp.l1w * sgn + lp.up * back);
      }
    }
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, off);
  if (lane == 0 && l1 != 0.0) atomicAdd(&sums[1], l1);
}

__global__ void loss_finalize_kernel(LossParams lp, const double* sums, double* loss,
                                     uint32_t* status) {
  const double size = (double)lp.H * lp.W * lp.C;
  const double nwin = (double)lp.Hv * lp.Wv * lp.C;
  const double l = (1.0 - lp.lam) * (sums[1] / size) + lp.lam * (1.0 - sums[0] / nwin) / 2.0;
  *loss = l;
  if (!isfinite(l) && status) atomicOr(status, SS_FLAG_NONFINITE);  // errors.py:24-29
}

}  // namespace ss

using namespace ss;

extern "C" {

size_t ss_loss_bytes(int32_t height, int32_t width, int32_t channels) {
  const int64_t hv = height - HALO, wv = width - HALO;
  if (hv <= 0 || wv <= 0) return 256;
  const int64_t wp = (wv + SW - 1) / SW * SW;
  return align_up(2 * sizeof(double)) + align_up((size_t)3 * channels * hv * wp * sizeof(float));
}

int ss_render_loss(const float* image, const float* target, int32_t height, int32_t width,
                   int32_t channels, double lam, double c1, double c2, void* scratch,
                   double* loss_dev, float* d_image, uint32_t* status, void* stream) {
  if (channels < 1 || channels > 3) {
    set_error("render_loss supports 1-3 channels");
    return SS_ERR_DATA;
  }
  if (height < WIN || width < WIN) {
    set_error("image smaller than the SSIM window");  // losses.py:111-112
    return SS_ERR_DATA;
  }
  cudaStream_t st = as_stream(stream);
  LossParams lp{};
  lp.H = height, lp.W = width, lp.Hv = height - HALO, lp.Wv = width - HALO, lp.C = channels;
  lp.Wp = (lp.Wv + SW - 1) / SW * SW;
  double tot = 0;
  for (int k = 0; k < WIN; ++k) {  // losses.py:36-40 (normalised separably)
    const double a = k - WIN / 2;
    lp.g[k] = std::exp(-(a * a) / (2.0 * 1.5 * 1.5));
    tot += lp.g[k];
  }
  for (int k = 0; k < WIN; ++k) lp.g[k] /= tot;
  for (int k = 0; k < WIN; ++k) lp.gf[k] = (float)lp.g[k];
  lp.c1 = c1, lp.c2 = c2, lp.lam = lam;
  lp.up = -lam / (2.0 * (double)lp.Hv * lp.Wv * channels);
  lp.l1w = (1.0 - lam) / ((double)height * width * channels);
  double* sums = static_cast<double*>(scratch);
  float* maps = reinterpret_cast<float*>(static_cast<char*>(scratch) + align_up(2 * sizeof(double)));
  SS_CUDA(cudaMemsetAsync(sums, 0, 2 * sizeof(double), st));
  dim3 blk(32 * WPB);
  dim3 g1((unsigned)cdiv(lp.Wv, SW), (unsigned)cdiv(cdiv(lp.Hv, RCH), WPB), (unsigned)channels);
  prof_begin(PH_SSIM_MAP, st);
  ssim_map_kernel<<<g1, blk, 0, st>>>(lp, image, target, maps, sums);
  SS_CHECK_LAUNCH("ssim_map_kernel");
  prof_end(PH_SSIM_MAP, st);
  dim3 g2((unsigned)cdiv(lp.W, SW), (unsigned)cdiv(cdiv(lp.H, RCH), WPB), (unsigned)channels);
  prof_begin(PH_SSIM_GRAD, st);
  ssim_grad_kernel<<<g2, blk, 0, st>>>(lp, image, target, maps, d_image, sums);
  SS_CHECK_LAUNCH("ssim_grad_kernel");
  prof_end(PH_SSIM_GRAD, st);
  loss_finalize_kernel<<<1, 1, 0, st>>>(lp, sums, loss_dev, status);
  SS_CHECK_LAUNCH("loss_finalize_kernel");
  return SS_OK;
}

}  // extern "C"
