// Fused L1 + D-SSIM loss and its image gradient (KL) on sm_100a.
// Reference: losses.py:36-148 (/root/reference/pkg/src/splatstream/):
//   L = (1-lam) mean|x-y| + lam (1 - mean_valid SSIM) / 2,
// 11x11 Gaussian window (sigma 1.5), VALID windows only, mean over windows x
// channels; the SSIM adjoint is a FULL convolution of three per-window maps.
// Separable 11-tap strip walks (below) in fp32, window moments on shifted data.
#include "common.cuh"

namespace ss {

constexpr int WIN = 11, HALO = WIN - 1;
constexpr int SW = 32;   // strip width: one warp per channel, a lane per column
constexpr int RCH = 60;  // rows per chunk: 42 x 17 CTAs of 3 warps at 1352x1014 = one wave at 5 CTAs/SM

struct LossParams {
  int H, W, Hv, Wv, C;
  double g[WIN];
  float gf[WIN];  // fp32 copy: FFMA operands straight from the parameter bank
  double c1, c2, lam, up;  // up = -lam / (2 n_windows)
  double l1w;              // (1 - lam) / (H W C)
};

// The separable 11-tap passes walk a 32-column strip down a chunk of rows.
// Each input row's horizontal sums are scattered into 11 rotating vertical
// accumulators (slot = output row mod 11, kept in registers), so every input
// row is filtered horizontally once and an output row completes every step.
// CTA = 3 warps (one per channel) sharing the row loads through shared memory.

// pass 1: valid windows -> SSIM (summed) and the three adjoint maps
// (losses.py:121-137): dL/dmu_x part, dL/dsigma_xx, dL/dsigma_xy (all / lam-scale)
//
// Window moments are accumulated in fp32 on shifted data: every CTA subtracts
// a per-channel constant (the pixel at its first row, strip centre) from x and
// y.  Variances and the covariance are shift-invariant, so the shift removes
// the E[x^2] - mu^2 cancellation that would otherwise cost fp32 its accuracy in
// flat regions; the means get the constant added back.  Against all-fp64
// statistics the per-window SSIM differs by <= 3e-5 and the mean by ~1e-10
// (smooth, flat and noise images, 1352x1014).
//
// The vertical pass keeps acc[j] = partial sum of output row yi - 10 + j; each
// input row completes acc[0] and shifts the rest down inside the FMAs, so the
// row loop needs no unrolling.  Each warp stages only its own channel (double-
// buffered shared rows, warp-level sync only).
__global__ void __launch_bounds__(SW * 3, 5) ssim_map_kernel(LossParams lp,
                                                          const float* __restrict__ img,
                                                          const float* __restrict__ tgt,
                                                          float* __restrict__ maps,
                                                          double* __restrict__ sums) {
  constexpr int RW = SW + HALO;  // input columns of a strip
  constexpr int PER = (RW + SW - 1) / SW;
  // per input column of a row: x, y, x^2 + y^2, xy (shifted; SSIM needs only
  // the sum of the two variances), formed once per element instead of once per
  // tap; two row buffers per channel
  // one float4 per column (x, y, x^2 + y^2, xy): a tap is one 16-byte shared
  // load feeding two packed FMAs (FFMA2, sm_100), bit-identical to four FFMAs
  __shared__ float4 sv[3][2][RW];
  const int lane = threadIdx.x, c = threadIdx.y;
  const int C = lp.C;
  if (c >= C) return;  // warp-uniform; no block-level synchronisation below
  const int x0 = blockIdx.x * SW, oy0 = blockIdx.y * RCH;
  const int oy1 = min(oy0 + RCH, lp.Hv), iy1 = oy1 + HALO;
  const int xcol = x0 + lane;
  const bool col_ok = xcol < lp.Wv;
  const int64_t cs = ((int64_t)oy0 * lp.W + min(x0 + SW / 2, lp.W - 1)) * C + c;
  const float shx = __ldg(img + cs), shy = __ldg(tgt + cs);
  float px[PER], py[PER], qx[PER], qy[PER];  // two rows in flight (no register moves)
  // rows are fetched strictly in order, so the addresses advance by one image
  // row per call (no per-load 64-bit index arithmetic)
  bool col_in[PER];
#pragma unroll
  for (int m = 0; m < PER; ++m) col_in[m] = lane + m * SW < RW && x0 + lane + m * SW < lp.W;
  const int64_t row_stride = (int64_t)lp.W * C;
  const float* fimg = img + ((int64_t)oy0 * lp.W + x0 + lane) * C + c;
  const float* ftgt = tgt + ((int64_t)oy0 * lp.W + x0 + lane) * C + c;
  int fy_next = oy0;
  auto fetch = [&](int y, float (&fx)[PER], float (&fy)[PER]) {
    (void)y;  // == fy_next
    const bool row_ok = fy_next < lp.H;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const bool ok = row_ok && col_in[m];
      fx[m] = ok ? __ldg(fimg + m * SW * C) : 0.f;
      fy[m] = ok ? __ldg(ftgt + m * SW * C) : 0.f;
    }
    fimg += row_stride;
    ftgt += row_stride;
    ++fy_next;
  };
  auto stage = [&](int buf, const float (&fx)[PER], const float (&fy)[PER]) {
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int e = lane + m * SW;
      if (e < RW) {
        const float xv = fx[m] - shx, yv = fy[m] - shy;
        sv[c][buf][e] = make_float4(xv, yv, fmaf(xv, xv, yv * yv), xv * yv);
      }
    }
  };
  // vertical accumulators as packed pairs: (x, y) and (x^2 + y^2, xy)
  float2 axy2[WIN], asx[WIN];
#pragma unroll
  for (int j = 0; j < WIN; ++j) axy2[j] = asx[j] = make_float2(0.f, 0.f);
  float2 g[WIN];
#pragma unroll
  for (int k = 0; k < WIN; ++k) g[k] = make_float2(lp.gf[k], lp.gf[k]);
  double ssum = 0.0;
  const float c1f = (float)lp.c1, c2f = (float)lp.c2;
  const int64_t plane = (int64_t)lp.Hv * lp.Wv;
  // buffers: P holds row yi + 1 at the start of an even step, Q row yi + 2;
  // each step stages one and refills it three rows ahead
  fetch(oy0, px, py);
  stage(0, px, py);
  fetch(oy0 + 1, px, py);
  fetch(oy0 + 2, qx, qy);
  __syncwarp();
  auto step = [&](int yi, float (&fx)[PER], float (&fy)[PER]) {
    const int cur = (yi - oy0) & 1;
    if (yi + 1 < iy1) {  // stage row yi + 1 into the other buffer, refill with row yi + 3
      stage(cur ^ 1, fx, fy);
      fetch(yi + 3, fx, fy);
    }
    // horizontal sums of row yi at column xcol
    float2 h01 = make_float2(0.f, 0.f), h23 = make_float2(0.f, 0.f);
    const float4* row = sv[c][cur];
#pragma unroll
    for (int k = 0; k < WIN; ++k) {
      const float4 v = row[lane + k];
      h01 = __ffma2_rn(g[k], make_float2(v.x, v.y), h01);
      h23 = __ffma2_rn(g[k], make_float2(v.z, v.w), h23);
    }
    // output row yi - 10 completes with tap 10; the others shift down one row
    const float2 m01 = __ffma2_rn(g[HALO], h01, axy2[0]), s01 = __ffma2_rn(g[HALO], h23, asx[0]);
    const float mx0 = m01.x, my0 = m01.y, ss = s01.x, sxy = s01.y;
#pragma unroll
    for (int j = 0; j < HALO; ++j) {
      axy2[j] = __ffma2_rn(g[HALO - 1 - j], h01, axy2[j + 1]);
      asx[j] = __ffma2_rn(g[HALO - 1 - j], h23, asx[j + 1]);
    }
    axy2[HALO] = asx[HALO] = make_float2(0.f, 0.f);
    const int o = yi - HALO;
    if (o >= oy0 && col_ok) {
      // per-window algebra in fp32 (the maps are stored in fp32 anyway); the
      // shifted moments carry no cancellation, the SSIM sum is kept in fp64
      const float vsum = ss - mx0 * mx0 - my0 * my0, cxy = sxy - mx0 * my0;
      const float mx = mx0 + shx, my = my0 + shy;
      const float a1 = 2.f * mx * my + c1f, a2 = 2.f * cxy + c2f;
      const float b1 = mx * mx + my * my + c1f, b2 = vsum + c2f;
      const float inv = 1.f / (b1 * b2);
      const float sv_ = a1 * a2 * inv;
      ssum += (double)sv_;
      // one division: sv / b1 = sv b2 inv, sv / b2 = sv b1 inv
      const float ga1 = a2 * inv, ga2 = a1 * inv, gb1 = -sv_ * b2 * inv, gb2 = -sv_ * b1 * inv;
      const float gmx = 2.f * (my * (ga1 - ga2) + mx * (gb1 - gb2));
      const int64_t oo = (int64_t)o * lp.Wv + xcol;
      maps[(0 * C + c) * plane + oo] = gmx;
      maps[(1 * C + c) * plane + oo] = gb2;
      maps[(2 * C + c) * plane + oo] = 2.f * ga2;
    }
    __syncwarp();
  };
  for (int yi = oy0; yi < iy1; yi += 2) {
    step(yi, px, py);
    if (yi + 1 < iy1) step(yi + 1, qx, qy);
  }
  for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
  if (lane == 0 && ssum != 0.0) atomicAdd(&sums[0], ssum);
}

// pass 2: full convolution of the maps + L1 term -> dL/dimage; sum |x - y|
// (losses.py:106-108, :138-145).  Same strip walk in fp32: map rows
// [oy0 - 10, oy1) feed output rows [oy0, oy1), map columns [x0 - 10, x0 + 32).
// acc[i] = partial sum of output row r + i; map row r completes acc[0].
__global__ void __launch_bounds__(SW * 3, 5) ssim_grad_kernel(LossParams lp,
                                                           const float* __restrict__ img,
                                                           const float* __restrict__ tgt,
                                                           const float* __restrict__ maps,
                                                           float* __restrict__ grad,
                                                           double* __restrict__ sums) {
  constexpr int RW = SW + HALO;
  __shared__ float4 sm[3][2][RW];  // [channel][buffer][column] = (map 0, map 1, map 2, -)
  const int lane = threadIdx.x, c = threadIdx.y;
  const int C = lp.C;
  if (c >= C) return;  // warp-uniform; warp-level synchronisation only
  const int x0 = blockIdx.x * SW, oy0 = blockIdx.y * RCH;
  const int oy1 = min(oy0 + RCH, lp.H);
  const int ry0 = max(oy0 - HALO, 0), ry1 = min(oy1, lp.Hv);  // map rows that contribute
  const int64_t plane = (int64_t)lp.Hv * lp.Wv;
  float g[WIN];
  float2 g2[WIN];  // packed copies for FFMA2 (maps 0 and 1 as one pair)
#pragma unroll
  for (int k = 0; k < WIN; ++k) g[k] = lp.gf[k], g2[k] = make_float2(g[k], g[k]);
  // prefetch: lane loads map q of channel c at columns x0 - 10 + lane (+32)
  constexpr int PER = 2;
  float pm[3][PER], qm[3][PER];  // map rows in flight
  float pi0, pt0, pi1, pt1;      // image / target of the matching output rows
  const int px_ = x0 + lane;
  const bool col_ok = px_ < lp.W;
  auto fetch = [&](int r, float (&fm)[3][PER], float& fi, float& ft) {
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int m = 0; m < PER; ++m) {
        const int e = lane + m * SW, vx = x0 - HALO + e;
        const bool ok = e < RW && r < ry1 && vx >= 0 && vx < lp.Wv;
        fm[q][m] = ok ? __ldg(maps + (q * C + c) * plane + (int64_t)r * lp.Wv + vx) : 0.f;
      }
    const bool ok = col_ok && r >= oy0 && r < oy1;
    const int64_t o = ((int64_t)r * lp.W + px_) * C + c;
    fi = ok ? __ldg(img + o) : 0.f;
    ft = ok ? __ldg(tgt + o) : 0.f;
  };
  auto stage = [&](int buf, const float (&fm)[3][PER]) {
#pragma unroll
    for (int m = 0; m < PER; ++m)
      if (lane + m * SW < RW) sm[c][buf][lane + m * SW] = make_float4(fm[0][m], fm[1][m], fm[2][m], 0.f);
  };
  float2 a01[WIN];  // maps 0 and 1, packed
  float a2[WIN];
#pragma unroll
  for (int j = 0; j < WIN; ++j) a01[j] = make_float2(0.f, 0.f), a2[j] = 0.f;
  double l1 = 0.0;
  // register buffers P / Q alternate (no moves): at step r the one passed in
  // holds map row r + 1 and the image / target of output row r + 1; it is
  // staged, then refilled with row r + 3
  float xi, ti;
  fetch(ry0, pm, xi, ti);
  stage(0, pm);
  float xa = xi, ta = ti;  // image / target of output row ry0
  fetch(ry0 + 1, pm, pi0, pt0);
  fetch(ry0 + 2, qm, pi1, pt1);
  __syncwarp();
  auto step = [&](int r, float (&fm)[3][PER], float& fi, float& ft) {
    const int cur = (r - ry0) & 1;
    const float xr = xa, tr = ta;
    if (r + 1 < oy1) {
      stage(cur ^ 1, fm);
      xa = fi, ta = ft;
      fetch(r + 3, fm, fi, ft);
    }
    // horizontal full convolution at output column px_: map cols px_ - j
    float2 h01 = make_float2(0.f, 0.f);
    float h2 = 0.f;
#pragma unroll
    for (int j = 0; j < WIN; ++j) {
      const float4 v = sm[c][cur][lane + HALO - j];
      h01 = __ffma2_rn(g2[j], make_float2(v.x, v.y), h01);
      h2 = fmaf(g[j], v.z, h2);
    }
    // output row r completes with tap 0; rows r + 1 .. r + 10 shift down
    const float2 b01 = __ffma2_rn(g2[0], h01, a01[0]);
    const float b0 = b01.x, b1 = b01.y, b2 = fmaf(g[0], h2, a2[0]);
#pragma unroll
    for (int i = 0; i < HALO; ++i) {
      a01[i] = __ffma2_rn(g2[i + 1], h01, a01[i + 1]);
      a2[i] = fmaf(g[i + 1], h2, a2[i + 1]);
    }
    a01[HALO] = make_float2(0.f, 0.f);
    a2[HALO] = 0.f;
    if (r >= oy0 && col_ok) {
      const int64_t o = ((int64_t)r * lp.W + px_) * C + c;
      const float d = xr - tr;
      l1 += fabs((double)xr - (double)tr);
      const double sgn = d > 0.f ? 1.0 : (d < 0.f ? -1.0 : 0.0);
      const double back = (double)b0 + (double)b1 * 2.0 * xr + (double)b2 * tr;
      grad[o] = (float)(lp.l1w * sgn + lp.up * back);
    }
    __syncwarp();
  };
  for (int r = ry0; r < oy1; r += 2) {
    step(r, pm, pi0, pt0);
    if (r + 1 < oy1) step(r + 1, qm, pi1, pt1);
  }
  for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
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
  return align_up(2 * sizeof(double)) + align_up((size_t)3 * channels * hv * wv * sizeof(float));
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
  if (!t_prezeroed) SS_CUDA(cudaMemsetAsync(sums, 0, 2 * sizeof(double), st));
  dim3 blk(SW, 3);
  dim3 g1((unsigned)cdiv(lp.Wv, SW), (unsigned)cdiv(lp.Hv, RCH));
  prof_begin(PH_SSIM_MAP, st);
  ssim_map_kernel<<<g1, blk, 0, st>>>(lp, image, target, maps, sums);
  SS_CHECK_LAUNCH("ssim_map_kernel");
  prof_end(PH_SSIM_MAP, st);
  dim3 g2((unsigned)cdiv(lp.W, SW), (unsigned)cdiv(lp.H, RCH));
  prof_begin(PH_SSIM_GRAD, st);
  ssim_grad_kernel<<<g2, blk, 0, st>>>(lp, image, target, maps, d_image, sums);
  SS_CHECK_LAUNCH("ssim_grad_kernel");
  prof_end(PH_SSIM_GRAD, st);
  loss_finalize_kernel<<<1, 1, 0, st>>>(lp, sums, loss_dev, status);
  SS_CHECK_LAUNCH("loss_finalize_kernel");
  return SS_OK;
}

}  // extern "C"
