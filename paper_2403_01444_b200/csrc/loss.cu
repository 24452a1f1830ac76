// Fused L1 + D-SSIM loss and its image gradient (KL) on sm_100a.
// Reference: losses.py:36-148 (/root/reference/pkg/src/splatstream/):
//   L = (1-lam) mean|x-y| + lam (1 - mean_valid SSIM) / 2,
// 11x11 Gaussian window (sigma 1.5), VALID windows only, mean over windows x
// channels; the SSIM adjoint is a FULL convolution of three per-window maps.
// Separable 11-tap passes staged in shared memory; window statistics in fp64.
#include "common.cuh"

namespace ss {

constexpr int WIN = 11, HALO = WIN - 1;
constexpr int BX = 32, BY = 8;  // output tile per CTA (256 threads)

struct LossParams {
  int H, W, Hv, Wv, C;
  double g[WIN];
  double c1, c2, lam, up;  // up = -lam / (2 n_windows)
};

// pass 1: per valid window -> SSIM value (summed) and the three adjoint maps
// (losses.py:121-137): A = dL/dmu_x part, B = dL/dconv_xx, C = dL/dconv_xy
__global__ void __launch_bounds__(BX* BY) ssim_map_kernel(LossParams lp,
                                                          const float* __restrict__ img,
                                                          const float* __restrict__ tgt,
                                                          float* __restrict__ maps,
                                                          double* __restrict__ sums) {
  __shared__ float sx[BY + HALO][BX + HALO + 1], sy[BY + HALO][BX + HALO + 1];
  __shared__ double hs[5][BY + HALO][BX];
  const int c = blockIdx.z;
  const int ox = blockIdx.x * BX, oy = blockIdx.y * BY;
  const int tid = threadIdx.y * BX + threadIdx.x;
  for (int i = tid; i < (BY + HALO) * (BX + HALO); i += BX * BY) {
    const int ry = i / (BX + HALO), rx = i % (BX + HALO);
    const int py = oy + ry, px = ox + rx;
    float xv = 0.f, yv = 0.f;
    if (py < lp.H && px < lp.W) {
      const int64_t o = ((int64_t)py * lp.W + px) * lp.C + c;
      xv = img[o];
      yv = tgt[o];
    }
    sx[ry][rx] = xv;
    sy[ry][rx] = yv;
  }
  __syncthreads();
  for (int i = tid; i < (BY + HALO) * BX; i += BX * BY) {
    const int ry = i / BX, rx = i % BX;
    double a = 0, b = 0, xx = 0, yy = 0, xy = 0;
#pragma unroll
    for (int k = 0; k < WIN; ++k) {
      const double xv = sx[ry][rx + k], yv = sy[ry][rx + k], w = lp.g[k];
      a += w * xv;
      b += w * yv;
      xx += w * xv * xv;
      yy += w * yv * yv;
      xy += w * xv * yv;
    }
    hs[0][ry][rx] = a;
    hs[1][ry][rx] = b;
    hs[2][ry][rx] = xx;
    hs[3][ry][rx] = yy;
    hs[4][ry][rx] = xy;
  }
  __syncthreads();
  const int vx = ox + threadIdx.x, vy = oy + threadIdx.y;
  double s = 0.0;
  if (vx < lp.Wv && vy < lp.Hv) {
    double v[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < WIN; ++k)
#pragma unroll
      for (int q = 0; q < 5; ++q) v[q] += lp.g[k] * hs[q][threadIdx.y + k][threadIdx.x];
    const double mx = v[0], my = v[1];
    const double vxx = v[2] - mx * mx, vyy = v[3] - my * my, cxy = v[4] - mx * my;
    const double a1 = 2.0 * mx * my + lp.c1, a2 = 2.0 * cxy + lp.c2;
    const double b1 = mx * mx + my * my + lp.c1, b2 = vxx + vyy + lp.c2;
    s = (a1 * a2) / (b1 * b2);
    const double inv = 1.0 / (b1 * b2);
    const double ga1 = a2 * inv, ga2 = a1 * inv, gb1 = -s / b1, gb2 = -s / b2;
    const double gmx = 2.0 * my * ga1 + 2.0 * mx * gb1 - 2.0 * my * ga2 - 2.0 * mx * gb2;
    const int64_t plane = (int64_t)lp.Hv * lp.Wv;
    const int64_t o = (int64_t)vy * lp.Wv + vx;
    maps[(0 * lp.C + c) * plane + o] = (float)gmx;
    maps[(1 * lp.C + c) * plane + o] = (float)gb2;
    maps[(2 * lp.C + c) * plane + o] = (float)(2.0 * ga2);
  }
  // block sum of SSIM values
  __shared__ double red[BX * BY / 32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    double t = 0;
    for (int i = 0; i < BX * BY / 32; ++i) t += red[i];
    atomicAdd(&sums[0], t);
  }
}

// pass 2: full convolution of the maps + L1 term -> dL/dimage; sum |x - y|
__global__ void __launch_bounds__(BX* BY) ssim_grad_kernel(LossParams lp,
                                                           const float* __restrict__ img,
                                                           const float* __restrict__ tgt,
                                                           const float* __restrict__ maps,
                                                           float* __restrict__ grad,
                                                           double* __restrict__ sums) {
  __shared__ float sm[3][BY + HALO][BX + HALO + 1];
  __shared__ float hs[3][BY + HALO][BX];
  const int c = blockIdx.z;
  const int ox = blockIdx.x * BX, oy = blockIdx.y * BY;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const int64_t plane = (int64_t)lp.Hv * lp.Wv;
  // map rows/cols [o - HALO, o + B) (zero outside the valid range)
  for (int i = tid; i < (BY + HALO) * (BX + HALO); i += BX * BY) {
    const int ry = i / (BX + HALO), rx = i % (BX + HALO);
    const int vy = oy - HALO + ry, vx = ox - HALO + rx;
    const bool in = vy >= 0 && vx >= 0 && vy < lp.Hv && vx < lp.Wv;
    const int64_t o = (int64_t)vy * lp.Wv + vx;
#pragma unroll
    for (int q = 0; q < 3; ++q) sm[q][ry][rx] = in ? maps[(q * lp.C + c) * plane + o] : 0.f;
  }
  __syncthreads();
  for (int i = tid; i < (BY + HALO) * BX; i += BX * BY) {
    const int ry = i / BX, rx = i % BX;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float a = 0.f;
#pragma unroll
      for (int k = 0; k < WIN; ++k) a = fmaf((float)lp.g[k], sm[q][ry][rx + k], a);
      hs[q][ry][rx] = a;
    }
  }
  __syncthreads();
  const int px = ox + threadIdx.x, py = oy + threadIdx.y;
  double l1 = 0.0;
  if (px < lp.W && py < lp.H) {
    float b[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < WIN; ++k)
#pragma unroll
      for (int q = 0; q < 3; ++q) b[q] = fmaf((float)lp.g[k], hs[q][threadIdx.y + k][threadIdx.x], b[q]);
    const int64_t o = ((int64_t)py * lp.W + px) * lp.C + c;
    const float x = img[o], y = tgt[o];
    const float d = x - y;
    l1 = fabs((double)x - (double)y);
    const double size = (double)lp.H * lp.W * lp.C;
    const double sgn = d > 0.f ? 1.0 : (d < 0.f ? -1.0 : 0.0);
    const double back = (double)b[0] + (double)b[1] * 2.0 * x + (double)b[2] * y;
    grad[o] = (float)((1.0 - lp.lam) * sgn / size + lp.up * back);
  }
  __shared__ double red[BX * BY / 32];
  for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  if ((tid & 31) == 0) red[tid >> 5] = l1;
  __syncthreads();
  if (tid == 0) {
    double t = 0;
    for (int i = 0; i < BX * BY / 32; ++i) t += red[i];
    atomicAdd(&sums[1], t);
  }
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
  if (channels < 1 || channels > 4) {
    set_error("render_loss supports 1-4 channels");
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
  lp.c1 = c1, lp.c2 = c2, lp.lam = lam;
  lp.up = -lam / (2.0 * (double)lp.Hv * lp.Wv * channels);
  double* sums = static_cast<double*>(scratch);
  float* maps = reinterpret_cast<float*>(static_cast<char*>(scratch) + align_up(2 * sizeof(double)));
  prof_begin(PH_LOSS, st);
  SS_CUDA(cudaMemsetAsync(sums, 0, 2 * sizeof(double), st));
  dim3 blk(BX, BY);
  dim3 g1((unsigned)cdiv(lp.Wv, BX), (unsigned)cdiv(lp.Hv, BY), channels);
  ssim_map_kernel<<<g1, blk, 0, st>>>(lp, image, target, maps, sums);
  SS_CHECK_LAUNCH("ssim_map_kernel");
  dim3 g2((unsigned)cdiv(lp.W, BX), (unsigned)cdiv(lp.H, BY), channels);
  ssim_grad_kernel<<<g2, blk, 0, st>>>(lp, image, target, maps, d_image, sums);
  SS_CHECK_LAUNCH("ssim_grad_kernel");
  loss_finalize_kernel<<<1, 1, 0, st>>>(lp, sums, loss_dev, status);
  SS_CHECK_LAUNCH("loss_finalize_kernel");
  prof_end(PH_LOSS, st);
  return SS_OK;
}

}  // extern "C"
