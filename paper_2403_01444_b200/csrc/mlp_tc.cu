// NTC decoder on the 5th-generation tensor cores: forward (K2f, ntc.py:241-248)
// and backward (K2b, ntc.py:258-276).
//
// Both kernels are persistent: one CTA of 512 threads per SM walks 128-row
// tiles of the feature matrix X.  Row r of a tile lives in TMEM lane r; the
// four warps that share a TMEM lane quarter (warps w, w+4, w+8, w+12) split the
// accumulator columns, so every epilogue (tcgen05.ld, bias, ReLU, operand
// split, st.shared) runs on 16 warps instead of 4.  One elected thread issues
// the MMAs and commits them to an mbarrier.  The next tile's rows are
// prefetched into registers while the current tile's MMAs run.
//
// Precision:
//  * forward: kind::tf32 with every operand split into tf32 hi + lo and three
//    products per K step (3xTF32), i.e. fp32-level accuracy; mode 2 = tf32.
//    fp16-weight decoders (ss_mlp.precision = SS_MLP_F16, BASELINE config 1):
//    kind::f16 with weights, biases and activations rounded to fp16, one
//    product per K = 16 step, fp32 accumulation.
//  * backward: kind::f16 with bf16 hi + lo operands and three products per K
//    step (~16 mantissa bits, fp32 accumulation), because its transposed
//    operands need MN-major descriptors (16-bit types).  The ReLU decisions are
//    the forward's (relu_masks), so the gradient is that of the function the
//    forward evaluated.  For fp16-weight decoders the backward takes the same
//    fp16-rounded weights, inputs and hidden activations as the forward, so
//    it is the (straight-through) gradient of the fp16 forward.
#include "common.cuh"
#include "umma.cuh"

namespace ss {

// per-stage clock64 stamps of CTA 0, thread 0, first tiles (ss_debug_mlp_trace)
__device__ unsigned long long g_mlp_trace[2][64];
// forward event stamps of CTA 0: [0] epilogue thread 0, [1] MMA lane (ss_debug_mlp_events)
__device__ unsigned long long g_mlp_ev[2][128];
#define SS_EV(k, cnt)                                                              \
  do {                                                                           \
    if (blockIdx.x == 0 && (cnt) < 128) g_mlp_ev[k][(cnt)] = clock64();          \
    ++(cnt);                                                                     \
  } while (0)
#define SS_STAMP(k, i)                                                           \
  do {                                                                           \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (i) < 64) g_mlp_trace[k][i] = clock64(); \
  } while (0)

namespace {
constexpr int HIDT = 64;
constexpr int NT = 512;  // threads per CTA: 4 per row, each a 16-column slice

template <int IN, int NL>
struct TcLay {  // same packed layout as ntc.cu's Lay<IN, NL>
  static constexpr int W0 = 0, B0 = IN * HIDT, W1 = B0 + HIDT;
  static constexpr int B1 = W1 + (NL == 2 ? HIDT * HIDT : 0);
  static constexpr int W2 = B1 + (NL == 2 ? HIDT : 0);
  static constexpr int B2 = W2 + HIDT * 8;
};

__device__ __forceinline__ void to_async() {
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
}

__device__ __forceinline__ void sync_mma(uint64_t* bar, uint32_t& phase) {
  umma::mbar_wait(bar, phase);
  phase ^= 1;
  umma::fence_after();
}

// ---------------------------------------------------------------- tf32 pieces
// P = 3: 3xTF32, P = 1: tf32, P = 0: fp16 operands
template <int IN, int NL, int P>
struct TcFwdSmem {  // the weights only: activations live in TMEM
  static constexpr int PL = P == 3 ? 2 : 1;  // hi (+ lo) planes
  static constexpr uint32_t W0 = P == 0 ? umma::tile16_bytes(64, IN) : umma::tile_bytes(64, IN);
  static constexpr uint32_t W1 =
      NL == 2 ? (P == 0 ? umma::tile16_bytes(64, 64) : umma::tile_bytes(64, 64)) : 0;
  static constexpr uint32_t W2 = P == 0 ? umma::tile16_bytes(16, 64) : umma::tile_bytes(16, 64);
  static constexpr uint32_t oW0 = 0;
  static constexpr uint32_t oW1 = oW0 + PL * W0;
  static constexpr uint32_t oW2 = oW1 + PL * W1;
  static constexpr uint32_t BYTES = oW2 + PL * W2;
};

// write x as (hi, lo) tf32 pair into the hi tile and (for P = 3) the lo tile
template <int P>
__device__ __forceinline__ void put(uint8_t* hi, uint32_t lo_off, uint32_t off, float x) {
  const float h = umma::to_tf32(x);
  *reinterpret_cast<float*>(hi + off) = h;
  if (P == 3) *reinterpret_cast<float*>(hi + lo_off + off) = umma::to_tf32(x - h);
}

// 4 consecutive columns (one 16-byte core row) as a tf32 hi/lo pair
template <int P>
__device__ __forceinline__ void put4(uint8_t* hi, uint32_t lo_off, uint32_t off, const float* v) {
  float4 h, l;
  h.x = umma::to_tf32(v[0]), h.y = umma::to_tf32(v[1]);
  h.z = umma::to_tf32(v[2]), h.w = umma::to_tf32(v[3]);
  *reinterpret_cast<float4*>(hi + off) = h;
  if (P == 3) {
    l.x = umma::to_tf32(v[0] - h.x), l.y = umma::to_tf32(v[1] - h.y);
    l.z = umma::to_tf32(v[2] - h.z), l.w = umma::to_tf32(v[3] - h.w);
    *reinterpret_cast<float4*>(hi + lo_off + off) = l;
  }
}

// K-major tf32 operand: descriptors of the hi and lo planes at k = 0; one
// 8-wide K step advances the start address by 256 bytes (16 in descriptor units).
struct Op32 {
  uint64_t hi, lo;
};
__device__ __forceinline__ Op32 op32(uint32_t addr, uint32_t lo_off, int cols) {
  return {umma::desc_k(addr, cols, 0), umma::desc_k(addr + lo_off, cols, 0)};
}

// one layer: acc[M=128, N] (+)= A[128, K] . B[N, K]^T over K = 8 * NK
template <int P, int NK>
__device__ __forceinline__ void mma_layer(uint32_t acc, const Op32& A, const Op32& B,
                                          uint32_t idesc) {
#pragma unroll
  for (int s = 0; s < NK; ++s) {
    const uint64_t d = 16ull * s;
    umma::mma_tf32(acc, A.hi + d, B.hi + d, idesc, s > 0);
    if (P == 3) {
      umma::mma_tf32(acc, A.hi + d, B.lo + d, idesc, 1);
      umma::mma_tf32(acc, A.lo + d, B.hi + d, idesc, 1);
    }
  }
}

// ---------------------------------------------------------------- bf16 pieces
// 16-bit operand: descriptors of the hi and lo planes at k = 0 and the
// descriptor increment of one 16-wide K step (2 core matrices along K)
struct Op16 {
  uint64_t hi, lo;
  uint32_t kstep;
};
__device__ __forceinline__ Op16 op16(uint32_t addr, uint32_t lo_off, int cols, int mn) {
  Op16 o;
  o.hi = mn ? umma::desc16_mn(addr, cols, 0) : umma::desc16_k(addr, cols, 0);
  o.lo = mn ? umma::desc16_mn(addr + lo_off, cols, 0) : umma::desc16_k(addr + lo_off, cols, 0);
  o.kstep = (mn ? 2u * umma::sbo16(cols) : 256u) >> 4;
  return o;
}

// acc (+)= A . B over K = 16 * NK with the 3-product bf16 split
template <int NK>
__device__ __forceinline__ void gemm3(uint32_t acc, const Op16& A, const Op16& B, uint32_t idesc,
                                      uint32_t accumulate) {
#pragma unroll
  for (int s = 0; s < NK; ++s) {
    const uint64_t da = (uint64_t)A.kstep * s, db = (uint64_t)B.kstep * s;
    umma::mma_bf16(acc, A.hi + da, B.hi + db, idesc, accumulate | (s > 0));
    umma::mma_bf16(acc, A.hi + da, B.lo + db, idesc, 1);
    umma::mma_bf16(acc, A.lo + da, B.hi + db, idesc, 1);
  }
}

// warp-collective form: called by a whole converged warp, one lane issues
template <int NK>
__device__ __forceinline__ void gemm3e(uint32_t acc, const Op16& A, const Op16& B, uint32_t idesc,
                                       uint32_t accumulate) {
#pragma unroll
  for (int s = 0; s < NK; ++s) {
    const uint64_t da = (uint64_t)A.kstep * s, db = (uint64_t)B.kstep * s;
    umma::mma_bf16_elect(acc, A.hi + da, B.hi + db, idesc, accumulate | (s > 0));
    umma::mma_bf16_elect(acc, A.hi + da, B.lo + db, idesc, 1);
    umma::mma_bf16_elect(acc, A.lo + da, B.hi + db, idesc, 1);
  }
}

// store 8 consecutive columns c0..c0+7 of row r as hi/lo bf16 (two 16-byte stores)
__device__ __forceinline__ void put8(uint8_t* tile, uint32_t lo_off, int r, int c0, int cols,
                                     const float* v) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint16_t h0, l0, h1, l1;
    umma::split_bf16(v[2 * j], h0, l0);
    umma::split_bf16(v[2 * j + 1], h1, l1);
    h[j] = (uint32_t)h0 | ((uint32_t)h1 << 16);
    l[j] = (uint32_t)l0 | ((uint32_t)l1 << 16);
  }
  const uint32_t off = umma::tile16_off(r, c0, cols);
  *reinterpret_cast<uint4*>(tile + off) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(tile + lo_off + off) = make_uint4(l[0], l[1], l[2], l[3]);
}

__device__ __forceinline__ void put_scalar(uint8_t* tile, uint32_t lo_off, int r, int c, int cols,
                                           float x) {
  uint16_t h, l;
  umma::split_bf16(x, h, l);
  const uint32_t off = umma::tile16_off(r, c, cols);
  *reinterpret_cast<uint16_t*>(tile + off) = h;
  *reinterpret_cast<uint16_t*>(tile + lo_off + off) = l;
}

// ---- fp16 operands of the fp16-weight decoder's backward (kind::f16, f16 A/B):
// weights, inputs and hidden activations are exact fp16 values (one plane);
// gradients and deltas are scaled into the fp16 range and split hi + lo
__device__ __forceinline__ void put8h(uint8_t* tile, int r, int c0, int cols, const float* v) {
  uint32_t h[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = umma::pack_f16(v[2 * j], v[2 * j + 1]);
  *reinterpret_cast<uint4*>(tile + umma::tile16_off(r, c0, cols)) = make_uint4(h[0], h[1], h[2], h[3]);
}
__device__ __forceinline__ void put8s(uint8_t* tile, uint32_t lo_off, int r, int c0, int cols,
                                      const float* v, float scale) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float a = v[2 * j] * scale, b = v[2 * j + 1] * scale;
    const float ha = umma::round_f16(a), hb = umma::round_f16(b);
    h[j] = umma::pack_f16(ha, hb);
    l[j] = umma::pack_f16(a - ha, b - hb);
  }
  const uint32_t off = umma::tile16_off(r, c0, cols);
  *reinterpret_cast<uint4*>(tile + off) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(tile + lo_off + off) = make_uint4(l[0], l[1], l[2], l[3]);
}
__device__ __forceinline__ void put_scalar_h(uint8_t* tile, int r, int c, int cols, float x) {
  *reinterpret_cast<__half*>(tile + umma::tile16_off(r, c, cols)) = __float2half_rn(x);
}
// one product per K step (both operands exact), or two with the A or the B
// operand split hi + lo (the A_lo B_lo term is below fp32 resolution)
template <int NK>
__device__ __forceinline__ void gemm1e(uint32_t acc, const Op16& A, const Op16& B, uint32_t idesc,
                                       uint32_t accumulate) {
#pragma unroll
  for (int s = 0; s < NK; ++s)
    umma::mma_bf16_elect(acc, A.hi + (uint64_t)A.kstep * s, B.hi + (uint64_t)B.kstep * s, idesc,
                         accumulate | (s > 0));
}
template <int NK, bool SPLIT_A>
__device__ __forceinline__ void gemm2e(uint32_t acc, const Op16& A, const Op16& B, uint32_t idesc,
                                       uint32_t accumulate) {
#pragma unroll
  for (int s = 0; s < NK; ++s) {
    const uint64_t da = (uint64_t)A.kstep * s, db = (uint64_t)B.kstep * s;
    umma::mma_bf16_elect(acc, A.hi + da, B.hi + db, idesc, accumulate | (s > 0));
    if (SPLIT_A) umma::mma_bf16_elect(acc, A.lo + da, B.hi + db, idesc, 1);
    else umma::mma_bf16_elect(acc, A.hi + da, B.lo + db, idesc, 1);
  }
}

// X row slices: thread quarter q owns column blocks 8q + 32b < IN
template <int IN>
struct XSlice {
  static constexpr int NB = (IN + 31) / 32;
  float v[NB][8];
  __device__ __forceinline__ void load(const float* __restrict__ X, int64_t row, int xs, int q,
                                       bool ok) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int c = 8 * q + 32 * b;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), d = a;
      if (ok && c < IN) {
        a = __ldg(reinterpret_cast<const float4*>(X + row * xs + c));
        d = __ldg(reinterpret_cast<const float4*>(X + row * xs + c + 4));
      }
      v[b][0] = a.x, v[b][1] = a.y, v[b][2] = a.z, v[b][3] = a.w;
      v[b][4] = d.x, v[b][5] = d.y, v[b][6] = d.z, v[b][7] = d.w;
    }
  }
};
}  // namespace

// ================================================================= forward
// Warp-specialised: 16 epilogue warps + 1 MMA warp.  Every activation operand
// lives in TMEM (tcgen05.mma with A from tensor memory), so a layer's epilogue
// is tcgen05.ld (accumulator) -> bias, ReLU, tf32 hi/lo split -> tcgen05.st
// (next layer's A operand); only the weights (B operands) are in shared
// memory.  Two 128-row tiles are in flight (slots 0 and 1): while the
// epilogue warps work on one slot, the MMA warp runs the other's layer.
// Handshakes are mbarriers (ready[s]: 16 warp arrivals after the TMEM
// stores; done[s]: tcgen05.commit), never a CTA-wide barrier.
//
// TMEM of slot s (base 256 s): [0, 64) A hi, [64, 128) A lo (X, then h1,
// then h2), [128, 192) acc1 / acc2, [192, 208) acc3.
constexpr int NT_FWD = NT + 32;

template <int IN, int NL, int P>
__global__ void __launch_bounds__(NT_FWD, 1) mlp_fwd_tc_kernel(int64_t n, const float* __restrict__ X,
                                                               int xs, const float* __restrict__ params,
                                                               float* __restrict__ out, int os,
                                                               uint64_t* __restrict__ relu_masks) {
  using L = TcLay<IN, NL>;
  using S = TcFwdSmem<IN, NL, P>;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t ready[2], done[2];
  __shared__ uint32_t tbase;
  __shared__ float sbias[64 + 64 + 8];
  const int tid = threadIdx.x, warp = tid >> 5;
  // ---- stage the weights as K-major B tiles (rows = output unit, cols = input)
  auto put_w = [&](uint32_t o, uint32_t plane, int nn, int k, int cols, float w) {
    if (P == 0)
      *reinterpret_cast<__half*>(sm + o + umma::tile16_off(nn, k, cols)) = __float2half_rn(w);
    else
      put<P>(sm + o, plane, umma::tile_off(nn, k, cols), w);
  };
  // params are (fan_in, fan_out) row-major: consecutive threads read
  // consecutive weights (coalesced, several loads in flight per thread)
#pragma unroll 4
  for (int i = tid; i < 64 * IN; i += NT_FWD) {
    const int k = i / 64, nn = i % 64;
    put_w(S::oW0, S::W0, nn, k, IN, __ldg(params + L::W0 + i));
  }
  if (NL == 2)
#pragma unroll 4
    for (int i = tid; i < 64 * 64; i += NT_FWD) {
      const int k = i / 64, nn = i % 64;
      put_w(S::oW1, S::W1, nn, k, 64, __ldg(params + L::W1 + i));
    }
#pragma unroll 2
  for (int i = tid; i < 16 * 64; i += NT_FWD) {
    const int k = i / 16, nn = i % 16;
    put_w(S::oW2, S::W2, nn, k, 64, nn < 8 ? __ldg(params + L::W2 + k * 8 + nn) : 0.f);
  }
  auto bias = [&](float b) { return P == 0 ? umma::round_f16(b) : b; };
  if (tid < 64) {
    sbias[tid] = bias(params[L::B0 + tid]);
    sbias[64 + tid] = NL == 2 ? bias(params[L::B1 + tid]) : 0.f;
  }
  if (tid < 8) sbias[128 + tid] = bias(params[L::B2 + tid]);
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      umma::mbar_init(&ready[s], NT / 32);
      umma::mbar_init(&done[s], 1);
    }
    umma::fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc(&tbase, 512);
  to_async();
  umma::fence_after();
  const uint32_t tmem = tbase;
  const int64_t ntiles = (n + 127) / 128;
  const int64_t G = gridDim.x;
  constexpr int NLAY = NL == 2 ? 3 : 2;  // MMA layers per tile

  if (warp == NT / 32) {
    // ================= MMA warp: one elected lane issues, in tile/slot order
    const Op32 dW0 = P == 0 ? Op32{umma::desc16_k(umma::smem_u32(sm + S::oW0), IN, 0), 0}
                            : op32(umma::smem_u32(sm + S::oW0), S::W0, IN);
    const Op32 dW1 = P == 0 ? Op32{umma::desc16_k(umma::smem_u32(sm + S::oW1), 64, 0), 0}
                            : op32(umma::smem_u32(sm + S::oW1), S::W1, 64);
    const Op32 dW2 = P == 0 ? Op32{umma::desc16_k(umma::smem_u32(sm + S::oW2), 64, 0), 0}
                            : op32(umma::smem_u32(sm + S::oW2), S::W2, 64);
    constexpr uint32_t id64 = P == 0 ? umma::idesc_f16(128, 64, 0, 0) : umma::idesc_tf32(128, 64, 0, 0);
    constexpr uint32_t id16 = P == 0 ? umma::idesc_f16(128, 16, 0, 0) : umma::idesc_tf32(128, 16, 0, 0);
    uint32_t ph[2] = {0u, 0u};
    int nev = 0;
    for (int64_t t0 = blockIdx.x; t0 < ntiles; t0 += 2 * G) {
      const bool two = t0 + G < ntiles;
#pragma unroll
      for (int l = 0; l < NLAY; ++l) {
        const int layer = l == NLAY - 1 ? 2 : l;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (s == 1 && !two) continue;
          umma::mbar_wait(&ready[s], ph[s]);
          ph[s] ^= 1;
          umma::fence_after();
          if ((tid & 31) == 0) SS_EV(1, nev);
          {  // warp-uniform issue, one elected lane (umma::*_elect)
            const uint32_t base = tmem + 256u * s;
            const Op32& B = layer == 0 ? dW0 : (layer == 1 ? dW1 : dW2);
            const uint32_t acc = base + (layer == 2 ? 192u : 128u);
            const uint32_t id = layer == 2 ? id16 : id64;
            // K steps: 8 (tf32) or 16 (fp16) elements, 8 TMEM columns and
            // 256 bytes of B either way
            constexpr int KS = P == 0 ? 16 : 8;
            constexpr int nk0 = IN / KS, nk = 64 / KS;
#pragma unroll
            for (int k = 0; k < nk; ++k) {
              if (layer == 0 && k >= nk0) break;
              const uint64_t d = 16ull * k;
              if (P == 0) {
                umma::mma_f16_ts_elect(acc, base + 8u * k, B.hi + d, id, k > 0);
                continue;
              }
              umma::mma_tf32_ts_elect(acc, base + 8u * k, B.hi + d, id, k > 0);
              if (P == 3) {
                umma::mma_tf32_ts_elect(acc, base + 8u * k, B.lo + d, id, 1);
                umma::mma_tf32_ts_elect(acc, base + 64u + 8u * k, B.hi + d, id, 1);
              }
            }
            umma::commit_elect(&done[s]);
            if ((tid & 31) == 0) SS_EV(1, nev);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ================= epilogue warps: thread (r, q) = row r, columns 16q..16q+15
    const int r = tid & 127, q = tid >> 7;
    const int c0 = 16 * q;
    const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t ph[2] = {0u, 0u};
    int nev = 0;
    XSlice<IN> xr[2];
    auto load_x = [&](int s, int64_t t) {
      xr[s].load(X, t * 128 + r, xs, q, t < ntiles && t * 128 + r < n);
    };
    auto arrive = [&](int s) {  // this warp's TMEM stores are complete
      umma::tmem_st_wait();
      umma::fence_before();
      __syncwarp();
      if ((tid & 31) == 0) umma::mbar_arrive(&ready[s]);
      if (tid == 0) SS_EV(0, nev);
    };
    auto put_x = [&](int s) {  // X slice -> A hi / lo columns of slot s
      const uint32_t base = tmem + 256u * s + lane;
#pragma unroll
      for (int b = 0; b < XSlice<IN>::NB; ++b) {
        const int c = 8 * q + 32 * b;
        if (c < IN && P == 0) {  // fp16 pairs: columns c/2 .. c/2 + 3
          uint32_t u[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) u[j] = umma::pack_f16(xr[s].v[b][2 * j], xr[s].v[b][2 * j + 1]);
          umma::tmem_st4u(base + (uint32_t)(c / 2), u);
        } else if (c < IN) {
          float h[8], l[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            h[j] = umma::to_tf32(xr[s].v[b][j]);
            l[j] = umma::to_tf32(xr[s].v[b][j] - h[j]);
          }
          umma::tmem_st8(base + (uint32_t)c, h);
          if (P == 3) umma::tmem_st8(base + 64u + (uint32_t)c, l);
        }
      }
      arrive(s);
    };
    auto wait_done = [&](int s) {
      umma::mbar_wait(&done[s], ph[s]);
      ph[s] ^= 1;
      umma::fence_after();
      if (tid == 0) SS_EV(0, nev);
    };
    // hidden layer: relu(acc + b) -> A hi / lo of slot s; ReLU mask quarter -> HBM
    auto hidden = [&](int s, int layer, int64_t t) {
      wait_done(s);
      const uint32_t base = tmem + 256u * s + lane;
      uint32_t m = 0;
      if (P == 0) {
        float v[16];
        umma::tmem_ld16(base + 128u + (uint32_t)c0, v);
        uint32_t u[8];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          v[j] = fmaxf(v[j] + sbias[64 * layer + c0 + j], 0.f);
          m |= (uint32_t)(v[j] > 0.f) << j;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = umma::pack_f16(v[2 * j], v[2 * j + 1]);
        umma::tmem_st8u(base + (uint32_t)(c0 / 2), u);
      } else {
        // two 8-column halves keep the live registers low (one CTA of 544
        // threads caps them at 96 per thread)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int cc = c0 + 8 * hf;
          float v[8], l[8];
          umma::tmem_ld8(base + 128u + (uint32_t)cc, v);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float x = fmaxf(v[j] + sbias[64 * layer + cc + j], 0.f);
            m |= (uint32_t)(x > 0.f) << (8 * hf + j);
            v[j] = umma::to_tf32(x);
            l[j] = umma::to_tf32(x - v[j]);
          }
          umma::tmem_st8(base + (uint32_t)cc, v);
          if (P == 3) umma::tmem_st8(base + 64u + (uint32_t)cc, l);
        }
      }
      arrive(s);
      // the backward reuses the forward's ReLU decisions (self-consistent
      // gradient): 16-bit quarter q of the row's 64-bit mask of this layer
      const int64_t row = t * 128 + r;
      if (relu_masks && row < n) {
        uint16_t* mk = reinterpret_cast<uint16_t*>(relu_masks + 2 * row);
        mk[4 * layer + q] = (uint16_t)m;
        if (NL == 1) mk[4 + q] = (uint16_t)m;
      }
    };
    auto finish = [&](int s, int64_t t) {
      wait_done(s);
      float o[8];
      if (q == 0) umma::tmem_ld8(tmem + 256u * s + lane + 192u, o);
      if (t + 2 * G < ntiles) {  // the slot's next tile
        put_x(s);
        load_x(s, t + 4 * G);
      }
      const int64_t row = t * 128 + r;
      if (q == 0 && row < n) {
        if (os == 8) {
          *reinterpret_cast<float4*>(out + row * 8) = make_float4(
              o[0] + sbias[128], o[1] + sbias[129], o[2] + sbias[130], o[3] + sbias[131]);
          *reinterpret_cast<float4*>(out + row * 8 + 4) =
              make_float4(o[4] + sbias[132], o[5] + sbias[133], o[6] + sbias[134], 0.f);
        } else {
#pragma unroll
          for (int k = 0; k < 7; ++k) out[row * os + k] = o[k] + sbias[128 + k];
        }
      }
    };
    int64_t t0 = blockIdx.x;
    if (t0 < ntiles) {
      load_x(0, t0);
      load_x(1, t0 + G);
      put_x(0);
      if (t0 + G < ntiles) put_x(1);
      load_x(0, t0 + 2 * G);
      load_x(1, t0 + 3 * G);
    }
    SS_STAMP(0, 0);
    int it = 0;
    for (; t0 < ntiles; t0 += 2 * G, ++it) {
      const int64_t t1 = t0 + G;
      const bool two = t1 < ntiles;
      SS_STAMP(0, 1 + 8 * it);
      hidden(0, 0, t0);
      SS_STAMP(0, 2 + 8 * it);
      if (two) hidden(1, 0, t1);
      SS_STAMP(0, 3 + 8 * it);
      if (NL == 2) {
        hidden(0, 1, t0);
        SS_STAMP(0, 4 + 8 * it);
        if (two) hidden(1, 1, t1);
      }
      SS_STAMP(0, 5 + 8 * it);
      finish(0, t0);
      SS_STAMP(0, 6 + 8 * it);
      if (two) finish(1, t1);
      SS_STAMP(0, 7 + 8 * it);
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) {
    umma::fence_after();
    umma::tmem_free(tmem, 512);
  }
}

// ================================================================= backward
// Per 128-row tile, every operand split into bf16 hi + lo.  With the forward's
// ReLU masks given, the delta chain does not depend on the recomputed
// activations, so the two chains run side by side in three MMA stages:
//
//   stage 1   H1 = X W0 (+ b0)                 DL = G W2^T
//             -> H1 = relu * m1                -> D_last = DL * m_last
//   stage 2   H2 = H1 W1 (+ b1)                D1 = D2 W1^T          (NL = 2)
//             dW1^T += D2^T [H1 | 1]  (col 64 = db1)
//             -> H2 = relu * m2                -> D1 *= m1
//   stage 3   dX = D1 W0^T -> HBM (table scatter)
//             dW0^T += D1^T [X | 1]   (col IN = db0)
//             dW2   += H_last^T G
//
// Stage 1 of the next tile is issued before stage 3's epilogue (dX) runs.  The
// weight-gradient accumulators (M = 64) stay in TMEM across the CTA's tiles and
// are flushed once with reductions into g_params.  Transposed operands are the
// same shared-memory tiles read through MN-major descriptors.  db2 is summed in
// registers.
namespace {
template <int IN, int NL>
struct TcBwdSmem {
  static constexpr int XC = IN + 8, HC = 72;
  static constexpr uint32_t W0 = umma::tile16_bytes(64, IN);
  static constexpr uint32_t W1 = NL == 2 ? umma::tile16_bytes(64, 64) : 0;
  static constexpr uint32_t W2 = umma::tile16_bytes(16, 64);
  static constexpr uint32_t X = umma::tile16_bytes(128, XC);
  static constexpr uint32_t H1 = umma::tile16_bytes(128, HC);
  static constexpr uint32_t H2 = NL == 2 ? umma::tile16_bytes(128, 64) : 0;
  static constexpr uint32_t G = umma::tile16_bytes(128, 16);
  static constexpr uint32_t D2 = NL == 2 ? umma::tile16_bytes(128, 64) : 0;
  static constexpr uint32_t D1 = umma::tile16_bytes(128, 64);
  // every tile is followed by its lo plane (same size)
  static constexpr uint32_t oW0 = 0, oW1 = oW0 + 2 * W0, oW2 = oW1 + 2 * W1;
  static constexpr uint32_t oX = oW2 + 2 * W2, oH1 = oX + 2 * X, oH2 = oH1 + 2 * H1;
  static constexpr uint32_t oG = oH2 + 2 * H2, oD2 = oG + 2 * G, oD1 = oD2 + 2 * D2;
  static constexpr uint32_t BYTES = oD1 + 2 * D1;
  // TMEM columns
  static constexpr uint32_t cH1 = 0, cDL = 64, cH2 = 128, cD1 = 192, cDX = 256;
  static constexpr uint32_t cW2 = 320, cW1 = 328, cW0 = 400;
};
}  // namespace

template <int IN, int NL, bool H16>
__global__ void __launch_bounds__(NT, 1) mlp_bwd_tc_kernel(
    int64_t n, const float* __restrict__ X, int xs, const float* __restrict__ g_out, int gs,
    const uint64_t* __restrict__ relu_masks, const float* __restrict__ params,
    float* __restrict__ dX, float* __restrict__ g_params) {
  using L = TcLay<IN, NL>;
  using S = TcBwdSmem<IN, NL>;
  constexpr int XC = S::XC, HC = S::HC;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bar_w;  // bar: activation / delta GEMMs, bar_w: weight gradients
  __shared__ uint32_t tbase;
  __shared__ float sbias[128];
  __shared__ float sdb2[4][8];
  const int tid = threadIdx.x, warp = tid >> 5, lane_id = tid & 31;
  const int r = tid & 127, q = tid >> 7;
  const int c0 = 16 * q;  // this thread's 16 columns of every 64-wide accumulator
  // H16: the fp16-weight decoder: fp16 operands (kind::f16 with f16 A/B); the
  // weights, inputs and activations are exact in one plane, the gradient chain
  // (G, D) is scaled by gsc into the fp16 range and split hi + lo, so every
  // GEMM takes one or two products instead of three
  auto rnd = [](float x) { return H16 ? umma::round_f16(x) : x; };
  // ---- weights as bf16 hi/lo tiles: W0t (j, f) = W0[f][j]; W1t (j, i) = W1[i][j];
  //      W2t (o, j) = W2[j][o] (rows 7..15 zero)
  auto putw = [&](uint32_t o, uint32_t lo, int r_, int c_, int cols, float x) {
    if (H16) put_scalar_h(sm + o, r_, c_, cols, x);
    else put_scalar(sm + o, lo, r_, c_, cols, x);
  };
  // (fan_in, fan_out) row-major params read in order: coalesced, several in flight
#pragma unroll 4
  for (int i = tid; i < 64 * IN; i += NT) {
    const int f = i / 64, j = i % 64;
    putw(S::oW0, S::W0, j, f, IN, rnd(__ldg(params + L::W0 + i)));
  }
  if (NL == 2)
#pragma unroll 4
    for (int i = tid; i < 64 * 64; i += NT) {
      const int k = i / 64, j = i % 64;
      putw(S::oW1, S::W1, j, k, 64, rnd(__ldg(params + L::W1 + i)));
    }
#pragma unroll 2
  for (int i = tid; i < 16 * 64; i += NT) {
    const int j = i / 16, o = i % 16;
    putw(S::oW2, S::W2, o, j, 64, o < 7 ? rnd(__ldg(params + L::W2 + j * 8 + o)) : 0.f);
  }
  if (tid < 64) {
    sbias[tid] = rnd(params[L::B0 + tid]);
    sbias[64 + tid] = NL == 2 ? rnd(params[L::B1 + tid]) : 0.f;
  }
  // constant columns: X col IN = 1 (db0), H1 col 64 = 1 (db1), G cols 8..15 = 0
  {
    const float pad[8] = {1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (q == 0) {
      if (H16) put8h(sm + S::oX, r, IN, XC, pad);
      else put8(sm + S::oX, S::X, r, IN, XC, pad);
    }
    if (q == 1) {
      if (H16) put8h(sm + S::oH1, r, 64, HC, pad);
      else put8(sm + S::oH1, S::H1, r, 64, HC, pad);
    }
    if (q == 2) put8(sm + S::oG, S::G, r, 8, 16, z);  // zero in both planes either way
  }
  // H16: the gradient scale of this CTA, a power of two that keeps G and the
  // deltas D_last = G W2^T (masked) and D1 = D2 W1^T within fp16:
  // |D_last| <= max|G| max_j sum_o |W2_jo|, |D1| <= |D2| max_k sum_n |W1_kn|
  float gsc = 1.f, igsc = 1.f;
  if (H16) {
    __shared__ float s_max[NT / 32][3];
    float gm = 0.f, r2 = 0.f, r1 = 0.f;
    const int64_t nt_ = (n + 127) / 128;
    const int64_t mine = nt_ > blockIdx.x ? (nt_ - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (gs == 8 && (reinterpret_cast<uintptr_t>(g_out) & 15) == 0) {
      // rows of 8 floats (the 8th is zero padding): two float4 per row, all in flight
#pragma unroll 4
      for (int64_t k = tid; k < mine * 256; k += NT) {
        const int64_t row = (blockIdx.x + (k >> 8) * gridDim.x) * 128 + ((k & 255) >> 1);
        if (row < n) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(g_out + row * 8) + (k & 1));
          gm = fmaxf(gm, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
      }
    } else {
      for (int64_t k = tid; k < mine * 128 * 7; k += NT) {
        const int64_t e = k % (128 * 7);
        const int64_t row = (blockIdx.x + (k / (128 * 7)) * gridDim.x) * 128 + e / 7;
        if (row < n) gm = fmaxf(gm, fabsf(__ldg(g_out + row * gs + e % 7)));
      }
    }
    if (tid < 64) {
      for (int o = 0; o < 7; ++o) r2 += fabsf(rnd(params[L::W2 + tid * 8 + o]));
      if (NL == 2)
        for (int k = 0; k < 64; ++k) r1 += fabsf(rnd(params[L::W1 + tid * 64 + k]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
      r2 = fmaxf(r2, __shfl_xor_sync(0xffffffffu, r2, o));
      r1 = fmaxf(r1, __shfl_xor_sync(0xffffffffu, r1, o));
    }
    if ((tid & 31) == 0) s_max[warp][0] = gm, s_max[warp][1] = r2, s_max[warp][2] = r1;
    __syncthreads();
    gm = r2 = r1 = 0.f;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w)
      gm = fmaxf(gm, s_max[w][0]), r2 = fmaxf(r2, s_max[w][1]), r1 = fmaxf(r1, s_max[w][2]);
    const float bound = gm * fmaxf(1.f, fmaxf(r2, NL == 2 ? r2 * r1 : 0.f));
    const int e = bound > 0.f ? (int)ceilf(log2f(bound)) : 0;
    const int sh = min(100, max(-100, 14 - e));
    gsc = exp2f((float)sh);
    igsc = exp2f((float)-sh);
  }
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::mbar_init(&bar_w, 1);
    umma::fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc(&tbase, 512);
  to_async();
  umma::fence_after();
  const uint32_t tmem = tbase;
  const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t aX = umma::smem_u32(sm + S::oX), aW0 = umma::smem_u32(sm + S::oW0);
  const uint32_t aW1 = umma::smem_u32(sm + S::oW1), aW2 = umma::smem_u32(sm + S::oW2);
  const uint32_t aH1 = umma::smem_u32(sm + S::oH1), aH2 = umma::smem_u32(sm + S::oH2);
  const uint32_t aG = umma::smem_u32(sm + S::oG), aD2 = umma::smem_u32(sm + S::oD2);
  const uint32_t aD1 = umma::smem_u32(sm + S::oD1);
  const Op16 oX_k = op16(aX, S::X, XC, 0), oX_mn = op16(aX, S::X, XC, 1);
  const Op16 oW0_k = op16(aW0, S::W0, IN, 0), oW0_mn = op16(aW0, S::W0, IN, 1);
  const Op16 oW1_k = op16(aW1, S::W1, 64, 0), oW1_mn = op16(aW1, S::W1, 64, 1);
  const Op16 oW2_mn = op16(aW2, S::W2, 64, 1);
  const Op16 oH1_k = op16(aH1, S::H1, HC, 0), oH1_mn = op16(aH1, S::H1, HC, 1);
  const Op16 oH2_mn = op16(aH2, S::H2, 64, 1);
  const Op16 oG_k = op16(aG, S::G, 16, 0), oG_mn = op16(aG, S::G, 16, 1);
  const Op16 oD2_k = op16(aD2, S::D2, 64, 0), oD2_mn = op16(aD2, S::D2, 64, 1);
  const Op16 oD1_k = op16(aD1, S::D1, 64, 0), oD1_mn = op16(aD1, S::D1, 64, 1);
  const Op16 oHl_mn = NL == 2 ? oH2_mn : oH1_mn;
  constexpr uint32_t idF = H16 ? umma::idesc_f16(128, 64, 0, 0) : umma::idesc_bf16(128, 64, 0, 0);
  constexpr uint32_t idB64 = H16 ? umma::idesc_f16(128, 64, 0, 1) : umma::idesc_bf16(128, 64, 0, 1);
  constexpr uint32_t idBX = H16 ? umma::idesc_f16(128, IN, 0, 1) : umma::idesc_bf16(128, IN, 0, 1);
  constexpr uint32_t idW2 = H16 ? umma::idesc_f16(64, 8, 1, 1) : umma::idesc_bf16(64, 8, 1, 1);
  constexpr uint32_t idW1 = H16 ? umma::idesc_f16(64, HC, 1, 1) : umma::idesc_bf16(64, HC, 1, 1);
  constexpr uint32_t idW0 = H16 ? umma::idesc_f16(64, XC, 1, 1) : umma::idesc_bf16(64, XC, 1, 1);
  uint32_t phase = 0, phase_w = 0, acc_w = 0;
  bool w_pending = false;  // weight-gradient GEMMs of the last tile still reading X, G, H, D
  auto wait_w = [&]() {
    if (w_pending) {
      sync_mma(&bar_w, phase_w);
      w_pending = false;
    }
  };
  float db2[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int64_t ntiles = (n + 127) / 128;
  // register prefetch of this thread's slices of the X, g and mask rows
  XSlice<IN> xr;
  float gr[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  ulonglong2 mr = make_ulonglong2(0, 0);
  auto fetch = [&](int64_t t) {
    const int64_t row = t * 128 + r;
    const bool ok = t < ntiles && row < n;
    xr.load(X, row, xs, q, ok);
    if (q == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) gr[k] = (ok && k < 7) ? __ldg(g_out + row * gs + k) : 0.f;
    }
    mr = ok ? __ldg(reinterpret_cast<const ulonglong2*>(relu_masks) + row) : make_ulonglong2(0, 0);
  };
  // X and G of the prefetched tile -> smem (their previous readers have completed)
  auto stage_in = [&]() {
#pragma unroll
    for (int b = 0; b < XSlice<IN>::NB; ++b) {
      const int c = 8 * q + 32 * b;
      if (c < IN) {
        if (H16) put8h(sm + S::oX, r, c, XC, xr.v[b]);  // rounds to fp16
        else put8(sm + S::oX, S::X, r, c, XC, xr.v[b]);
      }
    }
    if (q == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) db2[k] += gr[k];
      if (H16) put8s(sm + S::oG, S::G, r, 0, 16, gr, gsc);
      else put8(sm + S::oG, S::G, r, 0, 16, gr);
    }
  };
  auto issue_stage1 = [&]() {
    to_async();
    if (warp == 0) {  // warp-uniform issue: descriptors stay in uniform registers
      umma::fence_after();
      if (H16) {
        gemm1e<IN / 16>(tmem + S::cH1, oX_k, oW0_k, idF, 0);
        gemm2e<1, true>(tmem + S::cDL, oG_k, oW2_mn, idB64, 0);
      } else {
        gemm3e<IN / 16>(tmem + S::cH1, oX_k, oW0_k, idF, 0);
        gemm3e<1>(tmem + S::cDL, oG_k, oW2_mn, idB64, 0);
      }
      umma::commit_elect(&bar);
    }
  };
  // a tile whose output gradients are all zero (Gaussians no pixel of the view
  // used) contributes nothing: its dX rows are zeroed and its MMAs skipped
  auto tile_zero = [&]() {
    bool z = true;
    if (q == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) z &= gr[k] == 0.f;
    }
    return __syncthreads_and(z) != 0;
  };
  bool issued = false;  // stage 1 of the current tile already in flight
  if (blockIdx.x < ntiles) fetch(blockIdx.x);
  int it = 0;
  SS_STAMP(1, 0);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int64_t row = t * 128 + r;
    if (!issued) {
      if (tile_zero()) {
#pragma unroll
        for (int b = 0; b < XSlice<IN>::NB; ++b) {
          const int c = 8 * q + 32 * b;
          if (c < IN && row < n) {
            *reinterpret_cast<float4*>(dX + row * xs + c) = make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4*>(dX + row * xs + c + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        fetch(t + gridDim.x);
        continue;
      }
      wait_w();
      stage_in();
      issue_stage1();
    }
    issued = false;
    SS_STAMP(1, 1 + 8 * it);
    const uint32_t mask1 = (uint32_t)(mr.x >> c0) & 0xFFFFu;  // the forward's ReLU decisions
    const uint32_t mask2 = (uint32_t)(mr.y >> c0) & 0xFFFFu;
    fetch(t + gridDim.x);  // next tile's rows, overlapped with this tile
    sync_mma(&bar, phase);
    SS_STAMP(1, 2 + 8 * it);
    // ---- epilogue 1: H1, D_last
    {
      float v[16];
      umma::tmem_ld16(tmem + S::cH1 + lane + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        v[j] = ((mask1 >> j) & 1) ? rnd(fmaxf(v[j] + sbias[c0 + j], 0.f)) : 0.f;
      if (H16) {
        put8h(sm + S::oH1, r, c0, HC, v);
        put8h(sm + S::oH1, r, c0 + 8, HC, v + 8);
      } else {
        put8(sm + S::oH1, S::H1, r, c0, HC, v);
        put8(sm + S::oH1, S::H1, r, c0 + 8, HC, v + 8);
      }
      umma::tmem_ld16(tmem + S::cDL + lane + c0, v);
      const uint32_t ml = NL == 2 ? mask2 : mask1;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = ((ml >> j) & 1) ? v[j] : 0.f;
      uint8_t* dst = sm + (NL == 2 ? S::oD2 : S::oD1);
      const uint32_t dlo = NL == 2 ? S::D2 : S::D1;
      if (H16) {  // already scaled (G was)
        put8s(dst, dlo, r, c0, 64, v, 1.f);
        put8s(dst, dlo, r, c0 + 8, 64, v + 8, 1.f);
      } else {
        put8(dst, dlo, r, c0, 64, v);
        put8(dst, dlo, r, c0 + 8, 64, v + 8);
      }
    }
    if (NL == 2) {
      // ---- stage 2: H2 = H1 W1;  D1 = D2 W1^T;  dW1^T += D2^T [H1 | 1]
      SS_STAMP(1, 3 + 8 * it);
      to_async();
      if (warp == 0) {
        umma::fence_after();
        if (H16) {
          gemm1e<4>(tmem + S::cH2, oH1_k, oW1_k, idF, 0);
          gemm2e<4, true>(tmem + S::cD1, oD2_k, oW1_mn, idB64, 0);
        } else {
          gemm3e<4>(tmem + S::cH2, oH1_k, oW1_k, idF, 0);
          gemm3e<4>(tmem + S::cD1, oD2_k, oW1_mn, idB64, 0);
        }
        umma::commit_elect(&bar);
        // dW1 reads D2 and H1 only: it runs under the H2 / D1 epilogue
        if (H16) gemm2e<8, true>(tmem + S::cW1, oD2_mn, oH1_mn, idW1, acc_w);
        else gemm3e<8>(tmem + S::cW1, oD2_mn, oH1_mn, idW1, acc_w);
      }
      sync_mma(&bar, phase);
      SS_STAMP(1, 4 + 8 * it);
      float v[16];
      umma::tmem_ld16(tmem + S::cH2 + lane + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        v[j] = ((mask2 >> j) & 1) ? rnd(fmaxf(v[j] + sbias[64 + c0 + j], 0.f)) : 0.f;
      if (H16) {
        put8h(sm + S::oH2, r, c0, 64, v);
        put8h(sm + S::oH2, r, c0 + 8, 64, v + 8);
      } else {
        put8(sm + S::oH2, S::H2, r, c0, 64, v);
        put8(sm + S::oH2, S::H2, r, c0 + 8, 64, v + 8);
      }
      umma::tmem_ld16(tmem + S::cD1 + lane + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = ((mask1 >> j) & 1) ? v[j] : 0.f;
      if (H16) {
        put8s(sm + S::oD1, S::D1, r, c0, 64, v, 1.f);
        put8s(sm + S::oD1, S::D1, r, c0 + 8, 64, v + 8, 1.f);
      } else {
        put8(sm + S::oD1, S::D1, r, c0, 64, v);
        put8(sm + S::oD1, S::D1, r, c0 + 8, 64, v + 8);
      }
    }
    // ---- stage 3: dX = D1 W0^T;  dW0^T += D1^T [X | 1];  dW2 += H_last^T G
    SS_STAMP(1, 5 + 8 * it);
    to_async();
    if (warp == 0) {
      umma::fence_after();
      if (H16) gemm2e<4, true>(tmem + S::cDX, oD1_k, oW0_mn, idBX, 0);
      else gemm3e<4>(tmem + S::cDX, oD1_k, oW0_mn, idBX, 0);
      umma::commit_elect(&bar);
      // dW0 / dW2 (and dW1 before them) read X, G, H, D: they run under the dX
      // epilogue; the next tile's staging waits for bar_w
      if (H16) {
        gemm2e<8, true>(tmem + S::cW0, oD1_mn, oX_mn, idW0, acc_w);
        gemm2e<8, false>(tmem + S::cW2, oHl_mn, oG_mn, idW2, acc_w);
      } else {
        gemm3e<8>(tmem + S::cW0, oD1_mn, oX_mn, idW0, acc_w);
        gemm3e<8>(tmem + S::cW2, oHl_mn, oG_mn, idW2, acc_w);
      }
      umma::commit_elect(&bar_w);
    }
    w_pending = true;
    sync_mma(&bar, phase);
    SS_STAMP(1, 6 + 8 * it);
    acc_w = 1;
    // ---- next tile's stage 1 runs under this tile's dX epilogue
    if (t + gridDim.x < ntiles && !tile_zero()) {
      wait_w();
      stage_in();
      issue_stage1();
      issued = true;
    }
    SS_STAMP(1, 7 + 8 * it);
#pragma unroll
    for (int b = 0; b < XSlice<IN>::NB; ++b) {
      const int c = 8 * q + 32 * b;
      if (c < IN) {  // warp-uniform
        float v[8];
        umma::tmem_ld8(tmem + S::cDX + lane + c, v);
        if (H16) {
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] *= igsc;
        }
        if (row < n) {
          *reinterpret_cast<float4*>(dX + row * xs + c) = make_float4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<float4*>(dX + row * xs + c + 4) = make_float4(v[4], v[5], v[6], v[7]);
        }
      }
    }
  }
  // ---- flush the weight gradients: M = 64 accumulators, row j = 16 (w & 3) + lane
  //      (lanes < 16); the four warps of a lane quarter take 8-column blocks 8q + 32b
  wait_w();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  if (acc_w) {
    const int j = (warp & 3) * 16 + lane_id;
    const bool own = lane_id < 16;
    if (q == 0) {
      float v[8];
      umma::tmem_ld8(tmem + S::cW2 + lane, v);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] *= igsc;
      if (own) {
        red_add_v4(g_params + L::W2 + j * 8, v[0], v[1], v[2], v[3]);
        red_add_v4(g_params + L::W2 + j * 8 + 4, v[4], v[5], v[6], 0.f);
      }
    }
    if (NL == 2) {
      for (int c = 8 * q; c < HC; c += 32) {
        float v[8];
        umma::tmem_ld8(tmem + S::cW1 + lane + c, v);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] *= igsc;
        if (own) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (c + k < 64) atomicAdd(g_params + L::W1 + (c + k) * 64 + j, v[k]);
            else if (c + k == 64) atomicAdd(g_params + L::B1 + j, v[k]);
          }
        }
      }
    }
    for (int c = 8 * q; c < XC; c += 32) {
      float v[8];
      umma::tmem_ld8(tmem + S::cW0 + lane + c, v);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] *= igsc;
      if (own) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (c + k < IN) atomicAdd(g_params + L::W0 + (c + k) * 64 + j, v[k]);
          else if (c + k == IN) atomicAdd(g_params + L::B0 + j, v[k]);
        }
      }
    }
  }
  if (q == 0) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float s = warp_sum(db2[k]);
      if (lane_id == 0) sdb2[warp][k] = s;
    }
  }
  umma::fence_before();
  __syncthreads();
  if (tid < 7) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) s += sdb2[w][tid];
    atomicAdd(g_params + L::B2 + tid, s);
  }
  if (warp == 0) {
    umma::fence_after();
    umma::tmem_free(tmem, 512);
  }
}

// ================================================================= launch
static int g_mlp_mode = 1;  // 0 FFMA fp32, 1 tensor cores 3xTF32 / bf16x3, 2 tensor cores tf32

int mlp_mode() { return g_mlp_mode; }

static int num_sms_tc() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <int IN, int NL, int P>
static int launch_tc(int64_t n, const float* X, int xs, const float* params, float* out, int os,
                     uint64_t* masks, cudaStream_t st) {
  constexpr uint32_t smem = TcFwdSmem<IN, NL, P>::BYTES;
  auto k = mlp_fwd_tc_kernel<IN, NL, P>;
  SS_CUDA(smem_attr_once(k, (int)smem));
  const unsigned grid = (unsigned)std::min<int64_t>((n + 127) / 128, (int64_t)num_sms_tc());
  k<<<grid, NT_FWD, smem, st>>>(n, X, xs, params, out, os, masks);
  SS_CHECK_LAUNCH("mlp_fwd_tc_kernel");
  return SS_OK;
}

int mlp_fwd_tc(int in_pad, int n_hidden, int f16, int64_t n, const float* X, int xs,
               const float* params, float* out, int os, uint64_t* masks, cudaStream_t st) {
  const bool exact = g_mlp_mode != 2;
#define SS_TC(IN, NL)                                                                    \
  if (in_pad == IN && n_hidden == NL)                                                    \
    return f16 ? launch_tc<IN, NL, 0>(n, X, xs, params, out, os, masks, st)             \
               : exact ? launch_tc<IN, NL, 3>(n, X, xs, params, out, os, masks, st)     \
                       : launch_tc<IN, NL, 1>(n, X, xs, params, out, os, masks, st);
  SS_TC(16, 1) SS_TC(16, 2) SS_TC(32, 1) SS_TC(32, 2) SS_TC(64, 1) SS_TC(64, 2)
#undef SS_TC
  set_error("mlp_fwd_tc: unsupported decoder shape");
  return SS_ERR_DATA;
}

template <int IN, int NL, bool H16>
static int launch_bwd_tc(int64_t n, const float* X, int xs, const float* g, int gs,
                         const uint64_t* masks, const float* params, float* dX, float* g_params,
                         cudaStream_t st) {
  constexpr uint32_t smem = TcBwdSmem<IN, NL>::BYTES;
  static_assert(smem <= 220 * 1024, "backward tiles exceed shared memory");
  auto k = mlp_bwd_tc_kernel<IN, NL, H16>;
  SS_CUDA(smem_attr_once(k, (int)smem));
  const unsigned grid = (unsigned)std::min<int64_t>((n + 127) / 128, (int64_t)num_sms_tc());
  k<<<grid, NT, smem, st>>>(n, X, xs, g, gs, masks, params, dX, g_params);
  SS_CHECK_LAUNCH("mlp_bwd_tc_kernel");
  return SS_OK;
}

int mlp_bwd_tc(int in_pad, int n_hidden, int f16, int64_t n, const float* X, int xs,
               const float* g, int gs, const uint64_t* masks, const float* params, float* dX,
               float* g_params, cudaStream_t st) {
  if (!masks) {
    set_error("mlp_bwd_tc: the forward's ReLU masks are required");
    return SS_ERR_DATA;
  }
#define SS_TCB(IN, NL)                                                                 \
  if (in_pad == IN && n_hidden == NL)                                                  \
    return f16 ? launch_bwd_tc<IN, NL, true>(n, X, xs, g, gs, masks, params, dX, g_params, st) \
               : launch_bwd_tc<IN, NL, false>(n, X, xs, g, gs, masks, params, dX, g_params, st);
  SS_TCB(16, 1) SS_TCB(16, 2) SS_TCB(32, 1) SS_TCB(32, 2) SS_TCB(64, 1) SS_TCB(64, 2)
#undef SS_TCB
  set_error("mlp_bwd_tc: unsupported decoder shape");
  return SS_ERR_DATA;
}

}  // namespace ss

extern "C" int ss_set_mlp_mode(int32_t mode) {
  if (mode < 0 || mode > 2) return SS_ERR_DATA;
  ss::g_mlp_mode = mode;
  return SS_OK;
}
extern "C" int32_t ss_get_mlp_mode(void) { return ss::g_mlp_mode; }

// debug: clock64 stamps of CTA 0 (kernel 0 = forward, 1 = backward), 64 each
extern "C" int ss_debug_mlp_events(uint64_t* out) {
  SS_CUDA(cudaMemcpyFromSymbol(out, ss::g_mlp_ev, sizeof(ss::g_mlp_ev)));
  return SS_OK;
}

extern "C" int ss_debug_mlp_trace(uint64_t* out) {
  SS_CUDA(cudaMemcpyFromSymbol(out, ss::g_mlp_trace, sizeof(ss::g_mlp_trace)));
  return SS_OK;
}
