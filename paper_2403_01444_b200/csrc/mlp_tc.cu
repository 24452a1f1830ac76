// NTC decoder forward on the 5th-generation tensor cores (K2f, ntc.py:241-248).
//
// Persistent CTAs of 128 threads walk 128-row tiles of the feature matrix X.
// Per tile, three chained tcgen05.mma.kind::tf32 GEMMs (M = 128 rows,
// N = 64 / 64 / 16, K = in / 64 / 64) accumulate in TMEM; between them each
// thread owns one TMEM lane (= one row): tcgen05.ld, bias + ReLU, and the next
// layer's A tile is written back to shared memory.  Weights are staged once
// per CTA as K-major B tiles.
//
// Precision: P = 3 splits every operand into tf32 hi + lo parts and issues
// A_hi.B_hi + A_hi.B_lo + A_lo.B_hi (3xTF32), which restores fp32-level
// accuracy (the parity tests' 1e-3 gradient bar); P = 1 is plain tf32.
#include "common.cuh"
#include "umma.cuh"

namespace ss {

namespace {
constexpr int HIDT = 64;

template <int IN, int NL>
struct TcLay {  // same packed layout as ntc.cu's Lay<IN, NL>
  static constexpr int W0 = 0, B0 = IN * HIDT, W1 = B0 + HIDT;
  static constexpr int B1 = W1 + (NL == 2 ? HIDT * HIDT : 0);
  static constexpr int W2 = B1 + (NL == 2 ? HIDT : 0);
  static constexpr int B2 = W2 + HIDT * 8;
};

template <int IN, int NL, int P>
struct TcFwdSmem {
  static constexpr uint32_t W0 = umma::tile_bytes(64, IN);
  static constexpr uint32_t W1 = NL == 2 ? umma::tile_bytes(64, 64) : 0;
  static constexpr uint32_t W2 = umma::tile_bytes(16, 64);
  static constexpr uint32_t A = umma::tile_bytes(128, 64);
  static constexpr uint32_t oW0 = 0;
  static constexpr uint32_t oW1 = oW0 + (P == 3 ? 2 : 1) * W0;
  static constexpr uint32_t oW2 = oW1 + (P == 3 ? 2 : 1) * W1;
  static constexpr uint32_t oA0 = oW2 + (P == 3 ? 2 : 1) * W2;
  static constexpr uint32_t oA1 = oA0 + (P == 3 ? 2 : 1) * A;
  static constexpr uint32_t BYTES = oA1 + (P == 3 ? 2 : 1) * A;
};

// write x as (hi, lo) tf32 pair into the hi tile and (for P = 3) the lo tile
template <int P>
__device__ __forceinline__ void put(uint8_t* hi, uint32_t lo_off, uint32_t off, float x) {
  const float h = umma::to_tf32(x);
  *reinterpret_cast<float*>(hi + off) = h;
  if (P == 3) *reinterpret_cast<float*>(hi + lo_off + off) = umma::to_tf32(x - h);
}

// one layer: acc[M=128, N] (+)= A[128, K] . B[N, K]^T over K in steps of 8
template <int P>
__device__ __forceinline__ void mma_layer(uint32_t acc, uint32_t a, uint32_t a_lo_off, int acols,
                                          uint32_t b, uint32_t b_lo_off, int bcols, int K,
                                          uint32_t idesc) {
  for (int k = 0; k < K; k += 8) {
    umma::mma_tf32(acc, umma::desc_k(a, acols, k), umma::desc_k(b, bcols, k), idesc, k > 0);
    if (P == 3) {
      umma::mma_tf32(acc, umma::desc_k(a, acols, k), umma::desc_k(b + b_lo_off, bcols, k), idesc,
                     1);
      umma::mma_tf32(acc, umma::desc_k(a + a_lo_off, acols, k), umma::desc_k(b, bcols, k), idesc,
                     1);
    }
  }
}
}  // namespace

template <int IN, int NL, int P>
__global__ void __launch_bounds__(128, 1) mlp_fwd_tc_kernel(int64_t n, const float* __restrict__ X,
                                                            int xs, const float* __restrict__ params,
                                                            float* __restrict__ out, int os,
                                                            uint64_t* __restrict__ relu_masks) {
  using L = TcLay<IN, NL>;
  using S = TcFwdSmem<IN, NL, P>;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ float sbias[64 + 64 + 8];
  const int tid = threadIdx.x, warp = tid >> 5;
  // ---- stage the weights as K-major B tiles (rows = output unit, cols = input)
  for (int i = tid; i < 64 * IN; i += 128) {
    const int nn = i / IN, k = i % IN;
    put<P>(sm + S::oW0, S::W0, umma::tile_off(nn, k, IN), params[L::W0 + k * 64 + nn]);
  }
  if (NL == 2)
    for (int i = tid; i < 64 * 64; i += 128) {
      const int nn = i / 64, k = i % 64;
      put<P>(sm + S::oW1, S::W1, umma::tile_off(nn, k, 64), params[L::W1 + k * 64 + nn]);
    }
  for (int i = tid; i < 16 * 64; i += 128) {
    const int nn = i / 64, k = i % 64;
    put<P>(sm + S::oW2, S::W2, umma::tile_off(nn, k, 64), nn < 8 ? params[L::W2 + k * 8 + nn] : 0.f);
  }
  for (int i = tid; i < 64; i += 128) {
    sbias[i] = params[L::B0 + i];
    sbias[64 + i] = NL == 2 ? params[L::B1 + i] : 0.f;
  }
  if (tid < 8) sbias[128 + tid] = params[L::B2 + tid];
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc(&tbase, 256);
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tbase;
  const uint32_t acc1 = tmem, acc2 = tmem + 64, acc3 = tmem + 128;
  const uint32_t lane = (uint32_t)(warp * 32) << 16;
  const uint32_t sW0 = umma::smem_u32(sm + S::oW0), sW1 = umma::smem_u32(sm + S::oW1);
  const uint32_t sW2 = umma::smem_u32(sm + S::oW2);
  const uint32_t sA0 = umma::smem_u32(sm + S::oA0), sA1 = umma::smem_u32(sm + S::oA1);
  constexpr uint32_t id64 = umma::idesc_tf32(128, 64, 0, 0);
  constexpr uint32_t id16 = umma::idesc_tf32(128, 16, 0, 0);
  uint32_t phase = 0;
  const int64_t ntiles = (n + 127) / 128;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row = t * 128 + tid;
    // ---- X row -> A0 (IN columns)
#pragma unroll
    for (int k = 0; k < IN; k += 4) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < n) v = *reinterpret_cast<const float4*>(X + row * xs + k);
      put<P>(sm + S::oA0, S::A, umma::tile_off(tid, k, IN), v.x);
      put<P>(sm + S::oA0, S::A, umma::tile_off(tid, k + 1, IN), v.y);
      put<P>(sm + S::oA0, S::A, umma::tile_off(tid, k + 2, IN), v.z);
      put<P>(sm + S::oA0, S::A, umma::tile_off(tid, k + 3, IN), v.w);
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    if (tid == 0) {
      umma::fence_after();
      mma_layer<P>(acc1, sA0, S::A, IN, sW0, S::W0, IN, IN, id64);
      umma::commit(&bar);
    }
    umma::mbar_wait(&bar, phase);
    phase ^= 1;
    umma::fence_after();
    // ---- h1 = relu(acc1 + b0) -> A1 (64 columns)
    uint64_t m1 = 0, m2 = 0;
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 16) {
      float v[16];
      umma::tmem_ld16(acc1 + lane + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float h = fmaxf(v[j] + sbias[c0 + j], 0.f);
        m1 |= (uint64_t)(h > 0.f) << (c0 + j);
        put<P>(sm + S::oA1, S::A, umma::tile_off(tid, c0 + j, 64), h);
      }
    }
    uint32_t last = sA1;
    uint32_t last_lo = S::A;
    if (NL == 2) {
      umma::fence_proxy_async();
      umma::fence_before();
      __syncthreads();
      if (tid == 0) {
        umma::fence_after();
        mma_layer<P>(acc2, sA1, S::A, 64, sW1, S::W1, 64, 64, id64);
        umma::commit(&bar);
      }
      umma::mbar_wait(&bar, phase);
      phase ^= 1;
      umma::fence_after();
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        float v[16];
        umma::tmem_ld16(acc2 + lane + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float h = fmaxf(v[j] + sbias[64 + c0 + j], 0.f);
          m2 |= (uint64_t)(h > 0.f) << (c0 + j);
          put<P>(sm + S::oA0, S::A, umma::tile_off(tid, c0 + j, 64), h);
        }
      }
      last = sA0;
    } else {
      m2 = m1;
    }
    // the backward reuses the forward's ReLU decisions (self-consistent gradient)
    if (relu_masks && row < n)
      *reinterpret_cast<ulonglong2*>(relu_masks + 2 * row) = make_ulonglong2(m1, m2);
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    if (tid == 0) {
      umma::fence_after();
      mma_layer<P>(acc3, last, last_lo, 64, sW2, S::W2, 64, 64, id16);
      umma::commit(&bar);
    }
    umma::mbar_wait(&bar, phase);
    phase ^= 1;
    umma::fence_after();
    float o[8];
    umma::tmem_ld8(acc3 + lane, o);
    if (row < n) {
      if (os == 8) {
        *reinterpret_cast<float4*>(out + row * 8) =
            make_float4(o[0] + sbias[128], o[1] + sbias[129], o[2] + sbias[130], o[3] + sbias[131]);
        *reinterpret_cast<float4*>(out + row * 8 + 4) =
            make_float4(o[4] + sbias[132], o[5] + sbias[133], o[6] + sbias[134], 0.f);
      } else {
#pragma unroll
        for (int k = 0; k < 7; ++k) out[row * os + k] = o[k] + sbias[128 + k];
      }
    }
    umma::fence_before();
    __syncthreads();  // TMEM and the A tiles are reused by the next tile
  }
  if (warp == 0) {
    umma::fence_after();
    umma::tmem_free(tmem, 256);
  }
}

// ------------------------------------------------------------------ backward
// K2b on the tensor cores (ntc.py:258-276).  Persistent CTAs of 128 threads
// walk 128-row tiles; per tile, with every operand split into bf16 hi + lo
// parts (kind::f16, three products per K step, fp32 accumulation in TMEM):
//
//   recompute  H1 = relu(X W0 + b0), H2 = relu(H1 W1 + b1)      (M = 128)
//   deltas     DL = (G W2^T) * [H_last > 0]
//              D1 = (D2 W1^T) * [H1 > 0]                         (NL = 2)
//              dX = D1 W0^T  -> HBM for the table scatter
//   weights    dW2   += H_last^T G                                (M = 64, N = 8)
//              dW1^T += D2^T [H1 | 1]   (column 64 = db1)         (M = 64, N = 72)
//              dW0^T += D1^T [X | 1]    (column IN = db0)         (M = 64, N = IN + 8)
//
// The weight-gradient accumulators stay in TMEM across all tiles of the CTA
// and are flushed once with reductions into g_params.  Transposed operands are
// the same shared-memory tiles read through MN-major descriptors, so each
// activation is staged exactly once.  db2 is summed in registers.
namespace {
template <int IN, int NL>
struct TcBwdSmem {
  static constexpr int XC = IN + 8, HC = 72;
  static constexpr uint32_t W0 = umma::tile16_bytes(64, IN);
  static constexpr uint32_t W1 = NL == 2 ? umma::tile16_bytes(64, 64) : 0;
  static constexpr uint32_t W2 = umma::tile16_bytes(16, 64);
  static constexpr uint32_t X = umma::tile16_bytes(128, XC);
  static constexpr uint32_t H1 = umma::tile16_bytes(128, HC);
  static constexpr uint32_t H2 = umma::tile16_bytes(128, 64);  // H2, then D1
  static constexpr uint32_t G = umma::tile16_bytes(128, 16);
  static constexpr uint32_t D2 = NL == 2 ? umma::tile16_bytes(128, 64) : 0;
  // every tile is followed by its lo plane (same size)
  static constexpr uint32_t oW0 = 0, oW1 = oW0 + 2 * W0, oW2 = oW1 + 2 * W1;
  static constexpr uint32_t oX = oW2 + 2 * W2, oH1 = oX + 2 * X, oH2 = oH1 + 2 * H1;
  static constexpr uint32_t oG = oH2 + 2 * H2, oD2 = oG + 2 * G;
  static constexpr uint32_t BYTES = oD2 + 2 * D2;
  // TMEM columns
  static constexpr uint32_t cH1 = 0, cH2 = 64, cDL = 128, cD1 = 192, cDX = 256;
  static constexpr uint32_t cW2 = 320, cW1 = 328, cW0 = 400;
};

struct Op16 {
  uint32_t addr, lo;  // hi plane address, byte distance to the lo plane
  int cols, mn;       // stored tile columns, MN-major read
};

__device__ __forceinline__ uint64_t op_desc(const Op16& o, int k, int lo) {
  const uint32_t a = o.addr + (lo ? o.lo : 0u);
  return o.mn ? umma::desc16_mn(a, o.cols, k) : umma::desc16_k(a, o.cols, k);
}

// acc (+)= A . B over K (multiple of 16) with the 3-product bf16 split
__device__ __forceinline__ void gemm3(uint32_t acc, const Op16& A, const Op16& B, int K,
                                      uint32_t idesc, uint32_t accumulate) {
  for (int k = 0; k < K; k += 16) {
    umma::mma_bf16(acc, op_desc(A, k, 0), op_desc(B, k, 0), idesc, accumulate | (k > 0));
    umma::mma_bf16(acc, op_desc(A, k, 0), op_desc(B, k, 1), idesc, 1);
    umma::mma_bf16(acc, op_desc(A, k, 1), op_desc(B, k, 0), idesc, 1);
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

__device__ __forceinline__ void sync_mma(uint64_t* bar, uint32_t& phase) {
  umma::mbar_wait(bar, phase);
  phase ^= 1;
  umma::fence_after();
}

__device__ __forceinline__ void to_async() {
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
}

// TMEM row (64 columns from col) -> f(row values, column block) in blocks of 16
template <class Fn>
__device__ __forceinline__ void tmem_row64(uint32_t taddr, Fn&& fn) {
#pragma unroll
  for (int c0 = 0; c0 < 64; c0 += 16) {
    float v[16];
    umma::tmem_ld16(taddr + c0, v);
    fn(v, c0);
  }
}
}  // namespace

template <int IN, int NL>
__global__ void __launch_bounds__(128, 1) mlp_bwd_tc_kernel(
    int64_t n, const float* __restrict__ X, int xs, const float* __restrict__ g_out, int gs,
    const uint64_t* __restrict__ relu_masks, const float* __restrict__ params,
    float* __restrict__ dX, float* __restrict__ g_params) {
  using L = TcLay<IN, NL>;
  using S = TcBwdSmem<IN, NL>;
  constexpr int XC = S::XC, HC = S::HC;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ float sbias[128];
  const int tid = threadIdx.x, warp = tid >> 5, lane_id = tid & 31;
  // ---- weights as bf16 hi/lo tiles: W0t (j, f) = W0[f][j]; W1t (j, i) = W1[i][j];
  //      W2t (o, j) = W2[j][o] (rows 7..15 zero)
  for (int i = tid; i < 64 * IN; i += 128) {
    const int j = i / IN, f = i % IN;
    put_scalar(sm + S::oW0, S::W0, j, f, IN, params[L::W0 + f * 64 + j]);
  }
  if (NL == 2)
    for (int i = tid; i < 64 * 64; i += 128) {
      const int j = i / 64, k = i % 64;
      put_scalar(sm + S::oW1, S::W1, j, k, 64, params[L::W1 + k * 64 + j]);
    }
  for (int i = tid; i < 16 * 64; i += 128) {
    const int o = i / 64, j = i % 64;
    put_scalar(sm + S::oW2, S::W2, o, j, 64, o < 7 ? params[L::W2 + j * 8 + o] : 0.f);
  }
  if (tid < 64) {
    sbias[tid] = params[L::B0 + tid];
    sbias[64 + tid] = NL == 2 ? params[L::B1 + tid] : 0.f;
  }
  // constant columns: X col IN = 1 (db0), H1 col 64 = 1 (db1), the rest of the pads 0
  {
    float pad[8] = {1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    put8(sm + S::oX, S::X, tid, IN, XC, pad);
    put8(sm + S::oH1, S::H1, tid, 64, HC, pad);
    float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    put8(sm + S::oG, S::G, tid, 8, 16, z);
  }
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc(&tbase, 512);
  to_async();
  umma::fence_after();
  const uint32_t tmem = tbase;
  const uint32_t lane = (uint32_t)(warp * 32) << 16;
  const Op16 oX_k{umma::smem_u32(sm + S::oX), S::X, XC, 0};
  const Op16 oX_mn{oX_k.addr, S::X, XC, 1};
  const Op16 oW0_k{umma::smem_u32(sm + S::oW0), S::W0, IN, 0};
  const Op16 oW0_mn{oW0_k.addr, S::W0, IN, 1};
  const Op16 oW1_k{umma::smem_u32(sm + S::oW1), S::W1, 64, 0};
  const Op16 oW1_mn{oW1_k.addr, S::W1, 64, 1};
  const Op16 oW2_mn{umma::smem_u32(sm + S::oW2), S::W2, 64, 1};
  const Op16 oH1_k{umma::smem_u32(sm + S::oH1), S::H1, HC, 0};
  const Op16 oH1_mn{oH1_k.addr, S::H1, HC, 1};
  const Op16 oH2_k{umma::smem_u32(sm + S::oH2), S::H2, 64, 0};  // also D1
  const Op16 oH2_mn{oH2_k.addr, S::H2, 64, 1};
  const Op16 oG_k{umma::smem_u32(sm + S::oG), S::G, 16, 0};
  const Op16 oG_mn{oG_k.addr, S::G, 16, 1};
  const Op16 oD2_k{umma::smem_u32(sm + S::oD2), S::D2, 64, 0};
  const Op16 oD2_mn{oD2_k.addr, S::D2, 64, 1};
  const Op16 oHl_mn = NL == 2 ? oH2_mn : oH1_mn;
  constexpr uint32_t idF = umma::idesc_bf16(128, 64, 0, 0);
  constexpr uint32_t idB64 = umma::idesc_bf16(128, 64, 0, 1);
  constexpr uint32_t idBX = umma::idesc_bf16(128, IN, 0, 1);
  constexpr uint32_t idW2 = umma::idesc_bf16(64, 8, 1, 1);
  constexpr uint32_t idW1 = umma::idesc_bf16(64, HC, 1, 1);
  constexpr uint32_t idW0 = umma::idesc_bf16(64, XC, 1, 1);
  uint32_t phase = 0, acc_w = 0;
  float db2[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int64_t ntiles = (n + 127) / 128;
  // register prefetch of this thread's X and g rows for the first tile
  float xr[IN], gr[8];
  ulonglong2 mr;
  auto fetch = [&](int64_t t) {
    const int64_t row = t * 128 + tid;
    const bool ok = t < ntiles && row < n;
    mr = ok ? __ldg(reinterpret_cast<const ulonglong2*>(relu_masks) + row) : make_ulonglong2(0, 0);
#pragma unroll
    for (int k = 0; k < IN; k += 4) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ok) v = __ldg(reinterpret_cast<const float4*>(X + row * xs + k));
      xr[k] = v.x, xr[k + 1] = v.y, xr[k + 2] = v.z, xr[k + 3] = v.w;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) gr[k] = (ok && k < 7) ? __ldg(g_out + row * gs + k) : 0.f;
  };
  fetch(blockIdx.x);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row = t * 128 + tid;
    // ---- stage A: X -> smem, H1 = X W0 (+ b0)
#pragma unroll
    for (int k = 0; k < IN; k += 8) put8(sm + S::oX, S::X, tid, k, XC, xr + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) db2[k] += gr[k];
    put8(sm + S::oG, S::G, tid, 0, 16, gr);
    to_async();
    if (tid == 0) {
      umma::fence_after();
      gemm3(tmem + S::cH1, oX_k, oW0_k, IN, idF, 0);
      umma::commit(&bar);
    }
    const uint64_t mask1 = mr.x, mask2 = mr.y;  // the forward's ReLU decisions
    fetch(t + gridDim.x);  // next tile's rows, overlapped with this tile
    sync_mma(&bar, phase);
    tmem_row64(tmem + S::cH1 + lane, [&](float (&v)[16], int c0) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        v[j] = ((mask1 >> (c0 + j)) & 1) ? fmaxf(v[j] + sbias[c0 + j], 0.f) : 0.f;
      put8(sm + S::oH1, S::H1, tid, c0, HC, v);
      put8(sm + S::oH1, S::H1, tid, c0 + 8, HC, v + 8);
    });
    if (NL == 2) {
      // ---- stage B: H2 = H1 W1 (+ b1)
      to_async();
      if (tid == 0) {
        umma::fence_after();
        gemm3(tmem + S::cH2, oH1_k, oW1_k, 64, idF, 0);
        umma::commit(&bar);
      }
      sync_mma(&bar, phase);
      tmem_row64(tmem + S::cH2 + lane, [&](float (&v)[16], int c0) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          v[j] = ((mask2 >> (c0 + j)) & 1) ? fmaxf(v[j] + sbias[64 + c0 + j], 0.f) : 0.f;
        put8(sm + S::oH2, S::H2, tid, c0, 64, v);
        put8(sm + S::oH2, S::H2, tid, c0 + 8, 64, v + 8);
      });
    }
    // ---- stage C: DL = G W2^T;  dW2 += H_last^T G
    to_async();
    if (tid == 0) {
      umma::fence_after();
      gemm3(tmem + S::cDL, oG_k, oW2_mn, 16, idB64, 0);
      gemm3(tmem + S::cW2, oHl_mn, oG_mn, 128, idW2, acc_w);
      umma::commit(&bar);
    }
    sync_mma(&bar, phase);
    {
      // NL = 2: DL = D2 (own tile); NL = 1: DL = D1 (the H2 tile)
      uint8_t* dst = sm + (NL == 2 ? S::oD2 : S::oH2);
      const uint32_t dlo = NL == 2 ? S::D2 : S::H2;
      tmem_row64(tmem + S::cDL + lane, [&](float (&v)[16], int c0) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ((mask2 >> (c0 + j)) & 1) ? v[j] : 0.f;
        put8(dst, dlo, tid, c0, 64, v);
        put8(dst, dlo, tid, c0 + 8, 64, v + 8);
      });
    }
    if (NL == 2) {
      // ---- stage D: D1 = D2 W1^T * mask1;  dW1^T += D2^T [H1 | 1]
      to_async();
      if (tid == 0) {
        umma::fence_after();
        gemm3(tmem + S::cD1, oD2_k, oW1_mn, 64, idB64, 0);
        gemm3(tmem + S::cW1, oD2_mn, oH1_mn, 128, idW1, acc_w);
        umma::commit(&bar);
      }
      sync_mma(&bar, phase);
      tmem_row64(tmem + S::cD1 + lane, [&](float (&v)[16], int c0) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ((mask1 >> (c0 + j)) & 1) ? v[j] : 0.f;
        put8(sm + S::oH2, S::H2, tid, c0, 64, v);
        put8(sm + S::oH2, S::H2, tid, c0 + 8, 64, v + 8);
      });
    }
    // ---- stage E: dX = D1 W0^T;  dW0^T += D1^T [X | 1]
    to_async();
    if (tid == 0) {
      umma::fence_after();
      gemm3(tmem + S::cDX, oH2_k, oW0_mn, 64, idBX, 0);
      gemm3(tmem + S::cW0, oH2_mn, oX_mn, 128, idW0, acc_w);
      umma::commit(&bar);
    }
    sync_mma(&bar, phase);
    acc_w = 1;
#pragma unroll
    for (int c0 = 0; c0 < IN; c0 += 16) {
      float v[16];
      umma::tmem_ld16(tmem + S::cDX + lane + c0, v);
      if (row < n) {
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(dX + row * xs + c0 + j) =
              make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
    umma::fence_before();
    __syncthreads();  // the tiles of this iteration are rewritten by the next
  }
  // ---- flush the weight gradients: M = 64 accumulators, row j = 16 w + lane (lane < 16)
  umma::fence_after();
  if (acc_w) {
    const int j = warp * 16 + lane_id;
    const bool own = lane_id < 16;
    {
      float v[8];
      umma::tmem_ld8(tmem + S::cW2 + lane, v);
      if (own) {
        red_add_v4(g_params + L::W2 + j * 8, v[0], v[1], v[2], v[3]);
        red_add_v4(g_params + L::W2 + j * 8 + 4, v[4], v[5], v[6], 0.f);
      }
    }
    if (NL == 2) {
      tmem_row64(tmem + S::cW1 + lane, [&](float (&v)[16], int c0) {
        if (own) {
#pragma unroll
          for (int q = 0; q < 16; ++q) atomicAdd(g_params + L::W1 + (c0 + q) * 64 + j, v[q]);
        }
      });
      float v[8];
      umma::tmem_ld8(tmem + S::cW1 + 64 + lane, v);
      if (own) atomicAdd(g_params + L::B1 + j, v[0]);
    }
#pragma unroll
    for (int c0 = 0; c0 < IN; c0 += 16) {
      float v[16];
      umma::tmem_ld16(tmem + S::cW0 + lane + c0, v);
      if (own) {
#pragma unroll
        for (int q = 0; q < 16; ++q) atomicAdd(g_params + L::W0 + (c0 + q) * 64 + j, v[q]);
      }
    }
    {
      float v[8];
      umma::tmem_ld8(tmem + S::cW0 + IN + lane, v);
      if (own) atomicAdd(g_params + L::B0 + j, v[0]);
    }
  }
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const float s = warp_sum(db2[k]);
    if (lane_id == 0) atomicAdd(g_params + L::B2 + k, s);
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) {
    umma::fence_after();
    umma::tmem_free(tmem, 512);
  }
}

template <int IN, int NL>
static int launch_bwd_tc(int64_t n, const float* X, int xs, const float* g, int gs,
                         const uint64_t* masks, const float* params, float* dX, float* g_params,
                         cudaStream_t st) {
  constexpr uint32_t smem = TcBwdSmem<IN, NL>::BYTES;
  static_assert(smem <= 220 * 1024, "backward tiles exceed shared memory");
  auto k = mlp_bwd_tc_kernel<IN, NL>;
  SS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<int64_t>((n + 127) / 128, (int64_t)sms);
  k<<<grid, 128, smem, st>>>(n, X, xs, g, gs, masks, params, dX, g_params);
  SS_CHECK_LAUNCH("mlp_bwd_tc_kernel");
  return SS_OK;
}

int mlp_bwd_tc(int in_pad, int n_hidden, int64_t n, const float* X, int xs, const float* g,
               int gs, const uint64_t* masks, const float* params, float* dX, float* g_params,
               cudaStream_t st) {
  if (!masks) {
    set_error("mlp_bwd_tc: the forward's ReLU masks are required");
    return SS_ERR_DATA;
  }
#define SS_TCB(IN, NL)                   \
  if (in_pad == IN && n_hidden == NL) \
    return launch_bwd_tc<IN, NL>(n, X, xs, g, gs, masks, params, dX, g_params, st);
  SS_TCB(16, 1) SS_TCB(16, 2) SS_TCB(32, 1) SS_TCB(32, 2) SS_TCB(64, 1) SS_TCB(64, 2)
#undef SS_TCB
  set_error("mlp_bwd_tc: unsupported decoder shape");
  return SS_ERR_DATA;
}

static int g_mlp_mode = 1;  // 0 FFMA fp32, 1 tensor cores 3xTF32, 2 tensor cores tf32

int mlp_mode() { return g_mlp_mode; }

template <int IN, int NL, int P>
static int launch_tc(int64_t n, const float* X, int xs, const float* params, float* out, int os,
                     uint64_t* masks, cudaStream_t st) {
  constexpr uint32_t smem = TcFwdSmem<IN, NL, P>::BYTES;
  auto k = mlp_fwd_tc_kernel<IN, NL, P>;
  SS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_sm = smem <= 100 * 1024 ? 2 : 1;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 127) / 128, (int64_t)sms * per_sm);
  k<<<grid, 128, smem, st>>>(n, X, xs, params, out, os, masks);
  SS_CHECK_LAUNCH("mlp_fwd_tc_kernel");
  return SS_OK;
}

int mlp_fwd_tc(int in_pad, int n_hidden, int64_t n, const float* X, int xs, const float* params,
               float* out, int os, uint64_t* masks, cudaStream_t st) {
  const bool exact = g_mlp_mode != 2;
#define SS_TC(IN, NL)                                                                    \
  if (in_pad == IN && n_hidden == NL)                                                    \
    return exact ? launch_tc<IN, NL, 3>(n, X, xs, params, out, os, masks, st)           \
                 : launch_tc<IN, NL, 1>(n, X, xs, params, out, os, masks, st);
  SS_TC(16, 1) SS_TC(16, 2) SS_TC(32, 1) SS_TC(32, 2) SS_TC(64, 1) SS_TC(64, 2)
#undef SS_TC
  set_error("mlp_fwd_tc: unsupported decoder shape");
  return SS_ERR_DATA;
}

}  // namespace ss

extern "C" int ss_set_mlp_mode(int32_t mode) {
  if (mode < 0 || mode > 2) return SS_ERR_DATA;
  ss::g_mlp_mode = mode;
  return SS_OK;
}
extern "C" int32_t ss_get_mlp_mode(void) { return ss::g_mlp_mode; }
