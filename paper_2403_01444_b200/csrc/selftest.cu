// Self-test of the tcgen05 building blocks (umma.cuh) on the device.
// D[M x N] = opA . opB with opA = A (M x K) when a_mn == 0 else TA^T where TA is
// (K x M); likewise opB^T = Bt (N x K) or TB (K x N).  Operand matrices are
// row-major fp32 in global memory and are staged as K-major tiles of their
// stored shape; `swap` exchanges LBO/SBO of the MN-major descriptors (probe).
// If `raw` the 128 TMEM lanes are dumped instead of the M rows.
//
// Measured on B200 / CUDA 12.9 / driver 580: K-major tf32 operands are exact
// for M = 128 and M = 64; every MN-major (transposed) tf32 operand variant,
// with either LBO/SBO assignment, leaves the accumulator untouched.  The
// kernels therefore only use K-major tiles.
#include "common.cuh"
#include "umma.cuh"

namespace ss {

__global__ void __launch_bounds__(128) umma_selftest_kernel(const float* __restrict__ A,
                                                            const float* __restrict__ B,
                                                            float* __restrict__ D, int M, int N,
                                                            int K, int a_mn, int b_mn, int swap,
                                                            int raw, int a_tmem) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int AR = a_mn ? K : M, AC = a_mn ? M : K;
  const int BR = b_mn ? K : N, BC = b_mn ? N : K;
  uint8_t* sa = sm;
  uint8_t* sb = sm + umma::tile_bytes(AR, AC);
  for (int i = tid; i < AR * AC; i += 128)
    *reinterpret_cast<float*>(sa + umma::tile_off(i / AC, i % AC, AC)) = umma::to_tf32(A[i]);
  for (int i = tid; i < BR * BC; i += 128)
    *reinterpret_cast<float*>(sb + umma::tile_off(i / BC, i % BC, BC)) = umma::to_tf32(B[i]);
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc(&tbase, a_tmem ? 256 : 64);
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tbase;
  if (a_tmem) {  // A (M = 128, K-major) -> TMEM columns 128.., row i in lane i
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    for (int c0 = 0; c0 < K; c0 += 8) {
      float v[8];
      for (int j = 0; j < 8; ++j) v[j] = umma::to_tf32(A[tid * K + c0 + j]);
      umma::tmem_st8(tmem + lane_base + 128u + (uint32_t)c0, v);
    }
    umma::tmem_st_wait();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
  }
  if (tid == 0) {
    const uint32_t a0 = umma::smem_u32(sa), b0 = umma::smem_u32(sb);
    const uint32_t id = umma::idesc_tf32(M, N, a_mn, b_mn);
    for (int k = 0; k < K; k += 8) {
      if (a_tmem) {
        umma::mma_tf32_ts(tmem, tmem + 128u + (uint32_t)k, umma::desc_k(b0, BC, k), id, k > 0);
        continue;
      }
      uint64_t da, db;
      if (a_mn)
        da = swap ? umma::desc(a0 + (k >> 3) * umma::tile_sbo(AC), 128u, umma::tile_sbo(AC))
                  : umma::desc_mn(a0, AC, k);
      else
        da = umma::desc_k(a0, AC, k);
      if (b_mn)
        db = swap ? umma::desc(b0 + (k >> 3) * umma::tile_sbo(BC), 128u, umma::tile_sbo(BC))
                  : umma::desc_mn(b0, BC, k);
      else
        db = umma::desc_k(b0, BC, k);
      umma::mma_tf32(tmem, da, db, id, k > 0);
    }
    umma::commit(&bar);
  }
  umma::mbar_wait(&bar, 0);
  umma::fence_after();
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  for (int c0 = 0; c0 < N; c0 += 8) {
    float v[8];
    umma::tmem_ld8(tmem + lane_base + (uint32_t)c0, v);
    int row = -1;
    if (M == 128 || raw) row = tid;
    else if (lane < 16) row = warp * 16 + lane;
    if (row >= 0)
      for (int j = 0; j < 8 && c0 + j < N; ++j) D[row * N + c0 + j] = v[j];
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free(tmem, a_tmem ? 256 : 64);
}

// kind::f16 (bf16) variant: operands rounded to bf16, K steps of 16,
// MN-major operands read from the stored (K x MN) tile via desc16_mn.
__global__ void __launch_bounds__(128) umma_selftest16_kernel(const float* __restrict__ A,
                                                              const float* __restrict__ B,
                                                              float* __restrict__ D, int M, int N,
                                                              int K, int a_mn, int b_mn, int swap,
                                                              int raw) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int AR = a_mn ? K : M, AC = a_mn ? M : K;
  const int BR = b_mn ? K : N, BC = b_mn ? N : K;
  uint8_t* sa = sm;
  uint8_t* sb = sm + umma::tile16_bytes(AR, AC);
  for (int i = tid; i < AR * AC; i += 128)
    *reinterpret_cast<__nv_bfloat16*>(sa + umma::tile16_off(i / AC, i % AC, AC)) =
        __float2bfloat16_rn(A[i]);
  for (int i = tid; i < BR * BC; i += 128)
    *reinterpret_cast<__nv_bfloat16*>(sb + umma::tile16_off(i / BC, i % BC, BC)) =
        __float2bfloat16_rn(B[i]);
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc(&tbase, 128);
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t a0 = umma::smem_u32(sa), b0 = umma::smem_u32(sb);
    const uint32_t id = umma::idesc_bf16(M, N, a_mn, b_mn);
    for (int k = 0; k < K; k += 16) {
      const uint64_t da = a_mn ? umma::desc16_mn(a0, AC, k, 0, swap) : umma::desc16_k(a0, AC, k);
      const uint64_t db = b_mn ? umma::desc16_mn(b0, BC, k, 0, swap) : umma::desc16_k(b0, BC, k);
      umma::mma_bf16(tmem, da, db, id, k > 0);
    }
    umma::commit(&bar);
  }
  umma::mbar_wait(&bar, 0);
  umma::fence_after();
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  for (int c0 = 0; c0 < N; c0 += 8) {
    float v[8];
    umma::tmem_ld8(tmem + lane_base + (uint32_t)c0, v);
    int row = -1;
    if (M == 128 || raw) row = tid;
    else if (lane < 16) row = warp * 16 + lane;
    if (row >= 0)
      for (int j = 0; j < 8 && c0 + j < N; ++j) D[row * N + c0 + j] = v[j];
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free(tmem, 128);
}

// Issue-rate probe: `count` back-to-back M = 128 MMAs (K = 8 tf32 / 16 bf16
// per instruction, fixed operands) issued by one thread; out[0] = cycles from
// the first issue to the commit's completion, out[1] = cycles spent issuing.
__global__ void __launch_bounds__(128) umma_rate_kernel(int kind, int N, int a_tmem, int count,
                                                        unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // operands: zeros, or (kind bit 6) pseudo-random values (data-dependent MMA rate)
  for (int i = tid; i < (128 * 64 * 4 + 128 * 128 * 2) / 4; i += 128) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 15;
    reinterpret_cast<uint32_t*>(sm)[i] = (kind & 64) ? (h & 0x3fff3fffu) | 0x3c003c00u : 0u;
  }
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
  if (tid == 0) {
    const uint32_t a0 = umma::smem_u32(sm), b0 = umma::smem_u32(sm + 128 * 64 * 4);
    // kind bits: 0 tf32 / 1 bf16; bit 1: MN-major A and B (bf16); bit 2:
    // SWIZZLE_128B K-major descriptors (bf16; timing only, data ignored);
    // bit 3: M = 64
    const int bf = kind & 1, mn = (kind >> 1) & 1, swz = (kind >> 2) & 1, M = (kind & 8) ? 64 : 128;
    uint64_t da = bf ? (mn ? umma::desc16_mn(a0, 128, 0) : umma::desc16_k(a0, 64, 0))
                     : umma::desc_k(a0, 32, 0);
    uint64_t db = bf ? (mn ? umma::desc16_mn(b0, 128, 0) : umma::desc16_k(b0, 64, 0))
                     : umma::desc_k(b0, 32, 0);
    if (swz) {
      da = umma::desc(a0, 16u, 1024u) | (2ull << 61);
      db = umma::desc(b0, 16u, 1024u) | (2ull << 61);
    }
    const uint32_t id = bf ? umma::idesc_bf16(M, N, mn, mn) : umma::idesc_tf32(M, N, 0, 0);
    unsigned long long c0 = clock64();
    // 16 MMAs per unrolled group, one code path per variant
#define SS_RATE_LOOP(CALL)                       \
  for (int i = 0; i < count; i += 16) {          \
    _Pragma("unroll") for (int j = 0; j < 16; ++j) CALL; \
  }
    if (kind & 32) {  // the decoder backward's weight-gradient GEMM: M = 64, A = D^T (MN-major,
                      // tile cols 64), B = [H | 1] (MN-major, tile cols N), K = 128 rows
      const uint64_t A0 = umma::desc16_mn(a0, 64, 0), B0 = umma::desc16_mn(b0, N, 0);
      const uint32_t ks_a = (2u * umma::sbo16(64)) >> 4, ks_b = (2u * umma::sbo16(N)) >> 4;
      const uint32_t idw = umma::idesc_bf16(64, N, 1, 1);
      for (int i = 0; i < count; i += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma::mma_bf16(tmem, A0 + (uint64_t)ks_a * k, B0 + (uint64_t)ks_b * k, idw, 1);
      }
    } else if (kind & 16) {  // bf16 3-product pattern over a K = 64 tile: A/B hi/lo alternate, K advances
      const uint64_t dal = da + (uint64_t)((64 * 16 * 2) >> 4), dbl = db + (uint64_t)((64 * 16 * 2) >> 4);
      for (int i = 0; i < count; i += 12) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t o = (uint64_t)(256u >> 4) * k;
          umma::mma_bf16(tmem, da + o, db + o, id, 1);
          umma::mma_bf16(tmem, da + o, dbl + o, id, 1);
          umma::mma_bf16(tmem, dal + o, db + o, id, 1);
        }
      }
    } else if (kind & 1) {
      SS_RATE_LOOP(umma::mma_bf16(tmem, da, db, id, 1))
    } else if (a_tmem) {
      SS_RATE_LOOP(umma::mma_tf32_ts(tmem, tmem + 128u, db, id, 1))
    } else {
      SS_RATE_LOOP(umma::mma_tf32(tmem, da, db, id, 1))
    }
#undef SS_RATE_LOOP
    const unsigned long long c1 = clock64();
    umma::commit(&bar);
    umma::mbar_wait(&bar, 0);
    const unsigned long long c2 = clock64();
    out[0] = c2 - c0;
    out[1] = c1 - c0;
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free(tmem, 256);
}

}  // namespace ss

// flags: bit0 a_mn, bit1 b_mn, bit2 swap, bit3 raw, bit4 bf16 (kind::f16),
// bit5 A from TMEM (tf32, M = 128, K-major)
extern "C" int ss_selftest_umma(int32_t M, int32_t N, int32_t K, int32_t flags, const float* A,
                                const float* B, float* D, void* stream) {
  const int bf16 = (flags >> 4) & 1;
  if ((M != 64 && M != 128) || N < 8 || N > 128 || N % 8 || K < 8 || K > 128 ||
      K % (bf16 ? 16 : 8) || (!bf16 && N > 64))
    return SS_ERR_DATA;
  const int a_mn = flags & 1, b_mn = (flags >> 1) & 1;
  if (bf16) {
    const size_t smem = ss::umma::tile16_bytes(a_mn ? K : M, a_mn ? M : K) +
                        ss::umma::tile16_bytes(b_mn ? K : N, b_mn ? N : K);
    auto k = ss::umma_selftest16_kernel;
    SS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<1, 128, smem, ss::as_stream(stream)>>>(A, B, D, M, N, K, a_mn, b_mn, (flags >> 2) & 1,
                                               (flags >> 3) & 1);
    SS_CHECK_LAUNCH("umma_selftest16_kernel");
    return SS_OK;
  }
  const size_t smem = ss::umma::tile_bytes(a_mn ? K : M, a_mn ? M : K) +
                      ss::umma::tile_bytes(b_mn ? K : N, b_mn ? N : K);
  auto k = ss::umma_selftest_kernel;
  SS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int a_tmem = (flags >> 5) & 1;
  if (a_tmem && (M != 128 || a_mn)) return SS_ERR_DATA;
  k<<<1, 128, smem, ss::as_stream(stream)>>>(A, B, D, M, N, K, a_mn, b_mn, (flags >> 2) & 1,
                                             (flags >> 3) & 1, a_tmem);
  SS_CHECK_LAUNCH("umma_selftest_kernel");
  return SS_OK;
}

// kind 0 tf32 / 1 bf16, a_tmem (tf32 only): see umma_rate_kernel
extern "C" int ss_debug_umma_rate(int32_t kind, int32_t N, int32_t a_tmem, int32_t count,
                                  uint64_t* out_dev, void* stream) {
  const size_t smem = 128 * 64 * 4 + 128 * 128 * 2;
  auto k = ss::umma_rate_kernel;
  SS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<1, 128, smem, ss::as_stream(stream)>>>(kind, N, a_tmem, count,
                                             reinterpret_cast<unsigned long long*>(out_dev));
  SS_CHECK_LAUNCH("umma_rate_kernel");
  return SS_OK;
}
