// Minimal sm_100a tcgen05 toolkit (inline PTX): TMEM allocation, UMMA shared-
// memory / instruction descriptors, kind::tf32 MMA, commit to mbarrier, TMEM
// loads.  Layout conventions (CUTLASS cute/atom/mma_traits_sm100.hpp):
//
//   A tile stored "K-major, no swizzle" for 32-bit elements: element (r, k) at
//     (r / 8) * SBO + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4      bytes
//   i.e. 8x16-byte core matrices, LBO = 128 (next core along K) and
//   SBO = 128 * ceil(cols / 4) (next group of 8 rows).  The same bytes read as
//   the MN-major operand of the transposed matrix with LBO and SBO swapped.
//
//   Accumulators: M = 128 -> row m in TMEM lane m; M = 64 -> rows 16w..16w+15
//   in lanes 32w..32w+15 (w = 0..3), column n at base column + n.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace ss {
namespace umma {

__device__ inline uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// tile geometry for a K-major 32-bit tile with `cols` columns (multiple of 4)
__host__ __device__ constexpr uint32_t tile_sbo(int cols) { return 128u * (uint32_t)(cols / 4); }
__host__ __device__ constexpr uint32_t tile_bytes(int rows, int cols) {
  return (uint32_t)(rows / 8) * tile_sbo(cols);
}
// byte offset of element (r, c) inside such a tile
__device__ __forceinline__ uint32_t tile_off(int r, int c, int cols) {
  return (uint32_t)(r >> 3) * tile_sbo(cols) + (uint32_t)(c >> 2) * 128u + (uint32_t)(r & 7) * 16u +
         (uint32_t)(c & 3) * 4u;
}

// shared-memory matrix descriptor, SWIZZLE_NONE, version 1 (sm_100)
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// K-major operand starting at column k0 (multiple of 8 for one MMA step)
__device__ __forceinline__ uint64_t desc_k(uint32_t tile, int cols, int k0, int row0 = 0) {
  return desc(tile + (uint32_t)(k0 >> 2) * 128u + (uint32_t)(row0 >> 3) * tile_sbo(cols), 128u,
              tile_sbo(cols));
}
// MN-major operand = transpose of a K-major tile: MN runs along the tile's
// columns (from column mn0), K along its rows (from row k0, multiple of 8)
__device__ __forceinline__ uint64_t desc_mn(uint32_t tile, int cols, int k0, int mn0 = 0) {
  return desc(tile + (uint32_t)(k0 >> 3) * tile_sbo(cols) + (uint32_t)(mn0 >> 2) * 128u,
              tile_sbo(cols), 128u);
}

// instruction descriptor: kind::tf32, fp32 accumulate
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                          // D format f32
         | (2u << 7) | (2u << 10)           // A, B format tf32
         | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16)
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// A operand read from TMEM ("TS" form): a_tmem addresses lane 0 of the A tile,
// row i in lane i, K element k in column k (32-bit), advanced by 8 columns per
// tf32 K step
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t a_tmem, uint64_t b,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}

// Warp-collective forms: the whole (converged) warp executes them with
// warp-uniform operands and one elected lane issues.  Keeping the issue in
// uniform control flow lets ptxas hold descriptors in uniform registers
// (no per-MMA R2UR).
__device__ __forceinline__ void mma_tf32_ts_elect(uint32_t tmem_d, uint32_t a_tmem, uint64_t b,
                                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_elect(uint64_t* mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
          smem_u32(mbar))
      : "memory");
}

__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  const uint32_t a = smem_u32(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  }
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// one warp allocates `cols` TMEM columns, address written to *dst (smem)
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_free(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}

// 32 lanes x 32 bits x 16 columns: thread i of the warp gets lane (base + i)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// 32 lanes x 32 bits x 16 columns store (thread i of the warp -> lane base + i);
// the caller issues tmem_st_wait() before the data is consumed
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- 16-bit operands (kind::f16 with bf16 inputs, fp32 accumulate)
//
// A 16-bit tile is stored with 8x8-element core matrices (8 rows x 16 bytes,
// 128 contiguous bytes): element (r, c) at
//   (r / 8) * SBO16 + (c / 8) * 128 + (r % 8) * 16 + (c % 8) * 2,  SBO16 = 16 * cols.
// K-major read (K along the columns): LBO = 128 (next core along K), SBO = SBO16.
// MN-major read of the same bytes (the transposed matrix, MN along the
// columns, K along the rows): SBO = 128 (next core along MN), LBO = SBO16
// (next 8 K-rows), cute/atom/mma_traits_sm100.hpp canonical INTERLEAVE forms.
__host__ __device__ constexpr uint32_t sbo16(int cols) { return 16u * (uint32_t)cols; }
__host__ __device__ constexpr uint32_t tile16_bytes(int rows, int cols) {
  return (uint32_t)(rows / 8) * sbo16(cols);
}
__device__ __forceinline__ uint32_t tile16_off(int r, int c, int cols) {
  return (uint32_t)(r >> 3) * sbo16(cols) + (uint32_t)(c >> 3) * 128u + (uint32_t)(r & 7) * 16u +
         (uint32_t)(c & 7) * 2u;
}
// K-major operand from column k0 (multiple of 16), rows from row0 (multiple of 8)
__device__ __forceinline__ uint64_t desc16_k(uint32_t tile, int cols, int k0, int row0 = 0) {
  return desc(tile + (uint32_t)(k0 >> 3) * 128u + (uint32_t)(row0 >> 3) * sbo16(cols), 128u,
              sbo16(cols));
}
// MN-major operand (transpose of the stored tile): K from row k0 (multiple of
// 16), MN from column mn0 (multiple of 8).  `swap` exchanges LBO/SBO (probe).
__device__ __forceinline__ uint64_t desc16_mn(uint32_t tile, int cols, int k0, int mn0 = 0,
                                              int swap = 0) {
  const uint32_t a = tile + (uint32_t)(k0 >> 3) * sbo16(cols) + (uint32_t)(mn0 >> 3) * 128u;
  return swap ? desc(a, 128u, sbo16(cols)) : desc(a, sbo16(cols), 128u);
}
// instruction descriptor: kind::f16 with bf16 A/B, fp32 accumulate
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                          // D format f32
         | (1u << 7) | (1u << 10)           // A, B format bf16
         | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16)
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// warp-collective form (see mma_tf32_ts_elect)
__device__ __forceinline__ void mma_bf16_elect(uint32_t tmem_d, uint64_t a, uint64_t b,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// ---- fp16 operands (kind::f16 with f16 A/B, fp32 accumulate): the decoder's
// fp16-weight mode.  In TMEM a 16-bit A operand packs two K elements per 32-bit
// column (element 2c in the low half of column c), so one K = 16 step spans 8
// columns, the same column stride as a tf32 K = 8 step.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                          // D format f32; A, B format f16 (0)
         | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16)
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16_ts_elect(uint32_t tmem_d, uint32_t a_tmem, uint64_t b,
                                                 uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}
// two floats -> one 32-bit column of f16 (a in the low half), round to nearest even
__device__ __forceinline__ uint32_t pack_f16(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ float round_f16(float x) { return __half2float(__float2half_rn(x)); }
__device__ __forceinline__ void tmem_st8u(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
__device__ __forceinline__ void tmem_st4u(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
               : "memory");
}

// x = hi + lo with hi = bf16(x) (round to nearest even), lo = bf16(x - hi):
// the 3-product split A_hi.B_hi + A_hi.B_lo + A_lo.B_hi keeps ~16 mantissa bits.
__device__ __forceinline__ void split_bf16(float x, uint16_t& hi, uint16_t& lo) {
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
  hi = __bfloat16_as_ushort(h);
  lo = __bfloat16_as_ushort(l);
}

// fp32 -> tf32 with round-to-nearest (kept in a 32-bit container)
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

}  // namespace umma
}  // namespace ss
