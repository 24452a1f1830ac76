// PROBE (not built into the library): see DESIGN.md, "tried and reverted".
// K4b for up to 2^18 keys: the whole stable LSD radix sort in ONE kernel on a
// 16-CTA thread-block cluster (non-portable size), the keys' permutation held
// in distributed shared memory.
//
// The onesweep sort (binsort.cu) pays a decoupled look-back chain per 8-bit
// pass; at 250k depth keys that chain, not bandwidth, sets its ~11 us per
// pass.  Here CTA c of the cluster owns positions [c E, c E + E) (E = 16384)
// of the permutation.  Per pass: every warp ranks its 512 elements stably
// (match.any + per-warp digit counters, gathering each key from global memory
// by its index), the CTA publishes its per-digit totals in shared memory, a
// cluster barrier, every CTA reads the 16 histograms over DSMEM to get the
// global start of each digit and the counts of the CTAs before it, and the
// elements are stored straight into their destination CTA's other buffer
// (st.shared::cluster).  A second cluster barrier publishes the pass.  Four
// passes over the 32-bit keys, then the sorted keys and indices are written
// out -- the same (key, index) order as binsort_run.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ss {

namespace {
constexpr int kCsCtas = 16, kCsThreads = 1024, kCsWarps = kCsThreads / 32;
constexpr int kCsElems = 16384;               // per CTA
constexpr int kCsPerWarp = kCsElems / kCsWarps;  // 512, 16 steps of 32
constexpr int kCsSteps = kCsPerWarp / 32;
// dynamic smem: two permutation buffers + per-warp digit counters
constexpr size_t kCsSmem = (2 * kCsElems + kCsWarps * 256) * sizeof(uint32_t);

__device__ __forceinline__ uint32_t lanemask_lt_cs() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
}  // namespace

__global__ void __cluster_dims__(kCsCtas, 1, 1) __launch_bounds__(kCsThreads, 1)
    cluster_sort_kernel(int n, uint32_t* __restrict__ keys, uint32_t* __restrict__ order) {
  extern __shared__ __align__(16) uint32_t cs_smem[];
  __shared__ uint32_t s_hist[256], s_base[256], s_wsum[kCsWarps];
  cg::cluster_group cluster = cg::this_cluster();
  uint32_t* buf[2] = {cs_smem, cs_smem + kCsElems};
  uint32_t* wc = cs_smem + 2 * kCsElems;  // [warp][digit]
  const int c = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int base = c * kCsElems;
  for (int i = tid; i < kCsElems; i += kCsThreads) buf[0][i] = (uint32_t)(base + i);  // identity
  cluster.sync();
  int cur = 0;
  for (int pass = 0; pass < 4; ++pass) {
    const int sh = 8 * pass;
    for (int i = tid; i < kCsWarps * 256; i += kCsThreads) wc[i] = 0;
    __syncthreads();
    // ---- stable rank within the warp's contiguous 512 elements
    uint32_t dr[kCsSteps];  // digit | (rank within the warp << 9); 256 = no element
    const int w0 = warp * kCsPerWarp;
#pragma unroll
    for (int s = 0; s < kCsSteps; ++s) {
      const int j = w0 + s * 32 + lane;
      dr[s] = base + j < n ? (__ldg(keys + buf[cur][j]) >> sh) & 255u : 256u;
    }
#pragma unroll
    for (int s = 0; s < kCsSteps; ++s) {
      const uint32_t d = dr[s];
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (d < 256u && lane == leader) {
        old = wc[warp * 256 + d];
        wc[warp * 256 + d] = old + __popc(peers);
      }
      old = __shfl_sync(0xffffffffu, old, leader);
      dr[s] = d | ((old + __popc(peers & lanemask_lt_cs())) << 9);
      __syncwarp();
    }
    __syncthreads();
    // ---- per digit: exclusive prefix over the warps, the CTA's total
    if (tid < 256) {
      uint32_t run = 0;
      for (int w = 0; w < kCsWarps; ++w) {
        const uint32_t t = wc[w * 256 + tid];
        wc[w * 256 + tid] = run;
        run += t;
      }
      s_hist[tid] = run;
    }
    cluster.sync();  // every CTA's histogram is published
    // ---- global start of each digit, plus the counts of the CTAs before this one
    if (tid < 256) {
      uint32_t tot = 0, before = 0;
#pragma unroll
      for (int r = 0; r < kCsCtas; ++r) {
        const uint32_t h = *cluster.map_shared_rank(s_hist + tid, r);
        tot += h;
        if (r < c) before += h;
      }
      // exclusive scan of tot over the 256 digits (8 warps)
      uint32_t x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_wsum[warp] = x;
      s_base[tid] = x - tot + before;
    }
    __syncthreads();
    if (tid < 256) {
      uint32_t add = 0;
      for (int w = 0; w < warp; ++w) add += s_wsum[w];
      s_base[tid] += add;
    }
    __syncthreads();
    // ---- stores into the destination CTAs' other buffer
    const int nxt = cur ^ 1;
#pragma unroll
    for (int s = 0; s < kCsSteps; ++s) {
      const uint32_t d = dr[s] & 511u;
      if (d < 256u) {
        const uint32_t p = s_base[d] + wc[warp * 256 + d] + (dr[s] >> 9);
        uint32_t* dst = cluster.map_shared_rank(buf[nxt], (int)(p / kCsElems));
        dst[p % kCsElems] = buf[cur][w0 + s * 32 + lane];
      }
    }
    cluster.sync();  // the pass is complete everywhere (and s_hist may be reused)
    cur = nxt;
  }
  // ---- sorted keys into the spare buffer, then both out (every CTA has
  // finished gathering keys by index before any key is overwritten)
  uint32_t* kb = buf[cur ^ 1];
  for (int i = tid; i < kCsElems; i += kCsThreads)
    if (base + i < n) kb[i] = keys[buf[cur][i]];
  cluster.sync();
  for (int i = tid; i < kCsElems; i += kCsThreads)
    if (base + i < n) {
      order[base + i] = buf[cur][i];
      keys[base + i] = kb[i];
    }
}

// Whether n keys fit the cluster and a 16-CTA cluster of this kernel can run
// on the device (checked once); otherwise the caller uses the onesweep passes.
bool cluster_sort_ready(int64_t n) {
  static int state = 0;  // 0 unknown, 1 usable, -1 not available on this device
  if (n < 1 || n > (int64_t)kCsCtas * kCsElems) return false;
  if (state == 0) {
    state = -1;
    if (cudaFuncSetAttribute(cluster_sort_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed,
                             1) != cudaSuccess ||
        cudaFuncSetAttribute(cluster_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kCsSmem) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kCsCtas);
    cfg.blockDim = dim3(kCsThreads);
    cfg.dynamicSmemBytes = kCsSmem;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, (void*)cluster_sort_kernel, &cfg) !=
            cudaSuccess ||
        clusters < 1) {
      cudaGetLastError();
      return false;
    }
    state = 1;
  }
  return state > 0;
}

// keys[0..n) sorted in place, order = the permutation (identity input implied)
int cluster_sort_run(int64_t n, uint32_t* keys, int32_t* order, cudaStream_t st) {
  cluster_sort_kernel<<<kCsCtas, kCsThreads, kCsSmem, st>>>(
      (int)n, keys, reinterpret_cast<uint32_t*>(order));
  SS_CHECK_LAUNCH("cluster_sort_kernel");
  return SS_OK;
}

}  // namespace ss
