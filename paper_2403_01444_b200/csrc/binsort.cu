// K4d: stable LSD radix sort of (tile key, depth rank) pairs whose count lives
// in device memory (rasterizer.py:155-175: per-tile member lists in depth
// order).  Because the pair count never has to reach the host, a whole
// Stage-1 iteration is stream-ordered without a synchronisation and can be
// captured in a CUDA graph; buffers are sized by a capacity bound and an
// overflow raises SS_FLAG_OVERFLOW on the device.
//
// Per 8-bit digit pass ("onesweep"): a CTA of 256 threads takes a logical
// tile id from an atomic ticket (so every predecessor is already running),
// ranks its tile of 256 x STEPS keys stably with warp match + per-warp digit
// counters (warp w owns the w-th eighth of the tile, in index order), publishes
// its per-digit counts and resolves its global offsets by decoupled look-back
// over the predecessors, stages the tile in shared memory in sorted order and
// writes it out in coalesced runs.  One histogram kernel serves all passes.
// Input order is the rank order the duplicate kernel emits, so LSD stability
// gives exactly the reference's (tile, rank) order.
#include "common.cuh"

namespace ss {

namespace {
constexpr int kBsThreads = 256;
constexpr int kBsWarps = kBsThreads / 32;
#ifndef SS_BS_STEPS_BIG
#define SS_BS_STEPS_BIG 12
#endif
#ifndef SS_BS_WIN
#define SS_BS_WIN 8
#endif
constexpr int kBsStepsBig = SS_BS_STEPS_BIG;  // items per lane (3072-item tiles: 8 / 12 / 16 measured 96 / 90 / 95 us on 3.3M tile pairs)
#ifndef SS_BS_STEPS_SMALL
#define SS_BS_STEPS_SMALL 8
#endif
constexpr int kBsStepsSmall = SS_BS_STEPS_SMALL;  // small sorts (e.g. the depth keys): 2048-item tiles measured best
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kCntMask = (1u << 30) - 1;
constexpr int kMaxPasses = 4;
constexpr int kWin = SS_BS_WIN;  // look-back window (predecessor flags read per round trip)

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
}  // namespace

BinSortWS binsort_plan(Carve& c, int64_t capacity, int max_passes) {
  BinSortWS w{};
  w.steps = capacity <= (int64_t)1 << 20 ? kBsStepsSmall : kBsStepsBig;
  const int64_t tile = (int64_t)kBsThreads * w.steps;
  w.max_blocks = (capacity + tile - 1) / tile;
  if (w.max_blocks < 1) w.max_blocks = 1;
  w.max_passes = max_passes;
  w.hist = c.take<uint32_t>(kMaxPasses * 256 + 64);  // [pass][digit], then tickets
  w.status = c.take<uint32_t>((size_t)max_passes * w.max_blocks * 256);
  return w;
}

static size_t binsort_clear_bytes(const BinSortWS&) {
  return (kMaxPasses * 256 + 64) * sizeof(uint32_t);
}

// one histogram kernel for all passes (8-bit digits; the last may be narrower)
__global__ void __launch_bounds__(256) bs_hist_kernel(const uint32_t* __restrict__ keys,
                                                      const int64_t* __restrict__ d_n,
                                                      int64_t cap, int key_bits,
                                                      uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[kMaxPasses][256];
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const int64_t n = min(*d_n, cap);
  const int passes = (key_bits + 7) / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    for (int p = 0; p < passes; ++p) {
      const int bits = min(8, key_bits - 8 * p);
      atomicAdd(&sh[p][(k >> (8 * p)) & ((1u << bits) - 1)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
    const uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

// pass over digit bits [shift, shift + bits); tiles of kBsThreads * STEPS items
template <int STEPS>
__global__ void __launch_bounds__(kBsThreads) bs_pass_kernel(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, const int64_t* __restrict__ d_n, int64_t cap, int shift, int bits,
    const uint32_t* __restrict__ hist, uint32_t* __restrict__ ticket, uint32_t* __restrict__ status) {
  __shared__ uint32_t s_bid;
  __shared__ uint32_t wh[kBsWarps][256];  // per-warp digit counts -> exclusive prefix over warps
  __shared__ uint32_t s_gbase[256];       // global position of this tile's first item of digit d
  __shared__ uint32_t s_lstart[256];      // tile-local start of digit d
  __shared__ uint32_t s_scan[256];
  constexpr int kBsSteps = STEPS, kBsTile = kBsThreads * STEPS;
  __shared__ uint32_t s_keys[kBsTile], s_vals[kBsTile];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // logical tile id from the ticket: every predecessor of a running CTA has
  // already been scheduled, whatever order the hardware dispatches blocks in
  if (tid == 0) s_bid = atomicAdd(ticket, 1u);
  for (int i = tid; i < kBsWarps * 256; i += kBsThreads) (&wh[0][0])[i] = 0;
  __syncthreads();
  const int64_t n = min(*d_n, cap);
  const uint32_t bid = s_bid;
  const int64_t base = (int64_t)bid * kBsTile;
  if (base >= n) return;  // block-uniform
  const uint32_t dmask = (1u << bits) - 1;
  // ---- load and rank (warp-contiguous segments, lane order within a step)
  uint32_t k[kBsSteps], v[kBsSteps], rk[kBsSteps];
  const int64_t wbase = base + warp * (kBsSteps * 32);
#pragma unroll
  for (int s = 0; s < kBsSteps; ++s) {  // all loads in flight before the ranking
    const int64_t i = wbase + s * 32 + lane;
    k[s] = i < n ? kin[i] : 0u;
    v[s] = i < n ? vin[i] : 0u;
  }
#pragma unroll
  for (int s = 0; s < kBsSteps; ++s) {
    const int64_t i = wbase + s * 32 + lane;
    const bool ok = i < n;
    const uint32_t d = ok ? ((k[s] >> shift) & dmask) : 256u;  // 256 = past the end
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (ok && lane == leader) {
      old = wh[warp][d];
      wh[warp][d] = old + __popc(peers);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rk[s] = old + __popc(peers & lanemask_lt());
    __syncwarp();
  }
  __syncthreads();
  // ---- per digit (thread = digit): counts -> exclusive prefix over warps
  const int d = tid;
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < kBsWarps; ++w) {
    const uint32_t t = wh[w][d];
    wh[w][d] = cnt;
    cnt += t;
  }
  // ---- decoupled look-back over the predecessors' per-digit counts
  uint32_t* my = status + (size_t)bid * 256 + d;
  uint32_t excl = 0;
  if (d >> bits) {
    // digit unused by a narrow pass (e.g. the 5-bit top pass of the tile key):
    // nothing to publish or look back for
  } else if (bid == 0) {
    atomicExch(my, kFlagInc | cnt);
  } else {
    atomicExch(my, kFlagAgg | cnt);
    // windowed look-back: kWin predecessors' flags in flight per round trip,
    // consumed nearest first up to the first inclusive prefix; a predecessor
    // that has not published yet is re-polled at the start of the next window
    int64_t p = (int64_t)bid - 1;
    bool done = false;
    while (!done) {
      uint32_t st[kWin];
#pragma unroll
      for (int j = 0; j < kWin; ++j)
        st[j] = p - j >= 0 ? ld_volatile(status + (size_t)(p - j) * 256 + d) : kFlagInc;
      int used = 0;
#pragma unroll
      for (int j = 0; j < kWin; ++j) {
        if (done || used < j) continue;  // stopped at an inclusive or unready flag
        if ((st[j] & ~kCntMask) == 0) continue;  // not published: re-poll from here
        excl += st[j] & kCntMask;
        used = j + 1;
        done = (st[j] & kFlagInc) != 0;
      }
      p -= used;
    }
    atomicExch(my, kFlagInc | (excl + cnt));
  }
  // ---- exclusive scans over digits (global digit offsets, tile-local starts):
  // warp shuffle scans, then the 8 warp totals
  const uint32_t h = hist[d];
  uint32_t sh = h, sl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t a = __shfl_up_sync(0xffffffffu, sh, off);
    const uint32_t b = __shfl_up_sync(0xffffffffu, sl, off);
    if (lane >= off) sh += a, sl += b;
  }
  if (lane == 31) {
    s_scan[warp] = sh;
    s_scan[32 + warp] = sl;
  }
  __syncthreads();
  uint32_t wh_ = 0, wl_ = 0;
#pragma unroll
  for (int w = 0; w < kBsWarps; ++w)
    if (w < warp) wh_ += s_scan[w], wl_ += s_scan[32 + w];
  const uint32_t g_excl = sh - h + wh_;
  const uint32_t l_excl = sl - cnt + wl_;
  s_lstart[d] = l_excl;
  s_gbase[d] = g_excl + excl;
  __syncthreads();
  // ---- stage in sorted order, then coalesced write-out
#pragma unroll
  for (int s = 0; s < kBsSteps; ++s) {
    const int64_t i = wbase + s * 32 + lane;
    if (i < n) {
      const uint32_t dd = (k[s] >> shift) & dmask;
      const uint32_t p = s_lstart[dd] + wh[warp][dd] + rk[s];
      s_keys[p] = k[s];
      s_vals[p] = v[s];
    }
  }
  __syncthreads();
  const int cnt_tile = (int)min((int64_t)kBsTile, n - base);
  for (int i = tid; i < cnt_tile; i += kBsThreads) {
    const uint32_t key = s_keys[i];
    const uint32_t dd = (key >> shift) & dmask;
    const uint32_t gp = s_gbase[dd] + (uint32_t)i - s_lstart[dd];
    kout[gp] = key;
    vout[gp] = s_vals[i];
  }
}

int binsort_passes(int key_bits) { return (key_bits + 7) / 8; }

// Sorts the (count *d_n, at most cap) pairs by the low `key_bits` (<= 32) bits
// into keys_out/vals_out, in ceil(key_bits / 8) passes ping-ponging with the
// tmp buffers.  The input must be in keys_out/vals_out for an even number of
// passes and in keys_tmp/vals_tmp for an odd one: see binsort_passes().
thread_local bool t_prezeroed = false;

int binsort_clear(const BinSortWS& w, int key_bits, cudaStream_t st) {
  if (t_prezeroed) return SS_OK;  // raster_zero_iteration did it
  const int passes = binsort_passes(key_bits);
  SS_CUDA(cudaMemsetAsync(w.hist, 0, binsort_clear_bytes(w), st));
  SS_CUDA(cudaMemsetAsync(w.status, 0, (size_t)passes * w.max_blocks * 256 * sizeof(uint32_t),
                          st));
  return SS_OK;
}

int binsort_run(const BinSortWS& w, uint32_t* keys_tmp, uint32_t* vals_tmp, uint32_t* keys_out,
                uint32_t* vals_out, const int64_t* d_n, int64_t cap, int key_bits,
                cudaStream_t st, bool hist_ready) {
  const int passes = binsort_passes(key_bits);
  if (key_bits < 1 || passes > w.max_passes) {
    set_error("binsort: key wider than the planned passes");
    return SS_ERR_DATA;
  }
  uint32_t *ka = (passes & 1) ? keys_tmp : keys_out, *va = (passes & 1) ? vals_tmp : vals_out;
  uint32_t *kb = (passes & 1) ? keys_out : keys_tmp, *vb = (passes & 1) ? vals_out : vals_tmp;
  if (!hist_ready) {  // otherwise the producer cleared and filled w.hist (bs_hist_add)
    SS_TRY(binsort_clear(w, key_bits, st));
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (sms <= 0) sms = 148;
    }
    const unsigned hgrid =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(cap, 256), 4 * sms));
    bs_hist_kernel<<<hgrid, 256, 0, st>>>(ka, d_n, cap, key_bits, w.hist);
    SS_CHECK_LAUNCH("bs_hist_kernel");
  }
  uint32_t* tickets = w.hist + kMaxPasses * 256;
  const unsigned grid = (unsigned)w.max_blocks;
  for (int p = 0; p < passes; ++p) {
    const int bits = std::min(8, key_bits - 8 * p);
    auto k = w.steps == kBsStepsSmall ? bs_pass_kernel<kBsStepsSmall> : bs_pass_kernel<kBsStepsBig>;
    k<<<grid, kBsThreads, 0, st>>>(ka, va, kb, vb, d_n, cap, 8 * p, bits, w.hist + 256 * p,
                                   tickets + p,
                                   w.status + (size_t)p * w.max_blocks * 256);
    SS_CHECK_LAUNCH("bs_pass_kernel");
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  return SS_OK;
}

}  // namespace ss
