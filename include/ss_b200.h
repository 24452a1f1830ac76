/*
 * ss_b200.h -- C ABI of the B200-native 3DGStream Stage-1 hot path.
 *
 * Every entry point replaces one function of the reference package
 * `splatstream` (paths relative to /root/reference/pkg/src/splatstream/);
 * the citation is on each declaration.  Conventions:
 *   - plain pointers and sizes only; all device memory is CALLER-OWNED
 *     (the library allocates nothing persistent).  Data-dependent scratch is
 *     sized with the *_bytes queries first (CUB style).
 *   - every function is stream-ordered on the `stream` argument (a
 *     cudaStream_t passed as void*), never synchronises the device, and
 *     returns an ss_status.  Device-detected numerical failures (zero-norm
 *     quaternion, non-finite loss) are OR-ed into a caller-provided device
 *     status word and mapped to NumericalError by the host.
 *   - float32 storage; float64 wherever bit-exactness with the float64
 *     reference needs it (hash positions, depth keys, tile rectangles).
 */
#ifndef SS_B200_H
#define SS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_MAX_LEVELS 32
#define SS_MAX_SH 16

/* status codes (errors.py:8-21; CLI exit-code mapping cli.py:40-43) */
typedef enum {
  SS_OK = 0,
  SS_ERR_DATA = 1,      /* DataError: bad shape/argument, point outside the AABB */
  SS_ERR_NUMERICAL = 2, /* NumericalError: zero-norm quaternion, non-finite loss */
  SS_ERR_CUDA = 3,      /* CUDA launch / runtime failure */
  SS_ERR_CAPACITY = 4   /* caller workspace too small: query *_bytes and retry */
} ss_status;

/* device status-word bits */
#define SS_FLAG_ZERO_QUAT 1u   /* |d_q| < 1e-12 (gaussians.py:46-47) */
#define SS_FLAG_NONFINITE 2u   /* check_finite("stage1 loss") (errors.py:24-29) */
#define SS_FLAG_OUTSIDE 4u     /* encode(): point outside the AABB (ntc.py:166-168) */
#define SS_FLAG_OVERFLOW 8u    /* tile-pair count exceeded the capacity */

/* HashGridConfig (ntc.py:30-61).  resolution[] = floor(base*growth^l) is
 * computed on the host in float64 with the reference formula (ntc.py:54-55). */
typedef struct ss_grid {
  int32_t n_levels, n_features, log2_table, reserved;
  int32_t resolution[SS_MAX_LEVELS];
  double aabb_min[3], aabb_max[3];
} ss_grid;

/* NeuralTransformationCache decoder (ntc.py:102-128): in -> hidden^n_hidden -> 7,
 * ReLU hidden layers.  Supported: in_dim <= 64, hidden_dim <= 64, n_hidden 1|2,
 * out_dim 7. */
/* precision: SS_MLP_FP32 -- fp32-accurate decoder (3xTF32 forward, bf16x3
 * backward on tensor cores); SS_MLP_F16 -- fp16 weights, biases and
 * activations with fp32 accumulation (BASELINE config 1's "fp16 MLP weights";
 * the reference itself is float64 throughout, ntc.py:241-276). */
#define SS_MLP_FP32 0
#define SS_MLP_F16 1
typedef struct ss_mlp {
  int32_t in_dim, hidden_dim, n_hidden, out_dim;
  int32_t precision;
} ss_mlp;

/* Device parameter layout: one packed fp32 vector W0 | b0 | [W1 | b1] | W2 | b2,
 * weights (fan_in, fan_out) row-major as in the reference (ntc.py:111), zero-
 * padded to in_pad (16|32|64) x 64 hidden x 8 outputs.  Zero padding is exact:
 * padded units stay 0 and receive exactly zero gradient, so Adam keeps them 0. */
typedef struct ss_mlp_layout {
  int32_t in_pad, hidden_pad, out_pad, n_hidden;
  int64_t w0, b0, w1, b1, w2, b2, total;
} ss_mlp_layout;
int ss_mlp_get_layout(const ss_mlp* mlp, ss_mlp_layout* out);

/* Camera (cameras.py:30-80): world_to_camera row-major 4x4. */
typedef struct ss_camera {
  double w2c[16];
  double fx, fy, cx, cy, near_clip;
  int32_t width, height;
} ss_camera;

/* RasterSettings (rasterizer.py:33-38) + the background colour argument. */
typedef struct ss_raster_settings {
  int32_t tile_size, reserved;
  double alpha_clamp, skip_alpha, stop_transmittance;
  double background[3];
} ss_raster_settings;

/* GaussianCloud, SoA fp32 (gaussians.py:179-216); sh is (n, sh_coeffs, 3). */
typedef struct ss_cloud {
  int64_t n;
  int32_t sh_coeffs, reserved;
  const float* means;
  const float* rotations;
  const float* log_scales;
  const float* opacity_logits;
  const float* sh;
} ss_cloud;

/* GradientBuffer (rasterizer.py:48-68).  Any pointer may be NULL to skip it. */
typedef struct ss_cloud_grads {
  float* d_means;          /* (n,3) */
  float* d_rotations;      /* (n,4) */
  float* d_log_scales;     /* (n,3) */
  float* d_opacity_logits; /* (n,)  */
  float* d_sh;             /* (n,K,3) */
  float* viewspace;        /* (n,) |dL/d mean2d| */
  uint8_t* contributed;    /* (n,) */
} ss_cloud_grads;

/* ------------------------------------------------------------------ */
/* library                                                             */
/* ------------------------------------------------------------------ */
const char* ss_last_error(void);
int32_t ss_version(void);
/* sizeof of the ABI structs (0 grid, 1 mlp, 2 mlp_layout, 3 camera, 4 settings,
 * 5 cloud, 6 cloud_grads, 7 stage1) so bindings can verify their layout */
size_t ss_struct_size(int32_t which);
/* number of kernel launches issued by this library since load (telemetry) */
int64_t ss_launch_count(void);
/* Phase timing: when enabled, CUDA events are recorded on the launching
 * stream around each hot-path phase (as event-record nodes when the stream is
 * being captured into a CUDA graph, so replays re-record them);
 * ss_profile_read returns the ms of the last instance of each phase (-1 when
 * never recorded since ss_profile_enable). */
int ss_profile_enable(int32_t on);
int32_t ss_profile_enabled(void);
int32_t ss_profile_count(void);
const char* ss_profile_name(int32_t phase);
int ss_profile_read(double* ms, int32_t n);

/* ------------------------------------------------------------------ */
/* NTC: hash-grid encode / decoder / lazy Adam   (ntc.py, optim.py)    */
/* ------------------------------------------------------------------ */
/* NeuralTransformationCache.encode (ntc.py:161-203): corner rows (n,L,8) int32
 * and trilinear weights (n,L,8) f32; float64 position math. */
int ss_ntc_encode(const ss_grid* grid, int64_t n, const float* means, int32_t* corner_idx,
                  float* corner_w, uint32_t* status, void* stream);

/* per-level touched-row mask (the EncodeContext.touched sets, ntc.py:187),
 * mask is (L, T) bytes, OR-ed (caller zeroes it). */
int ss_ntc_touched(const ss_grid* grid, int64_t n, const float* means, const int32_t* rows,
                   uint8_t* mask, void* stream);

/* NeuralTransformationCache.forward (ntc.py:219-248): out7 (n,7) = [d_mu | d_q];
 * feats (n, L*F) = the interpolated features (gather_features, ntc.py:205-216),
 * nullable. */
int ss_ntc_forward(const ss_grid* grid, const ss_mlp* mlp, int64_t n, const float* means,
                   const int32_t* rows, const float* tables, const float* params, float* out7,
                   float* feats, void* stream);

/* NeuralTransformationCache.backward (ntc.py:250-288).  Accumulates (+=) into
 * g_tables (L,T,F) and g_params; caller zeroes them.  `scratch` must hold
 * ss_ntc_backward_bytes(mlp) bytes. */
size_t ss_ntc_backward_bytes(const ss_mlp* mlp);
int ss_ntc_backward(const ss_grid* grid, const ss_mlp* mlp, int64_t n, const float* means,
                    const int32_t* rows, const float* tables, const float* params,
                    const float* g_out7, float* g_tables, float* g_params, void* scratch,
                    void* stream);

/* Adam.step (optim.py:33-66) via cache.adam_step (ntc.py:290-293):
 * lazy rows for the tables (row_mask (L*T) bytes, row width F), dense for the
 * MLP.  `step_dev` is a device int32 step counter incremented by this call
 * (bias correction uses the global step, optim.py:52-54).  Moments are kept in
 * float64 like the reference (eps = 1e-15 makes tiny gradients matter, D10).
 * Zeroes the grads
 * after use when zero_grads != 0. */
int ss_adam_step(int64_t n_table, float* tables, float* g_tables, double* m_tables,
                 double* v_tables, const uint8_t* row_mask, int32_t row_width,
                 int64_t n_params, float* params, float* g_params, double* m_params,
                 double* v_params, int32_t* step_dev, double lr, double beta1, double beta2,
                 double eps, int32_t zero_grads, void* stream);

/* ------------------------------------------------------------------ */
/* NTC transform (transform.py)                                        */
/* ------------------------------------------------------------------ */
/* apply_ntc (transform.py:53-96) fused with the NTC forward: for the `n_in`
 * Gaussians listed in `rows` (the inside-AABB set) writes means/rotations/sh
 * of `out` (other rows untouched: caller pre-copies the source cloud). */
int ss_apply_ntc(const ss_grid* grid, const ss_mlp* mlp, const ss_cloud* src, int64_t n_in,
                 const int32_t* rows, const float* tables, const float* params,
                 int32_t rotate_sh, float* out_means, float* out_rotations, float* out_sh,
                 float* out7, uint32_t* status, void* stream);

/* apply_ntc_backward (transform.py:99-135) chained with the NTC backward
 * (ntc.py:250-288): gradients on the transformed cloud -> += g_tables, g_params.
 * scratch: ss_apply_ntc_backward_bytes(n_in) bytes (the decoder output is
 * recomputed there). */
size_t ss_apply_ntc_backward_bytes(int64_t n_in);
int ss_apply_ntc_backward(const ss_grid* grid, const ss_mlp* mlp, const ss_cloud* src,
                          int64_t n_in, const int32_t* rows, const float* tables,
                          const float* params, int32_t rotate_sh, const float* d_means,
                          const float* d_rotations, const float* d_sh, float* g_tables,
                          float* g_params, void* scratch, void* stream);

/* The transform alone, for caches that are not this library's NTC (duck-typed
 * caches such as the reference's test stubs, test_transform.py:24-46):
 * apply given out7 = [d_mu | d_q] (transform.py:70-84) ... */
int ss_transform_apply(const ss_cloud* src, int64_t n_in, const int32_t* rows, const float* out7,
                       int32_t rotate_sh, float* out_means, float* out_rotations, float* out_sh,
                       uint32_t* status, void* stream);
/* ... and its vector-Jacobian product g_out7 (transform.py:111-134). */
int ss_transform_vjp(const ss_cloud* src, int64_t n_in, const int32_t* rows, const float* out7,
                     int32_t rotate_sh, const float* d_means, const float* d_rotations,
                     const float* d_sh, float* g_out7, void* stream);

/* ------------------------------------------------------------------ */
/* rasterizer (rasterizer.py)                                          */
/* ------------------------------------------------------------------ */
/* Workspace of a render, in two parts:
 *   geom: per-Gaussian / per-pixel buffers, ss_raster_geom_bytes(n, cam, settings)
 *   bins: per tile-pair buffers,            ss_raster_bin_bytes(n_pairs, cam, settings)
 * The same workspace pointers must be passed to the backward call. */
size_t ss_raster_geom_bytes(int64_t n, const ss_camera* cam, const ss_raster_settings* s);
size_t ss_raster_bin_bytes(int64_t n_pairs, int64_t n, const ss_camera* cam,
                           const ss_raster_settings* s);

/* rasterize_forward phase 1 (rasterizer.py:227-261 up to the tile counts):
 * projection + SH colour (fp64), stable depth sort, per-splat tile rectangles
 * and their prefix sum.  Writes [n_survivors, n_pairs] to `counts_host`
 * (pinned host int64[2]) asynchronously: synchronise `stream` before reading. */
int ss_raster_forward_begin(const ss_cloud* cloud, const ss_camera* cam,
                            const ss_raster_settings* s, void* geom, int64_t* counts_host,
                            void* stream);

/* rasterize_forward phase 2 (tile_bin rasterizer.py:107-175 + blending
 * :178-211, :264-281): key duplication, stable tile sort, tile ranges, tile
 * blend.  image (H,W,3) f32, alpha_map (H,W) f32, touch (n,) int32 (nullable). */
int ss_raster_forward_finish(const ss_cloud* cloud, const ss_camera* cam,
                             const ss_raster_settings* s, void* geom, void* bins,
                             int64_t n_pairs, float* image, float* alpha_map, int32_t* touch,
                             void* stream);

/* The same two calls for views whose pairs exceed the bin workspace (configs
 * with billions of tile pairs): the bins hold bin_capacity pairs
 * (ss_raster_bin_bytes(bin_capacity, ...)) and n_pairs is the view's count from
 * ss_raster_forward_begin; above the capacity the view is binned and blended
 * in bands of tile rows, each at most bin_capacity pairs (synchronises the
 * stream once per call to plan the bands; the backward bins each band again). */
int ss_raster_forward_finish_banded(const ss_cloud* cloud, const ss_camera* cam,
                                    const ss_raster_settings* s, void* geom, void* bins,
                                    int64_t bin_capacity, int64_t n_pairs, float* image,
                                    float* alpha_map, int32_t* touch, void* stream);
int ss_raster_backward_banded(const ss_cloud* cloud, const ss_camera* cam,
                              const ss_raster_settings* s, void* geom, void* bins,
                              int64_t bin_capacity, int64_t n_pairs, const float* d_image,
                              const ss_cloud_grads* grads, void* stream);

/* rasterize_backward (rasterizer.py:284-402).  Output arrays are written for
 * survivors only: caller zeroes them.  opacity_and_scales=0 skips
 * d_opacity_logits / d_log_scales work (Stage 1 consumes neither). */
int ss_raster_backward(const ss_cloud* cloud, const ss_camera* cam, const ss_raster_settings* s,
                       void* geom, void* bins, int64_t n_pairs, const float* d_image,
                       const ss_cloud_grads* grads, void* stream);

/* Tile lists of the last forward (rasterizer.py:107-175 output): per tile
 * [start,end) into the sorted pair array, and the sorted members (depth ranks,
 * exactly the reference's `members`) and the survivor order (`indices`). */
int ss_raster_tile_lists(const ss_camera* cam, const ss_raster_settings* s, const void* geom,
                         const void* bins, int64_t n_pairs, int64_t n, int32_t* tile_ranges,
                         int32_t* members, int32_t* indices, void* stream);

/* tile_bin (rasterizer.py:107-175) on precomputed projections: mean2d (n,2),
 * cov2d (n,2,2) and opacity (n,) float64, already in depth order.  Phase 1
 * writes [n, n_pairs] to counts_host; phase 2 fills the tile lists exactly
 * like ss_raster_tile_lists.  `geom` sized by ss_raster_geom_bytes. */
int ss_tile_bin_begin(int64_t n, const double* mean2d, const double* cov2d, const double* opacity,
                      const ss_camera* cam, const ss_raster_settings* s, void* geom,
                      int64_t* counts_host, void* stream);
int ss_tile_bin_finish(int64_t n, const ss_camera* cam, const ss_raster_settings* s, void* geom,
                       void* bins, int64_t n_pairs, int32_t* tile_ranges, int32_t* members,
                       void* stream);

/* ------------------------------------------------------------------ */
/* loss (losses.py)                                                    */
/* ------------------------------------------------------------------ */
/* render_loss (losses.py:84-148): (1-lam) L1 + lam (1-SSIM)/2 over valid
 * 11x11 windows, gradient d_image; images (H, W, channels) interleaved, 1-4 channels.  loss_dev: device double[1] (written).
 * scratch: ss_loss_bytes(h, w) bytes. */
size_t ss_loss_bytes(int32_t height, int32_t width, int32_t channels);
int ss_render_loss(const float* image, const float* target, int32_t height, int32_t width,
                   int32_t channels, double lam, double c1, double c2, void* scratch,
                   double* loss_dev, float* d_image, uint32_t* status, void* stream);

/* NTC warm-up (ntc.py:296-333, losses.py:151-180): one Adam
 * step of warmup_train on a device batch of n points (n, 3) fp32: touched rows
 * of the batch, decoder forward, identity-pull loss (the batch SUM of the
 * per-row terms lands in *loss_sum; the reference's loss is *loss_sum / n),
 * decoder backward + table scatter, lazy Adam (beta 0.9/0.999, eps 1e-15).
 * scratch: ss_ntc_warmup_bytes(n) bytes. */
size_t ss_ntc_warmup_bytes(int64_t n);
int ss_ntc_warmup_step(const ss_grid* grid, const ss_mlp* mlp, int64_t n, const float* batch,
                       float* tables, float* params, float* g_tables, float* g_params,
                       double* m_tables, double* v_tables, double* m_params, double* v_params,
                       uint8_t* row_mask, int32_t* step_dev, double lr, void* scratch,
                       double* loss_sum, uint32_t* status, void* stream);

/* ------------------------------------------------------------------ */
/* fused Stage-1 iteration (pipeline.py:262-277)                       */
/* ------------------------------------------------------------------ */
typedef struct ss_stage1 {
  /* configuration */
  ss_grid grid;
  ss_mlp mlp;
  ss_raster_settings settings;
  double lr, beta1, beta2, eps, lambda_dssim;
  int32_t rotate_sh, accumulate_stats;
  /* source (frozen previous-frame) cloud and its inside-AABB rows */
  ss_cloud src;
  int64_t n_in;
  const int32_t* rows;       /* inside rows in the order the NTC kernels use (e.g. Morton) */
  const int32_t* rows_index; /* optional: the inside rows in index order ... */
  const int32_t* rows_pos;   /* ... and the position of each in `rows` (coalesced transform) */
  /* NTC parameters, Adam state, gradients (caller-owned) */
  float *tables, *params, *g_tables, *g_params;
  double *m_tables, *v_tables, *m_params, *v_params;
  uint8_t* row_mask;
  int32_t* step_dev;
  /* transformed cloud (means/rotations/sh; scales/opacities shared with src) */
  float *t_means, *t_rotations, *t_sh;
  /* per-view render buffers */
  float *image, *alpha_map, *d_image;
  float *d_means, *d_rotations, *d_sh; /* transformed-cloud grads (n) */
  float* viewspace;
  uint8_t* contributed;
  float* stats_norm;      /* ViewspaceStats.norm_accum (adaptive.py:79-97), (n,) */
  int32_t* stats_count;   /* ViewspaceStats.view_count, (n,) */
  double* loss_dev;       /* last loss */
  double* loss_history;   /* optional (nullable): loss of iteration i at [i] */
  int64_t* pair_history;  /* optional (nullable): tile pairs of iteration i at [i] */
  int64_t history_len;    /* entries of the histories (iteration i -> [i % history_len]) */
  int32_t iteration;      /* host-side count of enqueued iterations */
  int32_t* iter_dev;      /* device-side iteration count: indexes the histories, so a
                             captured CUDA graph of an iteration stays correct on replay */
  uint32_t* status;
  void *geom, *bins, *loss_scratch, *ntc_scratch;
  int64_t bin_capacity; /* n_pairs the `bins` workspace holds; more raises
                           SS_FLAG_OVERFLOW in *status (the pairs beyond are dropped) */
  double ssim_c1, ssim_c2; /* LossConfig.ssim_c1 / ssim_c2 (losses.py:21-33); the window is
                              the reference default 11x11, sigma 1.5 */
  float* loss_accum;       /* nullable: every iteration adds its (unscaled) loss here, the
                              batch-loss sum of view-sharded training */
  int32_t defer_scatter;   /* != 0: ss_stage1_iter_grads stops after the decoder backward
                              (g_params final, dX in ntc_scratch); ss_stage1_table_scatter
                              then adds the table gradient (lets the caller start the
                              g_params all-reduce while the scatter runs) */
  int32_t reserved2;
} ss_stage1;

/* Start of a frame: touched-row mask, transformed <- source copy, zero Adam
 * state and gradients, step = 0 (clone_cache + reset_adam, pipeline.py:213-219). */
int ss_stage1_frame_begin(ss_stage1* st, void* stream);
/* Iteration part A: apply_ntc + projection/depth sort/tile counts.
 * counts_host (pinned int64[2]) receives [n_survivors, n_pairs]. */
int ss_stage1_iter_begin(ss_stage1* st, const ss_camera* cam, int64_t* counts_host, void* stream);
/* Iteration part B: binning, blend, loss, raster backward, transform+NTC
 * backward, lazy Adam, view-space stats.  The binning reads the pair count
 * from the device; n_pairs (>= 0) only asserts n_pairs <= bin_capacity. */
int ss_stage1_iter_finish(ss_stage1* st, const ss_camera* cam, const float* target,
                          int64_t n_pairs, void* stream);
/* Part B up to (and including) the NTC gradients but without the Adam step
 * (view-sharded data parallelism all-reduces g_tables/g_params in between).
 * n_pairs > bin_capacity (the count from part A): binned in bands of tile rows. */
int ss_stage1_iter_grads(ss_stage1* st, const ss_camera* cam, const float* target,
                         int64_t n_pairs, float grad_scale, void* stream);
int ss_stage1_apply_adam(ss_stage1* st, void* stream);
/* A batch of views sharing one parameter state (view-sharded training, the
 * mean of per-view gradients before one Adam step, transform.py:99-135 is
 * linear in the transformed-cloud gradients): ss_stage1_batch_view renders one
 * view and adds its transformed-cloud gradient (first != 0: also the NTC
 * forward + transform, and the gradients are overwritten instead of added);
 * ss_stage1_batch_ntc_grads then runs the transform VJP, decoder backward and
 * table scatter (unless defer_scatter) once for the whole batch.  Device pair
 * count (graph capturable). */
int ss_stage1_batch_view(ss_stage1* st, const ss_camera* cam, const float* target,
                         float grad_scale, int32_t first, void* stream);
int ss_stage1_batch_ntc_grads(ss_stage1* st, void* stream);
/* The hash-table scatter (ntc.py:278-288) of the last ss_stage1_iter_grads call
 * made with defer_scatter != 0: g_tables += the corner-weighted feature gradient. */
int ss_stage1_table_scatter(ss_stage1* st, void* stream);
/* One whole iteration (parts A and B, plus Adam when apply_adam != 0) with no
 * host synchronisation: the pair count stays on the device and the binning
 * is bounded by bin_capacity (overflow -> SS_FLAG_OVERFLOW).  Stream-ordered,
 * so consecutive iterations queue back to back (and can be graph-captured). */
int ss_stage1_iter(ss_stage1* st, const ss_camera* cam, const float* target, float grad_scale,
                   int32_t apply_adam, void* stream);
/* Forward only (render-only throughput, playback): apply_ntc + rasterize_forward
 * into st->image / st->alpha_map, with no host synchronisation. */
int ss_stage1_render(ss_stage1* st, const ss_camera* cam, void* stream);

/* device self-test of the tcgen05 building blocks: D (M x N) = opA . opB over
 * K, flags bit0/bit1 = A/B given transposed (MN-major operand), row-major fp32
 * device buffers (test infrastructure for the decoder kernels) */
/* decoder arithmetic: 0 = fp32 FFMA, 1 = tcgen05 3xTF32 (fp32-accurate, default),
 * 2 = tcgen05 tf32 */
int ss_set_mlp_mode(int32_t mode);
int32_t ss_get_mlp_mode(void);
// Debug: clock64 stamps of CTA 0 / thread 0 at the decoder kernels' stage
// boundaries (out: 2 x 64 uint64, forward then backward).
int ss_debug_mlp_trace(uint64_t* out);
/* Decoder-forward event clocks of CTA 0 (debug): out[0..127] epilogue thread 0
   (TMEM stores published / MMA completion seen), out[128..255] MMA lane
   (operands ready seen / MMAs committed). */
int ss_debug_mlp_events(uint64_t* out);
/* Debug: cycles of `count` back-to-back M = 128 tcgen05 MMAs (kind 0 tf32, 1 bf16;
   a_tmem: tf32 A operand from TMEM); out_dev[0] total incl. completion, [1] issue. */
int ss_debug_umma_rate(int32_t kind, int32_t N, int32_t a_tmem, int32_t count, uint64_t* out_dev,
                       void* stream);

int ss_selftest_umma(int32_t M, int32_t N, int32_t K, int32_t flags, const float* A,
                     const float* B, float* D, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SS_B200_H */
