// Fused Stage-1 iteration (pipeline.py:262-277): one stream-ordered sequence
// apply_ntc -> rasterize_forward -> render_loss -> rasterize_backward ->
// apply_ntc_backward -> lazy Adam (+ view-space stats), with no host work in
// between except the tile-pair count readback that sizes the sort.
#include "common.cuh"

namespace ss {

static ss_cloud transformed(const ss_stage1* st) {
  ss_cloud c = st->src;
  c.means = st->t_means;
  c.rotations = st->t_rotations;
  c.sh = st->t_sh;
  return c;
}

// ViewspaceStats.add (adaptive.py:92-94).  The view's image gradient was scaled
// by grad_scale (1/B in a batch); the statistic is of the per-view gradient, so
// the norm is scaled back by inv_scale = 1/grad_scale.
__global__ void stats_kernel(int64_t n, const float* __restrict__ vs,
                             const uint8_t* __restrict__ contrib, float* __restrict__ norm,
                             int32_t* __restrict__ count, float inv_scale) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  norm[i] += vs[i] * inv_scale;
  count[i] += contrib[i];
}

// loss / pair-count histories at the device-side iteration index
// (+ the batch-loss sum of view-sharded training)
__global__ void history_kernel(const double* __restrict__ loss, const int64_t* __restrict__ pairs,
                               double* loss_hist, int64_t* pair_hist, int64_t len,
                               int32_t* __restrict__ iter_dev, float* loss_accum) {
  if (iter_dev) {
    const int64_t slot = len > 0 ? *iter_dev % len : 0;
    if (loss_hist) loss_hist[slot] = *loss;
    if (pair_hist) pair_hist[slot] = *pairs;
    *iter_dev += 1;
  }
  if (loss_accum) *loss_accum += (float)*loss;
}

__global__ void scale_kernel(int64_t n, float* __restrict__ v, float s) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] *= s;
}

// ntc_scratch = [X | dX | out7 | g7 | relu] (ntc_scratch(), ss_apply_ntc_backward_bytes)
static NtcScratch scratch_of(const ss_stage1* st) {
  return ntc_scratch(st->ntc_scratch, &st->mlp, st->n_in);
}

static int64_t n_table(const ss_stage1* st) {
  return (int64_t)st->grid.n_levels * ((int64_t)1 << st->grid.log2_table) * st->grid.n_features;
}

static int64_t n_params(const ss_stage1* st) {
  ss_mlp_layout L{};
  ss_mlp_get_layout(&st->mlp, &L);
  return L.total;
}

}  // namespace ss

using namespace ss;

extern "C" {

int ss_stage1_frame_begin(ss_stage1* st, void* stream) {
  cudaStream_t s = as_stream(stream);
  const int64_t n = st->src.n, K = st->src.sh_coeffs;
  const int64_t T = (int64_t)1 << st->grid.log2_table;
  SS_CUDA(cudaMemsetAsync(st->row_mask, 0, (size_t)st->grid.n_levels * T, s));
  SS_TRY(ss_ntc_touched(&st->grid, st->n_in, st->src.means, st->rows, st->row_mask, stream));
  SS_CUDA(cudaMemcpyAsync(st->t_means, st->src.means, n * 3 * sizeof(float),
                          cudaMemcpyDeviceToDevice, s));
  SS_CUDA(cudaMemcpyAsync(st->t_rotations, st->src.rotations, n * 4 * sizeof(float),
                          cudaMemcpyDeviceToDevice, s));
  SS_CUDA(cudaMemcpyAsync(st->t_sh, st->src.sh, n * K * 3 * sizeof(float),
                          cudaMemcpyDeviceToDevice, s));
  const int64_t nt = n_table(st), np = n_params(st);
  SS_CUDA(cudaMemsetAsync(st->g_tables, 0, nt * sizeof(float), s));
  SS_CUDA(cudaMemsetAsync(st->g_params, 0, np * sizeof(float), s));
  SS_CUDA(cudaMemsetAsync(st->m_tables, 0, nt * sizeof(double), s));
  SS_CUDA(cudaMemsetAsync(st->v_tables, 0, nt * sizeof(double), s));
  SS_CUDA(cudaMemsetAsync(st->m_params, 0, np * sizeof(double), s));
  SS_CUDA(cudaMemsetAsync(st->v_params, 0, np * sizeof(double), s));
  SS_CUDA(cudaMemsetAsync(st->step_dev, 0, sizeof(int32_t), s));
  if (st->stats_norm) SS_CUDA(cudaMemsetAsync(st->stats_norm, 0, n * sizeof(float), s));
  if (st->stats_count) SS_CUDA(cudaMemsetAsync(st->stats_count, 0, n * sizeof(int32_t), s));
  st->iteration = 0;
  if (st->iter_dev) SS_CUDA(cudaMemsetAsync(st->iter_dev, 0, sizeof(int32_t), s));
  return SS_OK;
}

int ss_stage1_iter_begin(ss_stage1* st, const ss_camera* cam, int64_t* counts_host,
                         void* stream) {
  const NtcScratch ns = scratch_of(st);
  cudaStream_t s = as_stream(stream);
  // every per-iteration scratch region zeroed by one kernel (common.cuh)
  SS_TRY(raster_zero_iteration(st->geom, st->src.n, cam, &st->settings, st->bins,
                               st->bin_capacity, st->loss_scratch, 2 * sizeof(double), s));
  PrezeroScope scope(true);
  SS_TRY(ntc_forward_run(&st->grid, &st->mlp, st->n_in, st->src.means, st->rows, st->tables,
                         st->params, ns.X, ns.xs, ns.out7, 8, ns.relu, st->status, s));
  const bool perm = st->rows_index && st->rows_pos;
  SS_TRY(transform_run(&st->src, st->n_in, perm ? st->rows_index : st->rows,
                       perm ? st->rows_pos : nullptr, ns.out7, 8, st->rotate_sh, st->t_means,
                       st->t_rotations, st->t_sh, st->status, s));
  const ss_cloud tc = transformed(st);
  return raster_begin(&tc, cam, &st->settings, st->geom, counts_host, as_stream(stream));
}

}  // extern "C"

namespace ss {
// One view's render, loss and raster backward into the transformed-cloud
// gradients d_means / d_rotations / d_sh (accumulate: added to them, the
// views of a batch), plus the loss history and the view-space statistics.
static int stage1_view(ss_stage1* st, const ss_camera* cam, const float* target, int64_t n_pairs,
                       float grad_scale, int accumulate, cudaStream_t s) {
  // the view's scratch was zeroed with its raster_begin (ss_stage1_iter_begin,
  // ss_stage1_batch_view)
  PrezeroScope scope(true);
  // n_pairs above the workspace: the host-known count selects binning in bands
  // of tile rows (synchronous); otherwise the device count drives one band
  const int64_t cap = st->bin_capacity;
  const ss_cloud tc = transformed(st);
  SS_TRY(raster_finish(&tc, cam, &st->settings, st->geom, st->bins, cap, st->image,
                       st->alpha_map, nullptr, st->status, 1, s, n_pairs));
  SS_TRY(ss_render_loss(st->image, target, cam->height, cam->width, 3, st->lambda_dssim,
                        st->ssim_c1, st->ssim_c2, st->loss_scratch, st->loss_dev, st->d_image,
                        st->status, s));
  const bool hist = st->iter_dev && st->history_len > 0;
  if (hist || st->loss_accum) {
    history_kernel<<<1, 1, 0, s>>>(st->loss_dev, raster_counts(st->geom, tc.n, cam, &st->settings) + 1,
                                   st->loss_history, st->pair_history, st->history_len,
                                   hist ? st->iter_dev : nullptr, st->loss_accum);
    SS_CHECK_LAUNCH("history_kernel");
  }
  if (!(grad_scale > 0.0f)) {
    set_error("grad_scale must be positive");
    return SS_ERR_DATA;
  }
  if (grad_scale != 1.0f) {
    const int64_t m = (int64_t)cam->width * cam->height * 3;
    scale_kernel<<<(unsigned)cdiv(m, 256), 256, 0, s>>>(m, st->d_image, grad_scale);
    SS_CHECK_LAUNCH("scale_kernel");
  }
  ss_cloud_grads gr{};
  gr.d_means = st->d_means;
  gr.d_rotations = st->d_rotations;
  gr.d_sh = st->d_sh;
  gr.viewspace = st->viewspace;
  gr.contributed = st->contributed;
  SS_TRY(raster_backward(&tc, cam, &st->settings, st->geom, st->bins, cap, st->d_image, &gr, 0,
                         s, n_pairs, 1, st->status, accumulate));
  if (st->accumulate_stats && st->stats_norm && st->stats_count) {
    const int64_t n = st->src.n;
    stats_kernel<<<(unsigned)cdiv(n, 256), 256, 0, s>>>(n, st->viewspace, st->contributed,
                                                         st->stats_norm, st->stats_count,
                                                         1.0f / grad_scale);
    SS_CHECK_LAUNCH("stats_kernel");
  }
  return SS_OK;
}

// transform VJP, decoder backward and (unless deferred) the table scatter of
// the transformed-cloud gradients; live: skip rows no pixel saw (one view)
static int stage1_ntc_grads(ss_stage1* st, const uint8_t* live, cudaStream_t s) {
  const NtcScratch ns = scratch_of(st);
  const bool perm = st->rows_index && st->rows_pos;
  SS_TRY(transform_vjp_run(&st->src, st->n_in, perm ? st->rows_index : st->rows,
                           perm ? st->rows_pos : nullptr, ns.out7, 8, st->rotate_sh, st->d_means,
                           st->d_rotations, st->d_sh, ns.g7, 8, s, live));
  return ntc_backward_run(&st->grid, &st->mlp, st->n_in, st->src.means, st->rows, st->params,
                          ns.X, ns.xs, ns.g7, 8, ns.relu, ns.dX,
                          st->defer_scatter ? nullptr : st->g_tables, st->g_params, s);
}
}  // namespace ss

extern "C" {

int ss_stage1_iter_grads(ss_stage1* st, const ss_camera* cam, const float* target,
                         int64_t n_pairs, float grad_scale, void* stream) {
  cudaStream_t s = as_stream(stream);
  SS_TRY(stage1_view(st, cam, target, n_pairs, grad_scale, 0, s));
  SS_TRY(stage1_ntc_grads(st, st->contributed, s));
  st->iteration += 1;
  return SS_OK;
}

int ss_stage1_batch_view(ss_stage1* st, const ss_camera* cam, const float* target,
                         float grad_scale, int32_t first, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (first) {
    SS_TRY(ss_stage1_iter_begin(st, cam, nullptr, stream));
  } else {  // the parameters have not moved: same transformed cloud
    const ss_cloud tc = transformed(st);
    SS_TRY(raster_zero_iteration(st->geom, st->src.n, cam, &st->settings, st->bins,
                                 st->bin_capacity, st->loss_scratch, 2 * sizeof(double), s));
    PrezeroScope scope(true);
    SS_TRY(raster_begin(&tc, cam, &st->settings, st->geom, nullptr, s));
  }
  SS_TRY(stage1_view(st, cam, target, 0, grad_scale, first ? 0 : 1, s));
  st->iteration += 1;
  return SS_OK;
}

int ss_stage1_batch_ntc_grads(ss_stage1* st, void* stream) {
  return stage1_ntc_grads(st, nullptr, as_stream(stream));
}

int ss_stage1_table_scatter(ss_stage1* st, void* stream) {
  const NtcScratch ns = scratch_of(st);
  return ntc_scatter_run(&st->grid, st->n_in, st->src.means, st->rows, ns.dX, ns.xs,
                         st->g_tables, as_stream(stream));
}

int ss_stage1_apply_adam(ss_stage1* st, void* stream) {
  return ss_adam_step(n_table(st), st->tables, st->g_tables, st->m_tables, st->v_tables,
                      st->row_mask, st->grid.n_features, n_params(st), st->params, st->g_params,
                      st->m_params, st->v_params, st->step_dev, st->lr, st->beta1, st->beta2,
                      st->eps, 1, stream);
}

int ss_stage1_iter_finish(ss_stage1* st, const ss_camera* cam, const float* target,
                          int64_t n_pairs, void* stream) {
  SS_TRY(ss_stage1_iter_grads(st, cam, target, n_pairs, 1.0f, stream));
  return ss_stage1_apply_adam(st, stream);
}

int ss_stage1_render(ss_stage1* st, const ss_camera* cam, void* stream) {
  SS_TRY(ss_stage1_iter_begin(st, cam, nullptr, stream));
  const ss_cloud tc = transformed(st);
  return raster_finish(&tc, cam, &st->settings, st->geom, st->bins, st->bin_capacity, st->image,
                       st->alpha_map, nullptr, st->status, 1, as_stream(stream), 0);
}

int ss_stage1_iter(ss_stage1* st, const ss_camera* cam, const float* target, float grad_scale,
                   int32_t apply_adam, void* stream) {
  SS_TRY(ss_stage1_iter_begin(st, cam, nullptr, stream));
  SS_TRY(ss_stage1_iter_grads(st, cam, target, 0, grad_scale, stream));
  return apply_adam ? ss_stage1_apply_adam(st, stream) : SS_OK;
}

}  // extern "C"
