// Library-level state: last-error string, launch telemetry, SH rotation
// constants, MLP layout.  See include/ss_b200.h for the ABI contract.
#include <mutex>
#include <vector>

#include "common.cuh"

namespace ss {

static thread_local std::string t_last_error;
std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { t_last_error = msg; }

cudaError_t smem_attr_once(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;  // (kernel, device)
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& d : done)
    if (d.first == kernel && d.second == dev) return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(kernel, dev);
  return e;
}

// Band-l basis values at a unit direction (degree-l part of sh_basis).
static void band_values(int l, const double d[3], double* out) {
  double b[16];
  sh_basis<double>(l, d[0], d[1], d[2], b);
  for (int m = 0; m < 2 * l + 1; ++m) out[m] = b[l * l + m];
}

// Gauss-Jordan inverse with partial pivoting; returns the inf-norm condition.
static double invert(int n, std::vector<double> a, std::vector<double>& inv) {
  double anorm = 0;
  for (int i = 0; i < n; ++i) {
    double r = 0;
    for (int j = 0; j < n; ++j) r += std::fabs(a[i * n + j]);
    anorm = std::max(anorm, r);
  }
  inv.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(a[r * n + c]) > std::fabs(a[p * n + c])) p = r;
    if (std::fabs(a[p * n + c]) < 1e-12) return 1e300;
    for (int j = 0; j < n; ++j) {
      std::swap(a[c * n + j], a[p * n + j]);
      std::swap(inv[c * n + j], inv[p * n + j]);
    }
    double d = a[c * n + c];
    for (int j = 0; j < n; ++j) {
      a[c * n + j] /= d;
      inv[c * n + j] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      double f = a[r * n + c];
      for (int j = 0; j < n; ++j) {
        a[r * n + j] -= f * a[c * n + j];
        inv[r * n + j] -= f * inv[c * n + j];
      }
    }
  }
  double inorm = 0;
  for (int i = 0; i < n; ++i) {
    double r = 0;
    for (int j = 0; j < n; ++j) r += std::fabs(inv[i * n + j]);
    inorm = std::max(inorm, r);
  }
  return anorm * inorm;
}

// Pick 2l+1 sample directions with a well-conditioned S_{km} = Y_m(d_k) and
// store S^{-1}: the band rotation is M = S^{-1} E, E_{kb} = Y_b(R^T d_k).
static void build_band(int l, float (*dirs)[3], float* sinv) {
  const int n = 2 * l + 1;
  uint64_t state = 0x9E3779B97F4A7C15ull * (l + 1);
  auto uni = [&]() {
    state = state * 6364136223846793005ull + 1442695040888963407ull;
    return ((state >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
  };
  double best = 1e300;
  std::vector<double> best_inv, best_dirs(n * 3);
  for (int trial = 0; trial < 400; ++trial) {
    std::vector<double> dd(n * 3), s(n * n), inv;
    for (int k = 0; k < n; ++k) {
      double v[3], nrm;
      do {
        v[0] = uni(), v[1] = uni(), v[2] = uni();
        nrm = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
      } while (nrm < 0.2 || nrm > 1.0);
      for (int j = 0; j < 3; ++j) dd[k * 3 + j] = v[j] / nrm;
      band_values(l, &dd[k * 3], &s[k * n]);
    }
    double cond = invert(n, s, inv);
    if (cond < best) {
      best = cond;
      best_inv = inv;
      best_dirs = dd;
    }
  }
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < 3; ++j) dirs[k][j] = (float)best_dirs[k * 3 + j];
  for (int i = 0; i < n * n; ++i) sinv[i] = (float)best_inv[i];
}

void build_shrot_host(ShRotConst* h) {
  build_band(2, h->dirs2, &h->binvT2[0][0]);
  build_band(3, h->dirs3, &h->binvT3[0][0]);
}

}  // namespace ss

extern "C" {

const char* ss_last_error(void) { return ss::t_last_error.c_str(); }
int32_t ss_version(void) { return 1; }

size_t ss_struct_size(int32_t which) {
  switch (which) {
    case 0: return sizeof(ss_grid);
    case 1: return sizeof(ss_mlp);
    case 2: return sizeof(ss_mlp_layout);
    case 3: return sizeof(ss_camera);
    case 4: return sizeof(ss_raster_settings);
    case 5: return sizeof(ss_cloud);
    case 6: return sizeof(ss_cloud_grads);
    case 7: return sizeof(ss_stage1);
    default: return 0;
  }
}
int64_t ss_launch_count(void) { return ss::g_launches.load(); }

int ss_mlp_get_layout(const ss_mlp* mlp, ss_mlp_layout* out) {
  if (!mlp || !out) return SS_ERR_DATA;
  if (mlp->in_dim < 1 || mlp->in_dim > 64 || mlp->hidden_dim < 1 || mlp->hidden_dim > 64 ||
      mlp->n_hidden < 1 || mlp->n_hidden > 2 || mlp->out_dim != 7 ||
      (mlp->precision != SS_MLP_FP32 && mlp->precision != SS_MLP_F16)) {
    ss::set_error("unsupported decoder (in<=64, hidden<=64, 1-2 hidden layers, 7 outputs, precision fp32|f16)");
    return SS_ERR_DATA;
  }
  ss_mlp_layout L{};
  L.in_pad = mlp->in_dim <= 16 ? 16 : (mlp->in_dim <= 32 ? 32 : 64);
  L.hidden_pad = 64;
  L.out_pad = 8;
  L.n_hidden = mlp->n_hidden;
  L.w0 = 0;
  L.b0 = (int64_t)L.in_pad * 64;
  L.w1 = L.b0 + 64;
  L.b1 = L.w1 + (L.n_hidden == 2 ? 64 * 64 : 0);
  L.w2 = L.b1 + (L.n_hidden == 2 ? 64 : 0);
  L.b2 = L.w2 + 64 * 8;
  L.total = L.b2 + 8;
  *out = L;
  return SS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- phase timing
namespace ss {
static bool g_prof = false;
static cudaEvent_t g_ev[2 * PH_COUNT];
static bool g_ev_ready = false, g_used[PH_COUNT];
static const char* kPhaseNames[PH_COUNT] = {
    "gather", "decoder_forward", "transform", "project", "depth_sort", "rank_scan",
    "duplicate", "tile_sort", "ranges", "blend_forward", "ssim_map", "ssim_grad",
    "blend_backward", "gaussian_backward", "transform_vjp", "decoder_backward", "scatter",
    "adam"};

// Inside a CUDA-graph capture the events become external event-record nodes,
// so a replayed graph re-records them and the phases can be timed in replay.
static void prof_record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else cudaEventRecord(e, s);
}
void prof_begin(int phase, cudaStream_t s) {
  if (!g_prof) return;
  if (!g_ev_ready) {
    for (auto& e : g_ev) cudaEventCreate(&e);
    g_ev_ready = true;
  }
  prof_record(g_ev[2 * phase], s);
}
void prof_end(int phase, cudaStream_t s) {
  if (!g_prof || !g_ev_ready) return;
  prof_record(g_ev[2 * phase + 1], s);
  g_used[phase] = true;
}
}  // namespace ss

extern "C" {
int ss_profile_enable(int32_t on) {
  ss::g_prof = on != 0;
  for (bool& u : ss::g_used) u = false;
  if (on && !ss::g_ev_ready) {  // created outside any capture
    for (auto& e : ss::g_ev) cudaEventCreate(&e);
    ss::g_ev_ready = true;
  }
  return SS_OK;
}
int32_t ss_profile_enabled(void) { return ss::g_prof ? 1 : 0; }
const char* ss_profile_name(int32_t phase) {
  return phase >= 0 && phase < ss::PH_COUNT ? ss::kPhaseNames[phase] : "";
}
/* ms of the last recorded instance of each phase (-1 if never recorded since
 * ss_profile_enable); synchronises on the recorded events. */
int32_t ss_profile_count(void) { return ss::PH_COUNT; }

int ss_profile_read(double* ms, int32_t n) {
  for (int p = 0; p < n && p < ss::PH_COUNT; ++p) {
    ms[p] = -1.0;
    if (!ss::g_used[p] || !ss::g_prof) continue;
    float t = 0.f;
    SS_CUDA(cudaEventSynchronize(ss::g_ev[2 * p + 1]));
    SS_CUDA(cudaEventElapsedTime(&t, ss::g_ev[2 * p], ss::g_ev[2 * p + 1]));
    ms[p] = t;  // (g_used stays set: graph replays re-record the same events)
  }
  return SS_OK;
}
}
