// C ABI entry points (include/sigkit_b200.h): validation, launch geometry,
// batch chunking of the backward workspace.
#include <algorithm>
#include <atomic>
#include <cstdio>

#include "sigb_internal.h"
#include "sigb_level.cu"

namespace sigb {

static thread_local std::string g_last_error;
int g_policy = 0;
int g_tensor_cores = 1;
static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches += n; }

// -- optional event timing of the main kernels ---------------------------------------
namespace {
struct TimerSlot {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;  // one pair per launch since the last reset
  size_t used = 0;
};
bool g_timing = false;
TimerSlot g_slots[2];
}  // namespace

void timing_begin(int which, cudaStream_t stream) {
  if (!g_timing) return;
  TimerSlot& t = g_slots[which];
  if (t.used == t.ev.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    t.ev.emplace_back(a, b);
  }
  cudaEventRecord(t.ev[t.used].first, stream);
}

void timing_end(int which, cudaStream_t stream) {
  if (!g_timing) return;
  TimerSlot& t = g_slots[which];
  cudaEventRecord(t.ev[t.used].second, stream);
  ++t.used;
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
  return SIGB_ERR_CUDA;
}

namespace {

constexpr int kThreads = 256;
// Workspace budget per backward chunk (partials + checkpoints).
constexpr size_t kWorkspaceBudget = size_t(2) << 30;

template <typename T>
size_t smem_bytes(const sigb_plan* p, bool backward) {
  size_t mx = 0;
  for (const PartDesc& pd : p->h_parts) {
    SmemLayout l = smem_layout((int)p->d, p->max_len, pd.n, pd.tv_size, pd.tb_size, backward);
    mx = std::max(mx, (size_t)l.total * sizeof(T));
  }
  return mx;
}

int check_smem(size_t bytes) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (bytes > (size_t)optin)
    return fail(SIGB_ERR_UNSUPPORTED, "word-set part needs " + std::to_string(bytes) +
                                          " B of shared memory (device limit " + std::to_string(optin) + ")");
  return SIGB_OK;
}

template <typename T>
int forward_t(const sigb_plan* p, const void* X, int64_t B, int64_t L, const int64_t* bounds, int64_t K,
              void* out, int64_t out_ld, int64_t out_col0, int include_empty, void* state, T* ckpt,
              int64_t stride, int64_t nck, cudaStream_t stream) {
  const size_t smem = smem_bytes<T>(p, false);
  int rc = check_smem(smem);
  if (rc) return rc;
  SIGB_CUDA_TRY(cudaFuncSetAttribute(forward_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t grid = B * K * p->num_parts;
  if (grid == 0) return SIGB_OK;
  count_launch();
  if (!ckpt) timing_begin(0, stream);
  forward_kernel<T><<<(unsigned)grid, kThreads, smem, stream>>>(
      p->dev(), (const T*)X, L, bounds, K, (T*)out, out_ld, out_col0, include_empty, (T*)state, p->Wc, ckpt,
      stride, nck, p->max_n);
  if (!ckpt) timing_end(0, stream);
  SIGB_CUDA_TRY(cudaGetLastError());
  return SIGB_OK;
}

struct BwdGeometry {
  int64_t chunk;        // paths per chunk
  size_t partial_bytes;  // per chunk
  size_t ckpt_bytes;     // per chunk
  int64_t nck;
};

template <typename T>
BwdGeometry bwd_geometry(const sigb_plan* p, int64_t B, int64_t L, int64_t stride) {
  BwdGeometry g;
  const int64_t M = std::max<int64_t>(L - 1, 0);
  g.nck = stride > 0 ? M / stride + 1 : 0;
  const size_t per_path = sizeof(T) * ((size_t)p->num_parts * M * p->d + (size_t)p->num_parts * g.nck * p->max_n);
  g.chunk = std::max<int64_t>(1, std::min<int64_t>(B, per_path ? (int64_t)(kWorkspaceBudget / per_path) : B));
  g.partial_bytes = sizeof(T) * (size_t)g.chunk * p->num_parts * M * p->d;
  g.ckpt_bytes = sizeof(T) * (size_t)g.chunk * p->num_parts * g.nck * p->max_n;
  return g;
}

template <typename T>
int backward_t(const sigb_plan* p, const void* X, int64_t B, int64_t L, const void* S, int64_t s_ld,
               int64_t s_col0, int s_is_state, const void* g, int64_t g_ld, int64_t g_col0, int64_t stride,
               void* work, size_t work_bytes, void* dX, void* dinc, cudaStream_t stream) {
  const int64_t M = L - 1;
  if (B == 0) return SIGB_OK;
  if (M == 0) {
    SIGB_CUDA_TRY(cudaMemsetAsync(dX, 0, sizeof(T) * B * p->d, stream));
    return SIGB_OK;
  }
  BwdGeometry geo = bwd_geometry<T>(p, B, L, stride);
  if (work_bytes < geo.partial_bytes + geo.ckpt_bytes || work == nullptr)
    return fail(SIGB_ERR_DOMAIN, "backward workspace too small");
  T* partial = (T*)work;
  T* ckpt = stride > 0 ? (T*)((char*)work + geo.partial_bytes) : nullptr;
  const size_t smem = smem_bytes<T>(p, true);
  int rc = check_smem(smem);
  if (rc) return rc;
  SIGB_CUDA_TRY(cudaFuncSetAttribute(backward_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int64_t b0 = 0; b0 < B; b0 += geo.chunk) {
    const int64_t Bc = std::min(geo.chunk, B - b0);
    if (stride > 0) {
      rc = forward_t<T>(p, (const T*)X + b0 * L * p->d, Bc, L, nullptr, 1, nullptr, 0, 0, 0, nullptr, ckpt, stride,
                        geo.nck, stream);
      if (rc) return rc;
    }
    count_launch(2);
    timing_begin(1, stream);
    backward_kernel<T><<<(unsigned)(Bc * p->num_parts), kThreads, smem, stream>>>(
        p->dev(), (const T*)X, L, b0, (const T*)S, s_ld, s_col0, s_is_state, p->Wc, (const T*)g, g_ld, g_col0,
        ckpt, stride, geo.nck, p->max_n, partial);
    timing_end(1, stream);
    SIGB_CUDA_TRY(cudaGetLastError());
    const int64_t n = Bc * L * p->d;
    sample_grads_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(partial, Bc, p->num_parts, M, p->d, b0,
                                                                             (T*)dX, (T*)dinc);
    SIGB_CUDA_TRY(cudaGetLastError());
  }
  return SIGB_OK;
}


// policy 0: truncated > generated (small sparse sets) > fragment > level; 1: level only;
// 2: fragment > level; 4: generated > fragment > level (3, the level-slot kernels, was removed in r02:
// it ran at ~5% of the FMA pipe and only served sets the fragment planner cannot cut)
bool use_trunc(const sigb_plan* p) { return g_policy == 0 && p->trunc_depth >= 2 && trunc::supported(p->d, p->trunc_depth); }
bool use_jit(const sigb_plan* p) {
  if (!p->jit.eligible || p->jit.broken || g_policy == 1 || g_policy == 2) return false;
  if (g_policy == 4) return true;
  if (use_trunc(p)) return false;
  // sparse sets: few words per fragment (the fragment kernels replicate chains there)
  return !p->frag.ok || (double)p->Wc / std::max(p->frag.F, 1) < 12.0;
}
bool use_frag(const sigb_plan* p) {
  if (!p->frag.ok || g_policy == 1) return false;
  return g_policy == 2 || (!use_trunc(p) && !use_jit(p));
}

int check_common(const sigb_plan* p, int dtype, int64_t B, int64_t L) {
  if (!p) return fail(SIGB_ERR_DOMAIN, "plan is NULL");
  if (dtype != SIGB_F32 && dtype != SIGB_F64) return fail(SIGB_ERR_SHAPE, "unsupported dtype; use float64 or float32");
  if (B < 0) return fail(SIGB_ERR_SHAPE, "negative batch size");
  if (L < 1) return fail(SIGB_ERR_SHAPE, "paths need at least one sample point");
  return SIGB_OK;
}

}  // namespace
}  // namespace sigb

using namespace sigb;

extern "C" int sigb_version(void) { return 100; }
extern "C" int sigb_plan_kernel_kind(const sigb_plan* plan) {
  return plan ? (use_trunc(plan) ? 1 : use_jit(plan) ? 4 : use_frag(plan) ? 2 : 0) : -1;
}
extern "C" int sigb_set_kernel_policy(int policy) {
  if (policy < 0 || policy > 4 || policy == 3)
    return fail(SIGB_ERR_DOMAIN, "kernel policy must be 0 (auto), 1 (level kernels), 2 (fragment kernels) "
                                 "or 4 (generated kernels)");
  g_policy = policy;
  return SIGB_OK;
}
extern "C" int64_t sigb_forward_ctas(const sigb_plan* plan, int64_t B) {
  if (!plan || B < 0) return -1;
  return use_trunc(plan) ? trunc::forward_ctas(plan->d, plan->trunc_depth, B) : -1;
}
extern "C" int sigb_set_tensor_cores(int on) {
  const int prev = g_tensor_cores;
  g_tensor_cores = on ? 1 : 0;
  return prev;
}
extern "C" long long sigb_launch_count(void) { return g_launches.load(); }

extern "C" int sigb_timing_enable(int on) {
  g_timing = on != 0;
  for (TimerSlot& t : g_slots) t.used = 0;
  return SIGB_OK;
}

extern "C" int sigb_timing_read(int which, double* ms, int64_t* launches) {
  if (which < 0 || which > 1 || !ms) return fail(SIGB_ERR_DOMAIN, "timing slot must be 0 (forward) or 1 (backward)");
  TimerSlot& t = g_slots[which];
  double total = 0;
  for (size_t i = 0; i < t.used; ++i) {
    SIGB_CUDA_TRY(cudaEventSynchronize(t.ev[i].second));
    float x = 0;
    SIGB_CUDA_TRY(cudaEventElapsedTime(&x, t.ev[i].first, t.ev[i].second));
    total += x;
  }
  *ms = total;
  if (launches) *launches = (int64_t)t.used;
  t.used = 0;
  return SIGB_OK;
}
extern "C" const char* sigb_last_error(void) { return g_last_error.c_str(); }

extern "C" int sigb_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

extern "C" int sigb_wordset_tables(const uint64_t* d_codes, const int64_t* d_lengths, int64_t W, int64_t d,
                                   int64_t max_len, int64_t* d_letters, int64_t* d_prefix, int64_t* d_suffix,
                                   int64_t* d_level_start, uint64_t* d_packed, void* stream) {
  return launch_wordset_tables(d_codes, d_lengths, W, d, max_len, d_letters, d_prefix, d_suffix, d_level_start,
                               d_packed, (cudaStream_t)stream);
}

extern "C" int sigb_forward(const sigb_plan* plan, int dtype, const void* d_X, int64_t B, int64_t L, void* d_out,
                            int64_t out_ld, int64_t out_col0, int include_empty, void* d_state, void* stream) {
  int rc = check_common(plan, dtype, B, L);
  if (rc) return rc;
  DeviceGuard guard(plan->device);
  if (include_empty && out_col0 < 1) return fail(SIGB_ERR_SHAPE, "include_empty needs out_col0 >= 1");
  if (use_trunc(plan)) {
    return trunc::forward(dtype, plan->d, plan->trunc_depth, d_X, B, L, nullptr, 1, d_out, out_ld, out_col0, include_empty,
                          (cudaStream_t)stream);
  }
  if (use_jit(plan)) {
    rc = jit::forward(plan, dtype, d_X, B, L, d_out, out_ld, out_col0, include_empty, d_state, (cudaStream_t)stream);
    if (rc == SIGB_OK) return rc;
    if (g_policy == 4)
      return rc == jit::kPending ? fail(SIGB_ERR_UNSUPPORTED, "generated kernel not ready") : rc;
    // compiling in the background (jit::kPending) or failed: the fragment kernels serve the call
    if (plan->frag.ok)
      return frag::forward(plan, dtype, d_X, B, L, nullptr, 1, d_out, out_ld, out_col0, include_empty, d_state,
                           (cudaStream_t)stream);
  }
  if (use_frag(plan))
    return frag::forward(plan, dtype, d_X, B, L, nullptr, 1, d_out, out_ld, out_col0, include_empty, d_state,
                         (cudaStream_t)stream);
  if (dtype == SIGB_F32)
    return forward_t<float>(plan, d_X, B, L, nullptr, 1, d_out, out_ld, out_col0, include_empty, d_state, nullptr, 0,
                            0, (cudaStream_t)stream);
  return forward_t<double>(plan, d_X, B, L, nullptr, 1, d_out, out_ld, out_col0, include_empty, d_state, nullptr, 0,
                           0, (cudaStream_t)stream);
}

extern "C" int sigb_windows(const sigb_plan* plan, int dtype, const void* d_X, int64_t B, int64_t L,
                            const int64_t* d_bounds, int64_t K, void* d_out, void* stream) {
  int rc = check_common(plan, dtype, B, L);
  if (rc) return rc;
  DeviceGuard guard(plan->device);
  if (K < 1 || !d_bounds) return fail(SIGB_ERR_DOMAIN, "need at least one window");
  // windows = B*K virtual paths over the same register-resident kernels as sigb_forward
  if (use_trunc(plan))
    return trunc::forward(dtype, plan->d, plan->trunc_depth, d_X, B * K, L, d_bounds, K, d_out, plan->W, 0, 0,
                          (cudaStream_t)stream);
  // generated kernels have no windowed form: windows run on the fragment kernels
  if (plan->frag.ok && g_policy != 1 && !use_trunc(plan))
    return frag::forward(plan, dtype, d_X, B * K, L, d_bounds, K, d_out, plan->W, 0, 0, nullptr, (cudaStream_t)stream);
  if (dtype == SIGB_F32)
    return forward_t<float>(plan, d_X, B, L, d_bounds, K, d_out, plan->W, 0, 0, nullptr, nullptr, 0, 0,
                            (cudaStream_t)stream);
  return forward_t<double>(plan, d_X, B, L, d_bounds, K, d_out, plan->W, 0, 0, nullptr, nullptr, 0, 0,
                           (cudaStream_t)stream);
}

extern "C" int sigb_backward_workspace_size(const sigb_plan* plan, int dtype, int64_t B, int64_t L,
                                            int64_t ckpt_stride, size_t* bytes) {
  int rc = check_common(plan, dtype, B, L);
  if (rc) return rc;
  DeviceGuard guard(plan->device);
  if (ckpt_stride < 0) return fail(SIGB_ERR_DOMAIN, "checkpoint stride must be >= 1");
  if (B == 0 || L == 1) { *bytes = 0; return SIGB_OK; }
  if (use_trunc(plan)) {  // checkpoint_stride included (replay + reload in the truncated kernels)
    *bytes = trunc::backward_workspace(dtype, plan->d, plan->trunc_depth, B, L, ckpt_stride);
    return SIGB_OK;
  }
  if (use_jit(plan) && ckpt_stride == 0 &&
      jit::ensure(const_cast<sigb_plan*>(plan), dtype, true, jit::wait_default()) == SIGB_OK) {
    *bytes = jit::backward_workspace(plan, dtype, B, L);
    return SIGB_OK;
  }
  if (use_jit(plan) && ckpt_stride == 0 && plan->frag.ok) {  // generated kernel still compiling
    *bytes = frag::backward_workspace(plan, dtype, B, L);
    return SIGB_OK;
  }
  if (use_frag(plan) || (ckpt_stride > 0 && use_jit(plan) && plan->frag.ok)) {
    // checkpoint_stride on the fragment kernels (the generated kernels take none)
    *bytes = frag::backward_workspace(plan, dtype, B, L, ckpt_stride);
    return SIGB_OK;
  }
  if (dtype == SIGB_F32) {
    BwdGeometry g = bwd_geometry<float>(plan, B, L, ckpt_stride);
    *bytes = g.partial_bytes + g.ckpt_bytes;
  } else {
    BwdGeometry g = bwd_geometry<double>(plan, B, L, ckpt_stride);
    *bytes = g.partial_bytes + g.ckpt_bytes;
  }
  return SIGB_OK;
}

extern "C" int sigb_backward(const sigb_plan* plan, int dtype, const void* d_X, int64_t B, int64_t L,
                             const void* d_S, int64_t s_ld, int64_t s_col0, int s_is_state, const void* d_g,
                             int64_t g_ld, int64_t g_col0, int64_t ckpt_stride, void* d_work, size_t work_bytes,
                             void* d_dX, void* d_dinc, void* stream) {
  int rc = check_common(plan, dtype, B, L);
  if (rc) return rc;
  DeviceGuard guard(plan->device);
  if (ckpt_stride < 0) return fail(SIGB_ERR_DOMAIN, "checkpoint stride must be >= 1");
  if (!s_is_state && !plan->prefix_closed)
    return fail(SIGB_ERR_DOMAIN, "word set is not prefix-closed: pass the closure state from sigb_forward");
  if (use_trunc(plan) && B > 0 && L > 1) {
    if (s_is_state) { s_ld = plan->Wc; s_col0 = 0; }
    return trunc::backward(dtype, plan->d, plan->trunc_depth, d_X, B, L, d_S, s_ld, s_col0, d_g, g_ld, g_col0, d_work,
                           work_bytes, d_dX, d_dinc, (cudaStream_t)stream, ckpt_stride);
  }
  if (use_jit(plan) && ckpt_stride == 0 && B > 0 && L > 1) {
    if (s_is_state) { s_ld = plan->Wc; s_col0 = 0; }
    // the generated kernel once it is loaded and the caller's workspace was sized for it (the
    // workspace query may have run while it compiled); else the fragment kernels
    if (jit::ensure(const_cast<sigb_plan*>(plan), dtype, true, jit::wait_default()) == SIGB_OK &&
        work_bytes >= jit::backward_workspace(plan, dtype, B, L))
      return jit::backward(plan, dtype, d_X, B, L, d_S, s_ld, s_col0, d_g, g_ld, g_col0, d_work, work_bytes, d_dX,
                           d_dinc, (cudaStream_t)stream);
    if (g_policy == 4) return fail(SIGB_ERR_DOMAIN, "backward workspace too small for the generated kernel");
    if (plan->frag.ok)
      return frag::backward(plan, dtype, d_X, B, L, d_S, s_ld, s_col0, d_g, g_ld, g_col0, d_work, work_bytes, d_dX,
                            d_dinc, (cudaStream_t)stream);
  }
  if ((use_frag(plan) || (ckpt_stride > 0 && use_jit(plan) && plan->frag.ok)) && B > 0 && L > 1) {
    if (s_is_state) { s_ld = plan->Wc; s_col0 = 0; }
    return frag::backward(plan, dtype, d_X, B, L, d_S, s_ld, s_col0, d_g, g_ld, g_col0, d_work, work_bytes, d_dX,
                          d_dinc, (cudaStream_t)stream, ckpt_stride);
  }
  if (dtype == SIGB_F32)
    return backward_t<float>(plan, d_X, B, L, d_S, s_ld, s_col0, s_is_state, d_g, g_ld, g_col0, ckpt_stride, d_work,
                             work_bytes, d_dX, d_dinc, (cudaStream_t)stream);
  return backward_t<double>(plan, d_X, B, L, d_S, s_ld, s_col0, s_is_state, d_g, g_ld, g_col0, ckpt_stride, d_work,
                            work_bytes, d_dX, d_dinc, (cudaStream_t)stream);
}
