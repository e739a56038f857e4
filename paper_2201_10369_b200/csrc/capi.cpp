// The C ABI of libwino (include/wino.h): validation, host matrix construction, launch.
#include <cmath>
#include <mutex>
#include <string>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "wino_internal.h"
#include "huff_jit.h"

namespace wino {

namespace {
thread_local char g_err[512] = "";
thread_local int g_launches = 0;
thread_local int g_last_launches = 0;
}  // namespace

int set_error(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}
void count_launches(int n) { g_launches += n; }
void reset_launches() { g_launches = 0; }

namespace {
struct Rec {
  std::string family;
  cudaEvent_t a, b;
  int count;
};
std::mutex g_tmu;
bool g_timing = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
}  // namespace

bool timing_enabled() { return g_timing; }
cudaEvent_t timing_event() {
  std::lock_guard<std::mutex> lk(g_tmu);
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
void timing_record(const char* family, cudaEvent_t a, cudaEvent_t b, int count) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_recs.push_back(Rec{family, a, b, count});
}

}  // namespace wino

using namespace wino;

namespace {
int finish(int status) {
  if (status == WINO_OK) g_last_launches = g_launches;
  return status;
}

// RN32 of the R64 matrices.
void to_f32(const double* src, int count, float* dst) {
  for (int i = 0; i < count; i++) dst[i] = (float)src[i];
}
}  // namespace

extern "C" {

const char* wino_status_string(int status) {
  switch (status) {
    case WINO_OK: return "WINO_OK";
    case WINO_E_INVALID_ARG: return "WINO_E_INVALID_ARG";
    case WINO_E_BAD_SHAPE: return "WINO_E_BAD_SHAPE";
    case WINO_E_DUPLICATE_POINTS: return "WINO_E_DUPLICATE_POINTS";
    case WINO_E_INF_NOT_LAST: return "WINO_E_INF_NOT_LAST";
    case WINO_E_NONFINITE_POINT: return "WINO_E_NONFINITE_POINT";
    case WINO_E_WORKSPACE: return "WINO_E_WORKSPACE";
    case WINO_E_CUDA: return "WINO_E_CUDA";
    case WINO_E_UNSUPPORTED: return "WINO_E_UNSUPPORTED";
    default: return "WINO_E_UNKNOWN";
  }
}

const char* wino_last_error(void) { return g_err; }

int wino_last_launch_count(void) { return g_last_launches; }

int wino_huffman_jit_mode(int mode) { return huff_jit_set_mode(mode < 0 || mode > 2 ? 0 : mode); }

int wino_huffman_jit_classes(void) { return huff_jit_cache_size(); }

int wino_huffman_jit_compile_check(int dims, int m, int r, const double* points, size_t* cubin_bytes) {
  if (!points || !cubin_bytes) return set_error(WINO_E_INVALID_ARG, "NULL pointer");
  if (dims < 1 || dims > 2 || m < 1 || r < 1 || m + r - 1 > WINO_MAX_N)
    return set_error(WINO_E_BAD_SHAPE, "bad shape dims=%d m=%d r=%d", dims, m, r);
  std::string prog, cubin, log;
  const int s = huff_class_program(m, r, points, prog);
  if (s != WINO_OK) return set_error(s, "%s", build_error_detail(s));
  if (huff_jit_compile(huff_jit_source(dims, m, r, prog), cubin, log) != 0)
    return set_error(WINO_E_CUDA, "NVRTC: %s", log.substr(0, 900).c_str());
  *cubin_bytes = cubin.size();
  return WINO_OK;
}

int wino_timing_enable(int enable) {
  std::lock_guard<std::mutex> lk(g_tmu);
  const int prev = g_timing ? 1 : 0;
  g_timing = enable != 0;
  return prev;
}

void wino_timing_reset(void) {
  std::lock_guard<std::mutex> lk(g_tmu);
  for (auto& r : g_recs) {
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
}

int wino_timing_read(const char* family, double* total_ms, int* launches) {
  if (!family || !total_ms || !launches) return set_error(WINO_E_INVALID_ARG, "NULL pointer");
  std::lock_guard<std::mutex> lk(g_tmu);
  double tot = 0.0;
  int cnt = 0;
  for (auto& r : g_recs) {
    if (r.family != family) continue;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return set_error(WINO_E_CUDA, "cudaEventSynchronize: %s", cudaGetErrorString(e));
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    tot += ms;
    cnt += r.count;
  }
  *total_ms = tot;
  *launches = cnt;
  return WINO_OK;
}

int wino_supported(int dims, int m, int r) {
  if (dims == 1 || dims == 2) return sweep_supported(dims, m, r);
  if (dims == 0) return layer_supported(m, r);  // 0 = the layer kernels
  return 0;
}

int wino_points_to_matrices(int m, int r, const double* points, int n, double* AT, double* G, double* BT) {
  const int s = build_r64(m, r, points, n, AT, G, BT);
  if (s != WINO_OK) return set_error(s, "wino_points_to_matrices: %s", build_error_detail(s));
  return WINO_OK;
}

size_t wino_conv2d_workspace_bytes(int N, int C, int H, int W, int K, int r, int pad, int m) {
  if (N < 1 || C < 1 || H < 1 || W < 1 || K < 1 || r < 1 || m < 1 || pad < 0) return 0;
  if (H + 2 * pad < r || W + 2 * pad < r) return 0;
  return layer_workspace_bytes(N, C, H, W, K, r, pad, m);
}

int wino_conv2d_gemm_tile(int N, int C, int H, int W, int K, int r, int pad, int m) {
  if (N < 1 || C < 1 || H < 1 || W < 1 || K < 1 || r < 1 || m < 1 || pad < 0) return 0;
  if (H + 2 * pad < r || W + 2 * pad < r || !layer_supported(m, r)) return 0;
  return layer_gemm_tile(N, C, H, W, K, r, pad, m);
}

int wino_conv2d_fp32(const float* x, const float* w, float* y, int N, int C, int H, int W, int K, int r, int pad,
                     int m, const double* points, void* workspace, size_t workspace_bytes, double* d_sums,
                     double* d_maxs, void* stream) {
  return wino_conv2d_fp32_ex(x, w, y, N, C, H, W, K, r, pad, m, points, workspace, workspace_bytes, d_sums, d_maxs,
                             0u, stream);
}

static int conv_common(const float* x, const float* w, float* y, float* act, int pool, int N, int C, int H, int W,
                       int K, int r, int pad, int m, const double* points, void* workspace, size_t workspace_bytes,
                       double* d_sums, double* d_maxs, unsigned flags, void* stream) {
  reset_launches();
  if (!x || !w || !points || (!y && !act)) return set_error(WINO_E_INVALID_ARG, "NULL pointer");
  if (N < 0 || C < 1 || H < 1 || W < 1 || K < 0 || r < 1 || m < 1 || pad < 0)
    return set_error(WINO_E_INVALID_ARG, "negative batch / output channels, non-positive size or negative pad");
  if (flags & ~(WINO_CONV_TF32 | WINO_CONV_3XTF32 | WINO_CONV_SCORE_PER_IMAGE))
    return set_error(WINO_E_INVALID_ARG, "unknown flags");
  if ((d_sums == nullptr) != (d_maxs == nullptr))
    return set_error(WINO_E_INVALID_ARG, "d_sums and d_maxs must both be NULL or both non-NULL");
  if (act && pool != 1 && pool != 2) return set_error(WINO_E_INVALID_ARG, "pool must be 1 or 2");
  if (!y && (d_sums || (act && pool == 2 && m % 2 != 0)))
    return set_error(WINO_E_INVALID_ARG, "y is required for scoring and for pool 2 with odd m");
  if (H + 2 * pad < r || W + 2 * pad < r) return set_error(WINO_E_BAD_SHAPE, "empty output");
  if (reinterpret_cast<uintptr_t>(workspace) & 255u)
    return set_error(WINO_E_WORKSPACE, "workspace must be 256-byte aligned");
  if ((reinterpret_cast<uintptr_t>(d_sums) | reinterpret_cast<uintptr_t>(d_maxs)) & 7u)
    return set_error(WINO_E_INVALID_ARG, "statistics buffers must be 8-byte aligned");
  if (act && pool == 2 && (H + 2 * pad - r + 1 < 2 || W + 2 * pad - r + 1 < 2))
    return set_error(WINO_E_BAD_SHAPE, "pool 2 needs an output of at least 2 x 2");
  const int n = m + r - 1;
  if (n > WINO_MAX_N) return set_error(WINO_E_UNSUPPORTED, "n > WINO_MAX_N");
  if (!layer_supported(m, r)) return set_error(WINO_E_UNSUPPORTED, "no layer kernel for m=%d r=%d", m, r);
  std::vector<double> AT(m * n), G(n * r), BT(n * n);
  const int s = build_r64(m, r, points, n, AT.data(), G.data(), BT.data());
  if (s != WINO_OK) return set_error(s, "points: %s", build_error_detail(s));
  if (N == 0 || K == 0) return finish(WINO_OK);   // empty batch / no filters: nothing to enqueue
  std::vector<float> ATf(m * n), Gf(n * r), BTf(n * n);
  to_f32(AT.data(), m * n, ATf.data());
  to_f32(G.data(), n * r, Gf.data());
  to_f32(BT.data(), n * n, BTf.data());
  return finish(layer_launch(x, w, y, N, C, H, W, K, r, pad, m, ATf.data(), Gf.data(), BTf.data(), workspace,
                             workspace_bytes, d_sums, d_maxs, flags, (cudaStream_t)stream, act, act ? pool : 0));
}

int wino_conv2d_fp32_ex(const float* x, const float* w, float* y, int N, int C, int H, int W, int K, int r, int pad,
                        int m, const double* points, void* workspace, size_t workspace_bytes, double* d_sums,
                        double* d_maxs, unsigned flags, void* stream) {
  if (!y) {
    reset_launches();
    return set_error(WINO_E_INVALID_ARG, "NULL pointer");
  }
  return conv_common(x, w, y, nullptr, 0, N, C, H, W, K, r, pad, m, points, workspace, workspace_bytes, d_sums,
                     d_maxs, flags, stream);
}

int wino_conv2d_relu_pool_fp32(const float* x, const float* w, float* y, float* act, int N, int C, int H, int W,
                               int K, int r, int pad, int m, const double* points, void* workspace,
                               size_t workspace_bytes, double* d_sums, double* d_maxs, int pool, unsigned flags,
                               void* stream) {
  if (!act) {
    reset_launches();
    return set_error(WINO_E_INVALID_ARG, "NULL act");
  }
  return conv_common(x, w, y, act, pool, N, C, H, W, K, r, pad, m, points, workspace, workspace_bytes, d_sums,
                     d_maxs, flags, stream);
}

int wino_relu_pool_fp32(const float* x, float* y, int N, int C, int H, int W, int pool, void* stream) {
  reset_launches();
  if (!x || !y) return set_error(WINO_E_INVALID_ARG, "NULL pointer");
  if (N < 1 || C < 1 || H < 1 || W < 1 || (pool != 1 && pool != 2))
    return set_error(WINO_E_INVALID_ARG, "bad sizes or pool not 1|2");
  if (pool == 2 && (H < 2 || W < 2)) return set_error(WINO_E_BAD_SHAPE, "pool 2 needs H, W >= 2");
  return finish(relu_pool_launch(x, y, N, C, H, W, pool, (cudaStream_t)stream));
}

size_t wino_error_sweep_workspace_bytes(int dims, int m, int r, int n_cand, int64_t n_tiles) {
  if ((dims != 1 && dims != 2) || m < 1 || r < 1 || n_cand < 0 || n_tiles < 0) return 0;
  return sweep_workspace_bytes(dims, m, r, n_cand, n_tiles);
}

static int sweep_common(int dims, int m, int r, const double* point_sets, int n_cand, const float* d_tiles,
                        const float* g_tiles, int64_t n_tiles, double* d_sums, double* d_maxs, float* d_y,
                        int* cand_status, void* workspace, size_t ws_bytes, unsigned flags, void* stream) {
  reset_launches();
  if (dims != 1 && dims != 2) return set_error(WINO_E_INVALID_ARG, "dims must be 1 or 2");
  if (m < 1 || r < 1 || n_cand < 0 || n_tiles < 0) return set_error(WINO_E_INVALID_ARG, "bad sizes");
  if (n_cand > 0 && (!point_sets || !cand_status)) return set_error(WINO_E_INVALID_ARG, "NULL pointer");
  if (n_cand > 0 && n_tiles > 0 && (!d_tiles || !g_tiles)) return set_error(WINO_E_INVALID_ARG, "NULL tiles");
  if ((reinterpret_cast<uintptr_t>(d_tiles) | reinterpret_cast<uintptr_t>(g_tiles)) & 15u)
    return set_error(WINO_E_INVALID_ARG, "d_tiles / g_tiles must be 16-byte aligned (vector loads)");
  if ((reinterpret_cast<uintptr_t>(d_sums) | reinterpret_cast<uintptr_t>(d_maxs)) & 7u)
    return set_error(WINO_E_INVALID_ARG, "statistics buffers must be 8-byte aligned");
  if (reinterpret_cast<uintptr_t>(workspace) & 255u)
    return set_error(WINO_E_WORKSPACE, "workspace must be 256-byte aligned");
  if ((d_sums == nullptr) != (d_maxs == nullptr))
    return set_error(WINO_E_INVALID_ARG, "d_sums and d_maxs must both be NULL or both non-NULL");
  if (flags & ~(WINO_SWEEP_NOFMA | WINO_SWEEP_HUFFMAN | WINO_SWEEP_MIXED))
    return set_error(WINO_E_INVALID_ARG, "unknown flags");
  if ((flags & WINO_SWEEP_HUFFMAN) && (flags & WINO_SWEEP_MIXED))
    return set_error(WINO_E_INVALID_ARG, "WINO_SWEEP_HUFFMAN and WINO_SWEEP_MIXED are exclusive");
  const int n = m + r - 1;
  if (n > WINO_MAX_N) return set_error(WINO_E_UNSUPPORTED, "n > WINO_MAX_N");
  if (!sweep_supported(dims, m, r))
    return set_error(WINO_E_UNSUPPORTED, "no sweep kernel for dims=%d m=%d r=%d", dims, m, r);
  return finish(sweep_launch(dims, m, r, point_sets, cand_status, n_cand, d_tiles, g_tiles, n_tiles, d_sums,
                             d_maxs, d_y, workspace, ws_bytes, flags, (cudaStream_t)stream));
}

int wino_error_sweep(int dims, int m, int r, const double* point_sets, int n_cand, const float* d_tiles,
                     const float* g_tiles, int64_t n_tiles, double* d_sums, double* d_maxs, int* cand_status,
                     void* workspace, size_t workspace_bytes, unsigned flags, void* stream) {
  if (n_cand > 0 && (!d_sums || !d_maxs)) {
    reset_launches();
    return set_error(WINO_E_INVALID_ARG, "NULL stats");
  }
  return sweep_common(dims, m, r, point_sets, n_cand, d_tiles, g_tiles, n_tiles, d_sums, d_maxs, nullptr,
                      cand_status, workspace, workspace_bytes, flags, stream);
}

int wino_sweep_outputs(int dims, int m, int r, const double* point_sets, int n_cand, const float* d_tiles,
                       const float* g_tiles, int64_t n_tiles, float* d_y, double* d_sums, double* d_maxs,
                       int* cand_status, void* workspace, size_t workspace_bytes, unsigned flags, void* stream) {
  if (!d_y && n_cand > 0 && n_tiles > 0) {
    reset_launches();
    return set_error(WINO_E_INVALID_ARG, "NULL d_y");
  }
  return sweep_common(dims, m, r, point_sets, n_cand, d_tiles, g_tiles, n_tiles, d_sums, d_maxs, d_y, cand_status,
                      workspace, workspace_bytes, flags, stream);
}

}  // extern "C"
