// Internal helpers shared by the sm_100a kernels and the C ABI of libwino.
// Nothing here is visible across the ABI (include/wino.h is the boundary).
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

#include "../../include/wino.h"

namespace wino {

// ---- host-side status plumbing (capi.cpp) ---------------------------------------
int set_error(int status, const char* fmt, ...);
void count_launches(int n);   // adds to the per-call launch counter
void reset_launches();

// ---- host fp64 matrix builder, recipe R64 (host_builder.cpp) ----------------------
// Validates (m, r, points) and fills AT[m*n], G[n*r], BT[n*n].  Returns a wino_status,
// without touching the thread's last-error message (callers decide).
int build_r64(int m, int r, const double* points, int n, double* AT, double* G, double* BT);
const char* build_error_detail(int status);

// ---- launchers (sweep.cu, layer.cu) ------------------------------------------------
// fp32 matrices of one candidate, packed [AT (m*n) | G (n*r) | BT (n*n)].
int sweep_supported(int dims, int m, int r);
int sweep_max_cands_per_launch(int dims, int m, int r);
size_t sweep_workspace_bytes(int dims, int m, int r, int n_cand, int64_t n_tiles);
// Builds the candidates' matrices (R64 -> RN32) chunk by chunk on the host and launches
// K6 (refs) once, then K7+K8 per chunk.  point_sets: HOST [n_cand][n]; cand_status: HOST
// out (rejected candidates are skipped).
int sweep_launch(int dims, int m, int r, const double* point_sets, int* cand_status, int n_cand,
                 const float* d_tiles, const float* g_tiles, int64_t n_tiles,
                 double* d_sums, double* d_maxs, float* d_y, void* workspace, size_t ws_bytes,
                 unsigned flags, cudaStream_t stream);

int layer_supported(int m, int r);
size_t layer_workspace_bytes(int N, int C, int H, int W, int K, int r, int pad, int m);
int layer_gemm_tile(int N, int C, int H, int W, int K, int r, int pad, int m);
int layer_launch(const float* x, const float* w, float* y, int N, int C, int H, int W, int K,
                 int r, int pad, int m, const float* AT, const float* G, const float* BT,
                 void* workspace, size_t ws_bytes, double* d_sums, double* d_maxs,
                 unsigned flags, cudaStream_t stream, float* act = nullptr, int pool = 0);

int relu_pool_launch(const float* x, float* y, int N, int C, int H, int W, int pool, cudaStream_t stream);

// ---- kernel timing hook (capi.cpp): when enabled, brackets the launch with cudaEvents
// on `stream` under the name `family` (read back by wino_timing_read).
bool timing_enabled();
// `count`: launches the (start, stop) pair brackets (a PDL chain of sweep launches is timed
// as one interval: events between chained launches would serialise them)
void timing_record(const char* family, cudaEvent_t start, cudaEvent_t stop, int count = 1);
cudaEvent_t timing_event();
template <class F>
void timed_launch(const char* family, cudaStream_t stream, F&& launch) {
  if (!timing_enabled()) {
    launch();
    return;
  }
  cudaEvent_t a = timing_event(), b = timing_event();
  cudaEventRecord(a, stream);
  launch();
  cudaEventRecord(b, stream);
  timing_record(family, a, b);
}

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace wino
