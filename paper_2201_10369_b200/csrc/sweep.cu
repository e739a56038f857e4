// Error sweep over candidate point sets (PAPER.md P:465 error protocol, P:472 sweep),
// sm_100a.  Kernels:
//   K6 sweep_refs    : y64 = fp64 direct valid correlation of every tile (c-independent, once)
//   K7 sweep1d/2d    : per (candidate, tile) fp32 Winograd, fused in registers, scored
//                      against y64; per-warp partial statistics
//   K8 sweep_finalize: fixed-order reduction of the partials, accumulated into d_sums/d_maxs
//
// Design:
//  * Each thread owns TWO tiles and evaluates them as a pair with FFMA2
//    (fma.rn.f32x2): both halves use the same warp-uniform coefficient, which the
//    hardware broadcasts from a uniform register (SASS `FFMA2 R, R.F32x2, UR.F32, R`).
//    One FFMA2 issue = 64 lane-FMAs, so the FP32 pipe saturates at half the issue
//    slots, leaving the other half for the fp64 scoring (separate FP64 pipe), the
//    uniform coefficient loads and shared-memory traffic.
//  * Coefficients of up to ~8000/per candidates ride in the kernel parameter space
//    (__grid_constant__, 32 KB); indexing it with the warp-uniform candidate index
//    compiles to LDCU UR, c[0x0][UR+off].
//  * Tiles (and their y64) are staged once per CTA in shared memory and reused for
//    every candidate of the CTA's candidate group.
//  * Arithmetic is the canonical O5 order: every dot product is an
//    fmaf chain from +0 in ascending index order, 2D left product first, so outputs
//    are bit-identical to the oracle.  Rows of V are streamed: for each row i the
//    kernel forms T1 row i -> U row i, T2 row i -> V row i, M row i = U⊙V and
//    accumulates T3 += Aᵀ[:,i] M[i,:] -- per element the same chain as the oracle.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "wino_internal.h"

namespace wino {

typedef unsigned long long u64;

constexpr int kSwThreads = 128;        // 4 warps, one per SM sub-partition
constexpr int kParamFloats = 7424;     // coefficient floats per launch (29696 B)
constexpr int kMaxCandsLaunch = 512;   // + 2 KB of candidate indices: < 32764 B of params

struct MatsParam {
  float v[kParamFloats];
};
struct IdxParam {
  int idx[kMaxCandsLaunch];
};

struct SweepArgs {
  const float* d;
  const float* g;
  const double* y64;
  float* ydump;
  double* partial;     // [n_cand_launch][n_tblk][4 warps][8]
  long long n_tiles;
  int n_cand;          // candidates in this launch
  int cands_per_cta;
  int n_tblk;
  int ydump_cand0;     // not used for indexing: dump rows are addressed by dump_idx
};

// ------------------------------------------------------------------ lane arithmetic
// Pair<true>: two tiles per thread (FFMA2), Pair<false>: one tile (FFMA).
// NOFMA (paper arithmetic) uses scalar __fmul_rn/__fadd_rn: ptxas 12.9 contracts
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2, so the pair form cannot express it.
template <bool PAIR, bool NOFMA>
struct Lane;

template <bool NOFMA>
struct Lane<true, NOFMA> {
  typedef u64 T;
  static constexpr int W = 2;
  static __device__ __forceinline__ T pack(float a, float b) {
    T p;
    asm("mov.b64 %0, {%1,%2};" : "=l"(p) : "f"(a), "f"(b));
    return p;
  }
  static __device__ __forceinline__ float lo(T p) {
    float a, b;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(p));
    return a;
  }
  static __device__ __forceinline__ float hi(T p) {
    float a, b;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(p));
    return b;
  }
  static __device__ __forceinline__ T zero() { return 0ull; }
  // acc + a * c  (c broadcast to both halves)
  static __device__ __forceinline__ T fma(T a, float c, T acc) {
    if (NOFMA) {
      return pack(__fadd_rn(lo(acc), __fmul_rn(lo(a), c)), __fadd_rn(hi(acc), __fmul_rn(hi(a), c)));
    } else {
      T d;
      T cc = pack(c, c);
      asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(cc), "l"(acc));
      return d;
    }
  }
  // elementwise a * b + (+0): the Hadamard product of the C = 1 contraction (O5)
  static __device__ __forceinline__ T mul(T a, T b) {
    if (NOFMA) {
      return pack(__fadd_rn(0.0f, __fmul_rn(lo(a), lo(b))), __fadd_rn(0.0f, __fmul_rn(hi(a), hi(b))));
    } else {
      T d;
      T z = 0ull;
      asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(z));
      return d;
    }
  }
  static __device__ __forceinline__ float get(T v, int h) { return h ? hi(v) : lo(v); }
};

template <bool NOFMA>
struct Lane<false, NOFMA> {
  typedef float T;
  static constexpr int W = 1;
  static __device__ __forceinline__ T zero() { return 0.0f; }
  static __device__ __forceinline__ T fma(T a, float c, T acc) {
    return NOFMA ? __fadd_rn(acc, __fmul_rn(a, c)) : __fmaf_rn(a, c, acc);
  }
  static __device__ __forceinline__ T mul(T a, T b) {
    return NOFMA ? __fadd_rn(0.0f, __fmul_rn(a, b)) : __fmaf_rn(a, b, 0.0f);
  }
  static __device__ __forceinline__ float get(T v, int) { return v; }
};

// ------------------------------------------------------------------ statistics
struct Stat {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, m0 = 0.0, m1 = 0.0;
  int nonfin = 0;
  __device__ __forceinline__ void add(float y32, double y64) {
    const double e = (double)y32 - y64;
    if (isfinite(e)) {
      const double ae = fabs(e), ay = fabs(y64);
      s0 += ae;
      s1 = __fma_rn(e, e, s1);
      s2 += ay;
      m0 = fmax(m0, ae);
      m1 = fmax(m1, ay);
    } else {
      nonfin++;
    }
  }
  // butterfly over the warp (fixed order -> deterministic)
  __device__ __forceinline__ void warp_reduce() {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      m0 = fmax(m0, __shfl_xor_sync(0xffffffffu, m0, o));
      m1 = fmax(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    nonfin = __reduce_add_sync(0xffffffffu, nonfin);
  }
};

// Write the warp partial: {s0, s1, s2, n_scored, n_nonfinite, m0, m1, 0}
__device__ __forceinline__ void write_partial(double* p, const Stat& st, int n_valid_out) {
  p[0] = st.s0;
  p[1] = st.s1;
  p[2] = st.s2;
  p[3] = (double)(n_valid_out - st.nonfin);
  p[4] = (double)st.nonfin;
  p[5] = st.m0;
  p[6] = st.m1;
  p[7] = 0.0;
}

// ------------------------------------------------------------------ K6: fp64 references
template <int DIMS, int M, int R>
__global__ void sweep_refs_kernel(const float* __restrict__ d, const float* __restrict__ g,
                                  double* __restrict__ y64, long long n_tiles) {
  constexpr int N = M + R - 1;
  constexpr int DN = DIMS == 1 ? N : N * N, DG = DIMS == 1 ? R : R * R, DY = DIMS == 1 ? M : M * M;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  const float* dt = d + t * DN;
  const float* gt = g + t * DG;
  double* yt = y64 + t * DY;
  if (DIMS == 1) {
    for (int p = 0; p < M; p++) {
      double acc = 0.0;
      for (int j = 0; j < R; j++) acc = __dadd_rn(acc, __dmul_rn((double)gt[j], (double)dt[p + j]));
      yt[p] = acc;
    }
  } else {
    for (int p = 0; p < M; p++)
      for (int s = 0; s < M; s++) {
        double acc = 0.0;
        for (int u = 0; u < R; u++)
          for (int v = 0; v < R; v++)
            acc = __dadd_rn(acc, __dmul_rn((double)gt[u * R + v], (double)dt[(p + u) * N + s + v]));
        yt[p * M + s] = acc;
      }
  }
}

// ------------------------------------------------------------------ K7 (2D)
// smem: sd [NN][128] T (tiles), st2 [NN][128] T (T2 staging), sy [MM][W][128] double
template <int M, int R, bool PAIR, bool NOFMA, bool DUMP>
__global__ void __launch_bounds__(kSwThreads) sweep2d_kernel(SweepArgs a, const __grid_constant__ MatsParam P,
                                                             const __grid_constant__ IdxParam DI) {
  using L = Lane<PAIR, NOFMA>;
  using T = typename L::T;
  constexpr int W = L::W;
  constexpr int N = M + R - 1, NN = N * N, MM = M * M, RR = R * R;
  constexpr int OFF_G = M * N, OFF_B = M * N + N * R, PER = OFF_B + N * N;
  constexpr int TPB = kSwThreads * W;

  extern __shared__ __align__(16) unsigned char smem[];
  T* sd = reinterpret_cast<T*>(smem);
  T* st2 = sd + NN * kSwThreads;
  double* sy = reinterpret_cast<double*>(st2 + NN * kSwThreads);

  const int tid = threadIdx.x, warp = tid >> 5;
  const long long tile0 = (long long)blockIdx.x * TPB;
  const long long ntl = a.n_tiles - tile0 < TPB ? a.n_tiles - tile0 : TPB;  // tiles in this block

  // ---- stage the block's tiles (coalesced: the block's tiles are contiguous in memory)
  {
    float* sdf = reinterpret_cast<float*>(sd);
    const float* src = a.d + tile0 * NN;
    for (int idx = tid; idx < TPB * NN; idx += kSwThreads) {
      const int tl = idx / NN, e = idx - tl * NN;
      const float v = tl < ntl ? src[idx] : 0.0f;
      sdf[(e * kSwThreads + (tl % kSwThreads)) * W + tl / kSwThreads] = v;
    }
    if (!DUMP) {
      const double* ysrc = a.y64 + tile0 * MM;
      for (int idx = tid; idx < TPB * MM; idx += kSwThreads) {
        const int tl = idx / MM, o = idx - tl * MM;
        sy[(o * W + tl / kSwThreads) * kSwThreads + (tl % kSwThreads)] = tl < ntl ? ysrc[idx] : 0.0;
      }
    }
  }
  // ---- this thread's kernel tiles g (registers)
  T g[RR];
#pragma unroll
  for (int e = 0; e < RR; e++) {
    float gv[2] = {0.0f, 0.0f};
#pragma unroll
    for (int h = 0; h < W; h++) {
      const long long t = tile0 + tid + h * kSwThreads;
      if (t < a.n_tiles) gv[h] = a.g[t * RR + e];
    }
    if constexpr (PAIR) g[e] = L::pack(gv[0], gv[1]);
    else g[e] = gv[0];
  }
  int n_valid_out = 0;
#pragma unroll
  for (int h = 0; h < W; h++) n_valid_out += (tile0 + tid + h * kSwThreads < a.n_tiles) ? MM : 0;
  {
    // warp-level count of valid outputs (for n_scored)
    n_valid_out = __reduce_add_sync(0xffffffffu, n_valid_out);
  }
  __syncthreads();

  const int c_begin = blockIdx.y * a.cands_per_cta;
  const int c_end = min(a.n_cand, c_begin + a.cands_per_cta);
  for (int s = c_begin; s < c_end; s++) {
    const float* cm = P.v + s * PER;
    // T2 = Bᵀ d, column by column (d column q from smem), staged to smem
#pragma unroll
    for (int q = 0; q < N; q++) {
      T dc[N];
#pragma unroll
      for (int j = 0; j < N; j++) dc[j] = sd[(j * N + q) * kSwThreads + tid];
#pragma unroll
      for (int i = 0; i < N; i++) {
        T acc = L::zero();
#pragma unroll
        for (int j = 0; j < N; j++) acc = L::fma(dc[j], cm[OFF_B + i * N + j], acc);
        st2[(i * N + q) * kSwThreads + tid] = acc;
      }
    }
    T t3[M][N];
#pragma unroll
    for (int p = 0; p < M; p++)
#pragma unroll
      for (int l = 0; l < N; l++) t3[p][l] = L::zero();
#pragma unroll
    for (int i = 0; i < N; i++) {
      // U row i = (G g Gᵀ)[i,:]:  T1[i][q] = Σ_j G[i][j] g[j][q];  U[i][l] = Σ_q T1[i][q] G[l][q]
      T t1[R];
#pragma unroll
      for (int q = 0; q < R; q++) {
        T acc = L::zero();
#pragma unroll
        for (int j = 0; j < R; j++) acc = L::fma(g[j * R + q], cm[OFF_G + i * R + j], acc);
        t1[q] = acc;
      }
      T t2r[N];
#pragma unroll
      for (int q = 0; q < N; q++) t2r[q] = st2[(i * N + q) * kSwThreads + tid];
#pragma unroll
      for (int l = 0; l < N; l++) {
        T u = L::zero();
#pragma unroll
        for (int q = 0; q < R; q++) u = L::fma(t1[q], cm[OFF_G + l * R + q], u);
        // V[i][l] = Σ_q T2[i][q] Bᵀ[l][q]
        T v = L::zero();
#pragma unroll
        for (int q = 0; q < N; q++) v = L::fma(t2r[q], cm[OFF_B + l * N + q], v);
        const T mw = L::mul(u, v);
        // T3[p][l] += Aᵀ[p][i] Mw[i][l]  (ascending i, from +0)
#pragma unroll
        for (int p = 0; p < M; p++) t3[p][l] = L::fma(mw, cm[p * N + i], t3[p][l]);
      }
    }
    // Y[p][s] = Σ_l T3[p][l] Aᵀ[s][l]; score or dump
    Stat st;
#pragma unroll
    for (int p = 0; p < M; p++) {
#pragma unroll
      for (int q = 0; q < M; q++) {
        T y = L::zero();
#pragma unroll
        for (int l = 0; l < N; l++) y = L::fma(t3[p][l], cm[q * N + l], y);
        const int o = p * M + q;
#pragma unroll
        for (int h = 0; h < W; h++) {
          if (DUMP) {
            const long long t = tile0 + tid + h * kSwThreads;
            if (t < a.n_tiles) a.ydump[((long long)DI.idx[s] * a.n_tiles + t) * MM + o] = L::get(y, h);
          } else {
            st.add(L::get(y, h), sy[(o * W + h) * kSwThreads + tid]);
          }
        }
      }
    }
    if (!DUMP) {
      st.warp_reduce();
      if ((tid & 31) == 0) {
        double* pp = a.partial + (((long long)s * a.n_tblk + blockIdx.x) * 4 + warp) * 8;
        write_partial(pp, st, n_valid_out);
      }
    }
  }
}

// ------------------------------------------------------------------ K7 (1D)
// KP pairs (of W tiles) per thread; everything in registers.
template <int M, int R, bool PAIR, bool NOFMA, bool DUMP>
__global__ void __launch_bounds__(kSwThreads) sweep1d_kernel(SweepArgs a, const __grid_constant__ MatsParam P,
                                                             const __grid_constant__ IdxParam DI) {
  using L = Lane<PAIR, NOFMA>;
  using T = typename L::T;
  constexpr int W = L::W;
  constexpr int N = M + R - 1;
  constexpr int OFF_G = M * N, OFF_B = M * N + N * R, PER = OFF_B + N * N;
  constexpr int TPB = kSwThreads * W;

  const int tid = threadIdx.x, warp = tid >> 5;
  const long long tile0 = (long long)blockIdx.x * TPB;
  T d[N], g[R];
  double y64[W][M];
  int n_valid_out = 0;
  {
    float dv[W][N], gv[W][R];
#pragma unroll
    for (int h = 0; h < W; h++) {
      const long long t = tile0 + tid + h * kSwThreads;
      const bool ok = t < a.n_tiles;
      n_valid_out += ok ? M : 0;
#pragma unroll
      for (int j = 0; j < N; j++) dv[h][j] = ok ? a.d[t * N + j] : 0.0f;
#pragma unroll
      for (int j = 0; j < R; j++) gv[h][j] = ok ? a.g[t * R + j] : 0.0f;
#pragma unroll
      for (int j = 0; j < M; j++) y64[h][j] = (ok && !DUMP) ? a.y64[t * M + j] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < N; j++) {
      if constexpr (PAIR) d[j] = L::pack(dv[0][j], dv[W - 1][j]);
      else d[j] = dv[0][j];
    }
#pragma unroll
    for (int j = 0; j < R; j++) {
      if constexpr (PAIR) g[j] = L::pack(gv[0][j], gv[W - 1][j]);
      else g[j] = gv[0][j];
    }
  }
  n_valid_out = __reduce_add_sync(0xffffffffu, n_valid_out);

  const int c_begin = blockIdx.y * a.cands_per_cta;
  const int c_end = min(a.n_cand, c_begin + a.cands_per_cta);
  for (int s = c_begin; s < c_end; s++) {
    const float* cm = P.v + s * PER;
    T mw[N];
#pragma unroll
    for (int i = 0; i < N; i++) {
      T u = L::zero(), v = L::zero();
#pragma unroll
      for (int j = 0; j < R; j++) u = L::fma(g[j], cm[OFF_G + i * R + j], u);
#pragma unroll
      for (int j = 0; j < N; j++) v = L::fma(d[j], cm[OFF_B + i * N + j], v);
      mw[i] = L::mul(u, v);
    }
    Stat st;
#pragma unroll
    for (int p = 0; p < M; p++) {
      T y = L::zero();
#pragma unroll
      for (int i = 0; i < N; i++) y = L::fma(mw[i], cm[p * N + i], y);
#pragma unroll
      for (int h = 0; h < W; h++) {
        if (DUMP) {
          const long long t = tile0 + tid + h * kSwThreads;
          if (t < a.n_tiles) a.ydump[((long long)DI.idx[s] * a.n_tiles + t) * M + p] = L::get(y, h);
        } else {
          st.add(L::get(y, h), y64[h][p]);
        }
      }
    }
    if (!DUMP) {
      st.warp_reduce();
      if ((tid & 31) == 0) {
        double* pp = a.partial + (((long long)s * a.n_tblk + blockIdx.x) * 4 + warp) * 8;
        write_partial(pp, st, n_valid_out);
      }
    }
  }
}

// ------------------------------------------------------------------ K8: finalize
// One warp per candidate: lane l sums entries l, l+32, ... in order, then a butterfly.
__global__ void sweep_finalize_kernel(const double* __restrict__ partial, int n_entries, int n_cand,
                                      const __grid_constant__ IdxParam DI, double* __restrict__ d_sums,
                                      double* __restrict__ d_maxs) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n_cand) return;
  const double* p = partial + (long long)warp * n_entries * 8;
  double v[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int e = lane; e < n_entries; e += 32) {
    const double* q = p + (long long)e * 8;
#pragma unroll
    for (int f = 0; f < 5; f++) v[f] += q[f];
    v[5] = fmax(v[5], q[5]);
    v[6] = fmax(v[6], q[6]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int f = 0; f < 5; f++) v[f] += __shfl_xor_sync(0xffffffffu, v[f], o);
    v[5] = fmax(v[5], __shfl_xor_sync(0xffffffffu, v[5], o));
    v[6] = fmax(v[6], __shfl_xor_sync(0xffffffffu, v[6], o));
  }
  if (lane == 0) {
    const int c = DI.idx[warp];
    double* su = d_sums + (long long)c * WINO_SUMS;
    double* mx = d_maxs + (long long)c * WINO_MAXS;
    for (int f = 0; f < 5; f++) su[f] += v[f];
    mx[0] = fmax(mx[0], v[5]);
    mx[1] = fmax(mx[1], v[6]);
  }
}

// ------------------------------------------------------------------ dispatch
namespace {

typedef void (*SweepKernel)(SweepArgs, MatsParam, IdxParam);

struct SweepCfg {
  int dims, m, r;
  bool pair;
  SweepKernel k[2][2];   // [nofma][dump]
  void (*refs)(const float*, const float*, double*, long long);
};

template <int DIMS, int M, int R, bool PAIR>
SweepCfg make_cfg() {
  SweepCfg c;
  c.dims = DIMS;
  c.m = M;
  c.r = R;
  c.pair = PAIR;
  if constexpr (DIMS == 1) {
    c.k[0][0] = (SweepKernel)sweep1d_kernel<M, R, PAIR, false, false>;
    c.k[0][1] = (SweepKernel)sweep1d_kernel<M, R, PAIR, false, true>;
    c.k[1][0] = (SweepKernel)sweep1d_kernel<M, R, PAIR, true, false>;
    c.k[1][1] = (SweepKernel)sweep1d_kernel<M, R, PAIR, true, true>;
  } else {
    c.k[0][0] = (SweepKernel)sweep2d_kernel<M, R, PAIR, false, false>;
    c.k[0][1] = (SweepKernel)sweep2d_kernel<M, R, PAIR, false, true>;
    c.k[1][0] = (SweepKernel)sweep2d_kernel<M, R, PAIR, true, false>;
    c.k[1][1] = (SweepKernel)sweep2d_kernel<M, R, PAIR, true, true>;
  }
  c.refs = sweep_refs_kernel<DIMS, M, R>;
  return c;
}

const std::vector<SweepCfg>& cfgs() {
  static const std::vector<SweepCfg> v = {
      make_cfg<1, 1, 2, true>(), make_cfg<1, 2, 3, true>(), make_cfg<1, 3, 3, true>(),
      make_cfg<1, 4, 3, true>(), make_cfg<1, 5, 3, true>(), make_cfg<1, 6, 3, true>(),
      make_cfg<1, 7, 3, true>(), make_cfg<1, 8, 3, true>(), make_cfg<1, 4, 5, true>(),
      make_cfg<1, 6, 5, true>(),
      make_cfg<2, 1, 2, true>(), make_cfg<2, 2, 3, true>(), make_cfg<2, 3, 3, true>(),
      make_cfg<2, 4, 3, true>(), make_cfg<2, 5, 3, true>(), make_cfg<2, 6, 3, true>(),
      make_cfg<2, 4, 5, true>(), make_cfg<2, 6, 5, false>(), make_cfg<2, 7, 3, false>(),
      make_cfg<2, 8, 3, false>(),
  };
  return v;
}

const SweepCfg* find_cfg(int dims, int m, int r) {
  for (const auto& c : cfgs())
    if (c.dims == dims && c.m == m && c.r == r) return &c;
  return nullptr;
}

int per_cand(int m, int r) {
  const int n = m + r - 1;
  return m * n + n * r + n * n;
}

size_t smem_bytes(const SweepCfg& c) {
  if (c.dims == 1) return 0;
  const int n = c.m + c.r - 1, W = c.pair ? 2 : 1;
  return (size_t)2 * n * n * kSwThreads * 4 * W + (size_t)c.m * c.m * W * kSwThreads * 8;
}

long long n_tblk_of(const SweepCfg& c, int64_t n_tiles) {
  const int tpb = kSwThreads * (c.pair ? 2 : 1);
  return (n_tiles + tpb - 1) / tpb;
}

}  // namespace

int sweep_supported(int dims, int m, int r) { return find_cfg(dims, m, r) != nullptr; }

int sweep_max_cands_per_launch(int dims, int m, int r) {
  (void)dims;
  int c = kParamFloats / per_cand(m, r);
  return c < kMaxCandsLaunch ? c : kMaxCandsLaunch;
}

size_t sweep_workspace_bytes(int dims, int m, int r, int n_cand, int64_t n_tiles) {
  const SweepCfg* c = find_cfg(dims, m, r);
  if (!c) return 0;
  const int dy = dims == 1 ? m : m * m;
  const int cmax = std::min(n_cand, sweep_max_cands_per_launch(dims, m, r));
  size_t b = align_up((size_t)(n_tiles > 0 ? n_tiles : 1) * dy * sizeof(double), 256);
  b += align_up((size_t)(cmax > 0 ? cmax : 1) * n_tblk_of(*c, n_tiles) * 4 * 8 * sizeof(double), 256);
  return b;
}

int sweep_launch(int dims, int m, int r, const float* mats, const int* cand_ok, int n_cand,
                 const float* d_tiles, const float* g_tiles, int64_t n_tiles,
                 double* d_sums, double* d_maxs, float* d_y, void* workspace, size_t ws_bytes,
                 unsigned flags, cudaStream_t stream) {
  const SweepCfg* c = find_cfg(dims, m, r);
  if (!c) return set_error(WINO_E_UNSUPPORTED, "no sweep kernel for dims=%d m=%d r=%d", dims, m, r);
  const bool dump = d_y != nullptr;
  const int nofma = (flags & WINO_SWEEP_NOFMA) ? 1 : 0;
  const int per = per_cand(m, r);
  const int cmax = sweep_max_cands_per_launch(dims, m, r);
  const int dy = dims == 1 ? m : m * m;
  const long long n_tblk = n_tiles > 0 ? n_tblk_of(*c, n_tiles) : 0;
  if (n_tiles <= 0 || n_cand <= 0) return WINO_OK;

  double* y64 = nullptr;
  double* partial = nullptr;
  if (!dump) {
    const size_t need = sweep_workspace_bytes(dims, m, r, n_cand, n_tiles);
    if (!workspace || ws_bytes < need)
      return set_error(WINO_E_WORKSPACE, "sweep workspace %zu < %zu bytes", ws_bytes, need);
    y64 = reinterpret_cast<double*>(workspace);
    partial = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) +
                                        align_up((size_t)n_tiles * dy * sizeof(double), 256));
  }
  const size_t smem = smem_bytes(*c);
  SweepKernel kern = c->k[nofma][dump ? 1 : 0];
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_error(WINO_E_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  int launches = 0;
  if (!dump) {
    const int tpb = 256;
    c->refs<<<(unsigned)((n_tiles + tpb - 1) / tpb), tpb, 0, stream>>>(d_tiles, g_tiles, y64, (long long)n_tiles);
    launches++;
  }
  // candidate groups per CTA: aim for >= ~4 waves of CTAs per launch
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);

  MatsParam* P = new MatsParam;
  IdxParam* DI = new IdxParam;
  int i = 0;
  int status = WINO_OK;
  while (i < n_cand) {
    int nc = 0;
    while (i < n_cand && nc < cmax) {
      if (cand_ok[i]) {
        std::copy(mats + (size_t)i * per, mats + (size_t)(i + 1) * per, P->v + nc * per);
        DI->idx[nc] = i;
        nc++;
      }
      i++;
    }
    if (nc == 0) break;
    const long long want_ctas = 4LL * nsm * 2;
    int groups = (int)std::max(1LL, std::min<long long>(nc, (want_ctas + n_tblk - 1) / n_tblk));
    int cpc = (nc + groups - 1) / groups;
    groups = (nc + cpc - 1) / cpc;
    SweepArgs args;
    args.d = d_tiles;
    args.g = g_tiles;
    args.y64 = y64;
    args.ydump = d_y;
    args.partial = partial;
    args.n_tiles = (long long)n_tiles;
    args.n_cand = nc;
    args.cands_per_cta = cpc;
    args.n_tblk = (int)n_tblk;
    args.ydump_cand0 = 0;
    dim3 grid((unsigned)n_tblk, (unsigned)groups);
    kern<<<grid, kSwThreads, smem, stream>>>(args, *P, *DI);
    launches++;
    if (!dump) {
      const int threads = 256;
      const int blocks = (nc * 32 + threads - 1) / threads;
      sweep_finalize_kernel<<<blocks, threads, 0, stream>>>(partial, (int)(n_tblk * 4), nc, *DI, d_sums, d_maxs);
      launches++;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      status = set_error(WINO_E_CUDA, "sweep launch: %s", cudaGetErrorString(e));
      break;
    }
  }
  delete P;
  delete DI;
  count_launches(launches);
  return status;
}

}  // namespace wino
