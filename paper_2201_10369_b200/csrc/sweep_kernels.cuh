// Sweep kernel templates (K7) and their registry types; included by sweep.cu and the
// sweep_inst_*.cu translation units, which instantiate disjoint sets of kernels in
// parallel compilation units.  See sweep.cu for the design notes.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "wino_internal.h"

namespace wino {
typedef unsigned long long u64;

constexpr int kSwThreads = 128;        // 4 warps, one per SM sub-partition
constexpr int kParamFloats = 7424;     // coefficient floats per launch (29696 B)
constexpr int kMaxCandsLaunch = 512;   // + 2 KB of candidate indices: < 32764 B of params
constexpr int kMaxCpc = 32;            // candidates per CTA (smem accumulators)
constexpr int kPartial = 4;            // doubles per partial: s0, s1, m0, nonfin

struct __align__(16) MatsParam {
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
  double* partial;     // [n_cand_total][n_tgroups][kPartial], indexed by global candidate
  long long n_tiles;
  int n_cand;          // candidates in this launch
  int cands_per_cta;
  int n_tblk;          // tile blocks (kSwThreads * W tiles each)
  int tblk_per_cta;    // tile blocks per work item (a tile group)
  int n_tgroups;
  int n_cgroups;       // candidate groups in this launch; work items = n_cgroups * n_tgroups
};

// ------------------------------------------------------------------ lane arithmetic
// Lane<true>: two tiles per thread (FFMA2), Lane<false>: one tile (FFMA).
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

template <uint64_t MASK>
__device__ __forceinline__ constexpr bool nz(int k) {
  return ((MASK >> k) & 1ull) == 0ull;
}

// ------------------------------------------------------------------ statistics
struct Stat {
  // two independent accumulator sets (one per tile of the pair) halve the serial fp64
  // dependency chains; they are combined in a fixed order before the warp reduction
  double s0[2] = {0.0, 0.0}, s1[2] = {0.0, 0.0}, m0[2] = {0.0, 0.0};
  int nonfin = 0;
  // fast path: no finiteness test (a non-finite e makes s0 non-finite -> careful re-run)
  template <int K>
  __device__ __forceinline__ void add_fast(float y32, double y64) {
    const double e = (double)y32 - y64;
    const double ae = fabs(e);
    s0[K] += ae;
    s1[K] = __fma_rn(e, e, s1[K]);
    m0[K] = ae > m0[K] ? ae : m0[K];
  }
  // careful path; non-finite outputs are counted per set (set 1 in the high 16 bits)
  template <int K>
  __device__ __forceinline__ void add_careful(float y32, double y64) {
    const double e = (double)y32 - y64;
    if (isfinite(e)) {
      const double ae = fabs(e);
      s0[K] += ae;
      s1[K] = __fma_rn(e, e, s1[K]);
      m0[K] = ae > m0[K] ? ae : m0[K];
    } else {
      nonfin += K ? 65536 : 1;
    }
  }
  __device__ __forceinline__ bool finite() const {
    return isfinite(s0[0]) && isfinite(s1[0]) && isfinite(s0[1]) && isfinite(s1[1]);
  }
  // combine the two sets, then a butterfly over the warp (fixed order -> deterministic);
  // the result is in s0[0], s1[0], m0[0]
  __device__ __forceinline__ void warp_reduce() {
    double a = s0[0] + s0[1], b = s1[0] + s1[1], c = m0[1] > m0[0] ? m0[1] : m0[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      const double mo = __shfl_xor_sync(0xffffffffu, c, o);
      c = mo > c ? mo : c;
    }
    s0[0] = a;
    s1[0] = b;
    m0[0] = c;
    nonfin = __reduce_add_sync(0xffffffffu, nonfin & 0xffff) + __reduce_add_sync(0xffffffffu, nonfin >> 16);
  }
};

// fp32-pair scoring for the register-resident tile-pair kernel: per output pair (the two
// tiles of the thread) e = (y32 − hi) − lo with y64 = hi + lo split into fp32 (the first
// subtraction is exact whenever y32 and hi are within a factor 2, so e carries a relative
// error <= 2^-23), |e| by clearing the sign bits, Σ|e| and Σe² as FADD2 / FFMA2 pairs,
// max|e| per half.  8 instructions per output pair instead of 14 for the fp64 path, on
// the FP32 pipe.  Per thread and candidate 16 pairs are summed in fp32 and per warp 32
// threads, then fp64 from there on: the statistics stay within ~1e-6 relative of the
// fp64 definition (tolerance of the north star: 1 %).  Non-finite values fall through to
// the exact fp64 careful path.
struct Stat32 {
  u64 s0 = 0ull, s1 = 0ull, m0 = 0ull;
  static __device__ __forceinline__ void split(u64 p, float& a, float& b) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(p));
  }
  static __device__ __forceinline__ u64 join(float a, float b) {
    u64 p;
    asm("mov.b64 %0, {%1,%2};" : "=l"(p) : "f"(a), "f"(b));
    return p;
  }
  __device__ __forceinline__ void add(u64 y, u64 hi, u64 lo) {
    u64 e, t;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(y), "l"(hi));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(e) : "l"(t), "l"(lo));
    const u64 ae = e & 0x7fffffff7fffffffull;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s0) : "l"(s0), "l"(ae));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(s1) : "l"(e), "l"(s1));
    float a0, a1, m0a, m0b;
    split(ae, a0, a1);
    split(m0, m0a, m0b);
    m0 = join(fmaxf(m0a, a0), fmaxf(m0b, a1));
  }
  __device__ __forceinline__ bool finite() const {
    float a, b, c, d;
    split(s0, a, b);
    split(s1, c, d);
    return isfinite(a) && isfinite(b) && isfinite(c) && isfinite(d);
  }
  // warp totals (fixed butterfly order) as fp64
  __device__ __forceinline__ void warp_reduce(double& r0, double& r1, double& rm) const {
    float a, b;
    split(s0, a, b);
    float v0 = a + b;
    split(s1, a, b);
    float v1 = a + b;
    split(m0, a, b);
    float vm = fmaxf(a, b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(0xffffffffu, v0, o);
      v1 += __shfl_xor_sync(0xffffffffu, v1, o);
      vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, o));
    }
    r0 = v0;
    r1 = v1;
    rm = vm;
  }
  // cheaper variant (1D kernel, where the reduction is amortised over fewer tiles): max|e|
  // >= 0 orders like its bit pattern -> one redux.sync.max.u32; the two sums share one
  // butterfly (after the xor-16 exchange lanes < 16 carry Σ|e| and lanes >= 16 Σe²).
  // Results valid in lane 0.
  __device__ __forceinline__ void warp_reduce_lane0(double& r0, double& r1, double& rm) const {
    float a, b;
    split(s0, a, b);
    const float v0 = a + b;
    split(s1, a, b);
    const float v1 = a + b;
    split(m0, a, b);
    const unsigned vm = __float_as_uint(fmaxf(a, b));
    const bool upper = (threadIdx.x & 16) != 0;
    float v = upper ? v1 : v0;
    v += __shfl_xor_sync(0xffffffffu, upper ? v0 : v1, 16);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    r0 = v;
    r1 = __shfl_sync(0xffffffffu, v, 16);
    rm = __uint_as_float(__reduce_max_sync(0xffffffffu, vm));
  }
};

// ------------------------------------------------------------------ K6: fp64 references
template <int DIMS, int M, int R>
__global__ void __launch_bounds__(256) sweep_refs_kernel(const float* __restrict__ d, const float* __restrict__ g,
                                                         double* __restrict__ y64, long long n_tiles,
                                                         double* __restrict__ ref_part) {
  constexpr int N = M + R - 1;
  constexpr int DN = DIMS == 1 ? N : N * N, DG = DIMS == 1 ? R : R * R, DY = DIMS == 1 ? M : M * M;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0, mx = 0.0;
  if (t < n_tiles) {
    const float* dt = d + t * DN;
    const float* gt = g + t * DG;
    double* yt = y64 + t * DY;
    if (DIMS == 1) {
      for (int p = 0; p < M; p++) {
        double acc = 0.0;
        for (int j = 0; j < R; j++) acc = __dadd_rn(acc, __dmul_rn((double)gt[j], (double)dt[p + j]));
        yt[p] = acc;
        s += fabs(acc);
        mx = fmax(mx, fabs(acc));
      }
    } else {
      for (int p = 0; p < M; p++)
        for (int q = 0; q < M; q++) {
          double acc = 0.0;
          for (int u = 0; u < R; u++)
            for (int v = 0; v < R; v++)
              acc = __dadd_rn(acc, __dmul_rn((double)gt[u * R + v], (double)dt[(p + u) * N + q + v]));
          yt[p * M + q] = acc;
          s += fabs(acc);
          mx = fmax(mx, fabs(acc));
        }
    }
  }
  // fixed-order block reduction: warp butterflies, then thread 0 over the 8 warp results
  __shared__ double red[2][8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s;
    red[1][threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < 8; w++) {
      a += red[0][w];
      b = fmax(b, red[1][w]);
    }
    ref_part[blockIdx.x * 2] = a;
    ref_part[blockIdx.x * 2 + 1] = b;
  }
}

// ------------------------------------------------------------------ K7 (2D)
// One candidate on this thread's tile pair; scores (or dumps) the M x M outputs.
template <int M, int R, bool PAIR, bool NOFMA, bool DUMP, bool CAREFUL, uint64_t ZA, uint64_t ZG, uint64_t ZB>
__device__ __forceinline__ void eval2d(const float* __restrict__ cm, const typename Lane<PAIR, NOFMA>::T* sd,
                                       typename Lane<PAIR, NOFMA>::T* st2, const double* sy,
                                       const typename Lane<PAIR, NOFMA>::T (&g)[R * R], int tid, Stat& st,
                                       float* ydump_tile0, long long tile0, long long n_tiles) {
  using L = Lane<PAIR, NOFMA>;
  using T = typename L::T;
  constexpr int W = L::W;
  constexpr int N = M + R - 1, MM = M * M;
  constexpr int OFF_G = M * N, OFF_B = M * N + N * R;
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
      for (int j = 0; j < N; j++)
        if (nz<ZB>(i * N + j)) acc = L::fma(dc[j], cm[OFF_B + i * N + j], acc);
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
      for (int j = 0; j < R; j++)
        if (nz<ZG>(i * R + j)) acc = L::fma(g[j * R + q], cm[OFF_G + i * R + j], acc);
      t1[q] = acc;
    }
    T t2r[N];
#pragma unroll
    for (int q = 0; q < N; q++) t2r[q] = st2[(i * N + q) * kSwThreads + tid];
#pragma unroll
    for (int l = 0; l < N; l++) {
      T u = L::zero();
#pragma unroll
      for (int q = 0; q < R; q++)
        if (nz<ZG>(l * R + q)) u = L::fma(t1[q], cm[OFF_G + l * R + q], u);
      // V[i][l] = Σ_q T2[i][q] Bᵀ[l][q]
      T v = L::zero();
#pragma unroll
      for (int q = 0; q < N; q++)
        if (nz<ZB>(l * N + q)) v = L::fma(t2r[q], cm[OFF_B + l * N + q], v);
      const T mw = L::mul(u, v);
      // T3[p][l] += Aᵀ[p][i] Mw[i][l]  (ascending i, from +0)
#pragma unroll
      for (int p = 0; p < M; p++)
        if (nz<ZA>(p * N + i)) t3[p][l] = L::fma(mw, cm[p * N + i], t3[p][l]);
    }
  }
  // Y[p][q] = Σ_l T3[p][l] Aᵀ[q][l]; score or dump
#pragma unroll
  for (int p = 0; p < M; p++) {
#pragma unroll
    for (int q = 0; q < M; q++) {
      T y = L::zero();
#pragma unroll
      for (int l = 0; l < N; l++)
        if (nz<ZA>(q * N + l)) y = L::fma(t3[p][l], cm[q * N + l], y);
      const int o = p * M + q;
#pragma unroll
      for (int h = 0; h < W; h++) {
        if (DUMP) {
          const long long t = tile0 + tid + h * kSwThreads;
          if (t < n_tiles) ydump_tile0[(tid + h * kSwThreads) * MM + o] = L::get(y, h);
        } else if (CAREFUL) {
          if (h == 0) st.template add_careful<0>(L::get(y, h), sy[(o * W + h) * kSwThreads + tid]);
          else st.template add_careful<1>(L::get(y, h), sy[(o * W + h) * kSwThreads + tid]);
        } else {
          if (h == 0) st.template add_fast<0>(L::get(y, h), sy[(o * W + h) * kSwThreads + tid]);
          else st.template add_fast<1>(L::get(y, h), sy[(o * W + h) * kSwThreads + tid]);
        }
      }
    }
  }
}

// smem: sd [NN][128] T (tiles), st2 [NN][128] T (T2 staging), sy [MM][W][128] double,
//       sacc [kMaxCpc][4 warps][kPartial] double
template <int M, int R, bool PAIR, bool NOFMA, bool DUMP, uint64_t ZA, uint64_t ZG, uint64_t ZB>
__global__ void __launch_bounds__(kSwThreads) sweep2d_kernel(SweepArgs a, const __grid_constant__ MatsParam P,
                                                             const __grid_constant__ IdxParam DI) {
  using L = Lane<PAIR, NOFMA>;
  using T = typename L::T;
  constexpr int W = L::W;
  constexpr int N = M + R - 1, NN = N * N, MM = M * M, RR = R * R;
  constexpr int PER = M * N + N * R + N * N;
  constexpr int TPB = kSwThreads * W;

  extern __shared__ __align__(16) unsigned char smem[];
  T* sd = reinterpret_cast<T*>(smem);
  T* st2 = sd + NN * kSwThreads;
  double* sy = reinterpret_cast<double*>(st2 + NN * kSwThreads);
  double* sacc = sy + MM * W * kSwThreads;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // persistent CTAs walk the (candidate group, tile group) work items round-robin
  const int n_items = a.n_cgroups * a.n_tgroups;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
  const int cg = item / a.n_tgroups, tg = item - cg * a.n_tgroups;
  const int c_begin = cg * a.cands_per_cta;
  const int c_end = min(a.n_cand, c_begin + a.cands_per_cta);
  __syncthreads();  // the previous item's accumulators are flushed
  if (!DUMP)
    for (int k = tid; k < kMaxCpc * 4 * kPartial; k += kSwThreads) sacc[k] = 0.0;

  const int tb_begin = tg * a.tblk_per_cta;
  const int tb_end = min(a.n_tblk, tb_begin + a.tblk_per_cta);
  for (int tb = tb_begin; tb < tb_end; tb++) {
    const long long tile0 = (long long)tb * TPB;
    __syncthreads();  // previous block's smem no longer in use
    // Each thread stages its own W tiles: vector loads of the contiguous tile rows, stores
    // [e][tid] (pairs as 8-byte words) -> conflict-free shared-memory writes.
    {
      bool ok[W];
#pragma unroll
      for (int h = 0; h < W; h++) ok[h] = tile0 + tid + h * kSwThreads < a.n_tiles;
      if constexpr (NN % 4 == 0) {
#pragma unroll 3
        for (int e4 = 0; e4 < NN / 4; e4++) {
          float4 v[W];
#pragma unroll
          for (int h = 0; h < W; h++)
            v[h] = ok[h] ? __ldg(reinterpret_cast<const float4*>(a.d + (tile0 + tid + h * kSwThreads) * NN) + e4)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
          if constexpr (PAIR) {
            sd[(e4 * 4 + 0) * kSwThreads + tid] = L::pack(v[0].x, v[W - 1].x);
            sd[(e4 * 4 + 1) * kSwThreads + tid] = L::pack(v[0].y, v[W - 1].y);
            sd[(e4 * 4 + 2) * kSwThreads + tid] = L::pack(v[0].z, v[W - 1].z);
            sd[(e4 * 4 + 3) * kSwThreads + tid] = L::pack(v[0].w, v[W - 1].w);
          } else {
            reinterpret_cast<float*>(sd)[(e4 * 4 + 0) * kSwThreads + tid] = v[0].x;
            reinterpret_cast<float*>(sd)[(e4 * 4 + 1) * kSwThreads + tid] = v[0].y;
            reinterpret_cast<float*>(sd)[(e4 * 4 + 2) * kSwThreads + tid] = v[0].z;
            reinterpret_cast<float*>(sd)[(e4 * 4 + 3) * kSwThreads + tid] = v[0].w;
          }
        }
      } else {
#pragma unroll 4
        for (int e = 0; e < NN; e++) {
          float v[W];
#pragma unroll
          for (int h = 0; h < W; h++) v[h] = ok[h] ? __ldg(a.d + (tile0 + tid + h * kSwThreads) * NN + e) : 0.0f;
          if constexpr (PAIR) sd[e * kSwThreads + tid] = L::pack(v[0], v[W - 1]);
          else reinterpret_cast<float*>(sd)[e * kSwThreads + tid] = v[0];
        }
      }
      if (!DUMP) {
#pragma unroll
        for (int h = 0; h < W; h++) {
          const double* ysrc = a.y64 + (tile0 + tid + h * kSwThreads) * MM;
          if constexpr (MM % 2 == 0) {
#pragma unroll 4
            for (int o2 = 0; o2 < MM / 2; o2++) {
              const double2 v = ok[h] ? __ldg(reinterpret_cast<const double2*>(ysrc) + o2) : make_double2(0.0, 0.0);
              sy[((2 * o2) * W + h) * kSwThreads + tid] = v.x;
              sy[((2 * o2 + 1) * W + h) * kSwThreads + tid] = v.y;
            }
          } else {
#pragma unroll 4
            for (int o = 0; o < MM; o++) sy[(o * W + h) * kSwThreads + tid] = ok[h] ? __ldg(ysrc + o) : 0.0;
          }
        }
      }
    }
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
    __syncthreads();

    for (int s = c_begin; s < c_end; s++) {
      const float* cm = P.v + s * PER;
      Stat st;
      float* yd = DUMP ? a.ydump + ((long long)DI.idx[s] * a.n_tiles + tile0) * MM : nullptr;
      eval2d<M, R, PAIR, NOFMA, DUMP, false, ZA, ZG, ZB>(cm, sd, st2, sy, g, tid, st, yd, tile0, a.n_tiles);
      if (!DUMP) {
        if (__any_sync(0xffffffffu, !st.finite())) {
          st = Stat();
          eval2d<M, R, PAIR, NOFMA, false, true, ZA, ZG, ZB>(cm, sd, st2, sy, g, tid, st, nullptr, tile0, a.n_tiles);
        }
        st.warp_reduce();
        if (lane == 0) {
          double* acc = sacc + ((s - c_begin) * 4 + warp) * kPartial;
          acc[0] += st.s0[0];
          acc[1] += st.s1[0];
          acc[2] = st.m0[0] > acc[2] ? st.m0[0] : acc[2];
          acc[3] += (double)st.nonfin;
        }
      }
    }
  }
  if (!DUMP) {
    __syncthreads();
    for (int s = c_begin + tid; s < c_end; s += kSwThreads) {
      double v[kPartial] = {0.0, 0.0, 0.0, 0.0};
      for (int w = 0; w < 4; w++) {
        const double* acc = sacc + ((s - c_begin) * 4 + w) * kPartial;
        v[0] += acc[0];
        v[1] += acc[1];
        v[2] = acc[2] > v[2] ? acc[2] : v[2];
        v[3] += acc[3];
      }
      double* pp = a.partial + ((long long)DI.idx[s] * a.n_tgroups + tg) * kPartial;
      for (int f = 0; f < kPartial; f++) pp[f] = v[f];
    }
  }
  }  // work items
}

// ------------------------------------------------------------------ K7 (2D, tiles in registers)
// Variant of the tile-pair kernel for small n: the thread's two tiles d stay in registers
// and T2 is formed row by row from them (T2[i][q] = Σ_j Bᵀ[i][j] d[j][q], ascending j), so
// no candidate-dependent data touches shared memory; only y64 is staged.  Same chains.
template <int M, int R, bool PAIR, bool NOFMA, bool DUMP, bool CAREFUL, uint64_t ZA, uint64_t ZG, uint64_t ZB>
__device__ __forceinline__ void eval2d_r(const float* __restrict__ cm,
                                         const typename Lane<PAIR, NOFMA>::T (&d)[(M + R - 1) * (M + R - 1)],
                                         const typename Lane<PAIR, NOFMA>::T (&g)[R * R], const u64* syh,
                                         const u64* syl, int tid, Stat& st, Stat32& st32, float* ydump_tile0,
                                         long long tile0, long long n_tiles) {
  using L = Lane<PAIR, NOFMA>;
  using T = typename L::T;
  constexpr int W = L::W;
  constexpr int N = M + R - 1, MM = M * M;
  constexpr int OFF_G = M * N, OFF_B = M * N + N * R;
  T t3[M][N];
#pragma unroll
  for (int p = 0; p < M; p++)
#pragma unroll
    for (int l = 0; l < N; l++) t3[p][l] = L::zero();
#pragma unroll
  for (int i = 0; i < N; i++) {
    T t1[R];
#pragma unroll
    for (int q = 0; q < R; q++) {
      T acc = L::zero();
#pragma unroll
      for (int j = 0; j < R; j++)
        if (nz<ZG>(i * R + j)) acc = L::fma(g[j * R + q], cm[OFF_G + i * R + j], acc);
      t1[q] = acc;
    }
    T t2r[N];
#pragma unroll
    for (int q = 0; q < N; q++) {
      T acc = L::zero();
#pragma unroll
      for (int j = 0; j < N; j++)
        if (nz<ZB>(i * N + j)) acc = L::fma(d[j * N + q], cm[OFF_B + i * N + j], acc);
      t2r[q] = acc;
    }
#pragma unroll
    for (int l = 0; l < N; l++) {
      T u = L::zero();
#pragma unroll
      for (int q = 0; q < R; q++)
        if (nz<ZG>(l * R + q)) u = L::fma(t1[q], cm[OFF_G + l * R + q], u);
      T v = L::zero();
#pragma unroll
      for (int q = 0; q < N; q++)
        if (nz<ZB>(l * N + q)) v = L::fma(t2r[q], cm[OFF_B + l * N + q], v);
      const T mw = L::mul(u, v);
#pragma unroll
      for (int p = 0; p < M; p++)
        if (nz<ZA>(p * N + i)) t3[p][l] = L::fma(mw, cm[p * N + i], t3[p][l]);
    }
  }
#pragma unroll
  for (int p = 0; p < M; p++) {
#pragma unroll
    for (int q = 0; q < M; q++) {
      T y = L::zero();
#pragma unroll
      for (int l = 0; l < N; l++)
        if (nz<ZA>(q * N + l)) y = L::fma(t3[p][l], cm[q * N + l], y);
      const int o = p * M + q;
      if (DUMP) {
#pragma unroll
        for (int h = 0; h < W; h++) {
          const long long t = tile0 + tid + h * kSwThreads;
          if (t < n_tiles) ydump_tile0[(tid + h * kSwThreads) * MM + o] = L::get(y, h);
        }
      } else if (CAREFUL) {
        // exact fp64 path on y64 = hi + lo (the split is exact in fp64 to 2^-48 relative)
        const u64 hp = syh[o * kSwThreads + tid], lp = syl[o * kSwThreads + tid];
        float h0, h1, l0, l1;
        Stat32::split(hp, h0, h1);
        Stat32::split(lp, l0, l1);
        st.template add_careful<0>(L::get(y, 0), (double)h0 + (double)l0);
        st.template add_careful<1>(L::get(y, 1), (double)h1 + (double)l1);
      } else {
        st32.add(y, syh[o * kSwThreads + tid], syl[o * kSwThreads + tid]);
      }
    }
  }
}

// smem: sy [MM][W][128] double, sacc [kMaxCpc][4 warps][kPartial] double
template <int M, int R, bool PAIR, bool NOFMA, bool DUMP, uint64_t ZA, uint64_t ZG, uint64_t ZB>
__global__ void __launch_bounds__(kSwThreads) sweep2d_reg_kernel(SweepArgs a, const __grid_constant__ MatsParam P,
                                                                 const __grid_constant__ IdxParam DI) {
  using L = Lane<PAIR, NOFMA>;
  using T = typename L::T;
  constexpr int W = L::W;
  constexpr int N = M + R - 1, NN = N * N, MM = M * M, RR = R * R;
  constexpr int PER = M * N + N * R + N * N;
  constexpr int TPB = kSwThreads * W;
  static_assert(PAIR, "sweep2d_reg_kernel evaluates tile pairs");
  extern __shared__ __align__(16) unsigned char smem[];
  u64* syh = reinterpret_cast<u64*>(smem);            // [MM][128] (hi_A, hi_B)
  u64* syl = syh + MM * kSwThreads;                    // [MM][128] (lo_A, lo_B)
  double* sacc = reinterpret_cast<double*>(syl + MM * kSwThreads);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = a.n_cgroups * a.n_tgroups;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int cg = item / a.n_tgroups, tg = item - cg * a.n_tgroups;
    const int c_begin = cg * a.cands_per_cta;
    const int c_end = min(a.n_cand, c_begin + a.cands_per_cta);
    __syncthreads();  // the previous item's accumulators are flushed
    if (!DUMP)
      for (int k = tid; k < kMaxCpc * 4 * kPartial; k += kSwThreads) sacc[k] = 0.0;
    const int tb_begin = tg * a.tblk_per_cta;
    const int tb_end = min(a.n_tblk, tb_begin + a.tblk_per_cta);
    for (int tb = tb_begin; tb < tb_end; tb++) {
      const long long tile0 = (long long)tb * TPB;
      bool ok[W];
#pragma unroll
      for (int h = 0; h < W; h++) ok[h] = tile0 + tid + h * kSwThreads < a.n_tiles;
      T d[NN], g[RR];
#pragma unroll
      for (int e = 0; e < NN; e++) {
        float v[2] = {0.0f, 0.0f};
#pragma unroll
        for (int h = 0; h < W; h++)
          if (ok[h]) v[h] = __ldg(a.d + (tile0 + tid + h * kSwThreads) * NN + e);
        if constexpr (PAIR) d[e] = L::pack(v[0], v[1]);
        else d[e] = v[0];
      }
#pragma unroll
      for (int e = 0; e < RR; e++) {
        float v[2] = {0.0f, 0.0f};
#pragma unroll
        for (int h = 0; h < W; h++)
          if (ok[h]) v[h] = __ldg(a.g + (tile0 + tid + h * kSwThreads) * RR + e);
        if constexpr (PAIR) g[e] = L::pack(v[0], v[1]);
        else g[e] = v[0];
      }
      // each thread stages (and later reads) only its own y64 slots: no barrier needed
      if (!DUMP) {
#pragma unroll 4
        for (int o = 0; o < MM; o++) {
          float hi[2], lo[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const double v = ok[h] ? __ldg(a.y64 + (tile0 + tid + h * kSwThreads) * MM + o) : 0.0;
            hi[h] = __double2float_rn(v);
            lo[h] = __double2float_rn(v - (double)hi[h]);
          }
          syh[o * kSwThreads + tid] = Stat32::join(hi[0], hi[1]);
          syl[o * kSwThreads + tid] = Stat32::join(lo[0], lo[1]);
        }
      }
      for (int s = c_begin; s < c_end; s++) {
        const float* cm = P.v + s * PER;
        Stat st;
        Stat32 st32;
        float* yd = DUMP ? a.ydump + ((long long)DI.idx[s] * a.n_tiles + tile0) * MM : nullptr;
        eval2d_r<M, R, PAIR, NOFMA, DUMP, false, ZA, ZG, ZB>(cm, d, g, syh, syl, tid, st, st32, yd, tile0,
                                                            a.n_tiles);
        if (!DUMP) {
          double r0, r1, rm, rn = 0.0;
          if (__any_sync(0xffffffffu, !st32.finite())) {
            eval2d_r<M, R, PAIR, NOFMA, false, true, ZA, ZG, ZB>(cm, d, g, syh, syl, tid, st, st32, nullptr, tile0,
                                                                a.n_tiles);
            st.warp_reduce();
            r0 = st.s0[0];
            r1 = st.s1[0];
            rm = st.m0[0];
            rn = (double)st.nonfin;
          } else {
            st32.warp_reduce(r0, r1, rm);
          }
          if (lane == 0) {
            double* acc = sacc + ((s - c_begin) * 4 + warp) * kPartial;
            acc[0] += r0;
            acc[1] += r1;
            acc[2] = rm > acc[2] ? rm : acc[2];
            acc[3] += rn;
          }
        }
      }
    }
    if (!DUMP) {
      __syncthreads();
      for (int s = c_begin + tid; s < c_end; s += kSwThreads) {
        double v[kPartial] = {0.0, 0.0, 0.0, 0.0};
        for (int w = 0; w < 4; w++) {
          const double* acc = sacc + ((s - c_begin) * 4 + w) * kPartial;
          v[0] += acc[0];
          v[1] += acc[1];
          v[2] = acc[2] > v[2] ? acc[2] : v[2];
          v[3] += acc[3];
        }
        double* pp = a.partial + ((long long)DI.idx[s] * a.n_tgroups + tg) * kPartial;
        for (int f = 0; f < kPartial; f++) pp[f] = v[f];
      }
    }
  }
}

// ------------------------------------------------------------------ K7 (1D)
// Tile pairs in registers; scoring as in the register-resident 2D kernel: fp32 pairs
// (Stat32) on y64 = hi + lo, exact fp64 careful path for non-finite outputs.
template <int M, int R, bool PAIR, bool NOFMA, bool DUMP, bool CAREFUL, uint64_t ZA, uint64_t ZG, uint64_t ZB>
__device__ __forceinline__ void eval1d(const float* __restrict__ cm, const typename Lane<PAIR, NOFMA>::T (&d)[M + R - 1],
                                       const typename Lane<PAIR, NOFMA>::T (&g)[R], const u64 (&yh)[M],
                                       const u64 (&yl)[M], Stat& st, Stat32& st32, float* yd, long long tile0,
                                       long long n_tiles, int tid) {
  using L = Lane<PAIR, NOFMA>;
  using T = typename L::T;
  constexpr int W = L::W;
  constexpr int N = M + R - 1;
  constexpr int OFF_G = M * N, OFF_B = M * N + N * R;
  T mw[N];
#pragma unroll
  for (int i = 0; i < N; i++) {
    T u = L::zero(), v = L::zero();
#pragma unroll
    for (int j = 0; j < R; j++)
      if (nz<ZG>(i * R + j)) u = L::fma(g[j], cm[OFF_G + i * R + j], u);
#pragma unroll
    for (int j = 0; j < N; j++)
      if (nz<ZB>(i * N + j)) v = L::fma(d[j], cm[OFF_B + i * N + j], v);
    mw[i] = L::mul(u, v);
  }
#pragma unroll
  for (int p = 0; p < M; p++) {
    T y = L::zero();
#pragma unroll
    for (int i = 0; i < N; i++)
      if (nz<ZA>(p * N + i)) y = L::fma(mw[i], cm[p * N + i], y);
    if (DUMP) {
#pragma unroll
      for (int h = 0; h < W; h++) {
        const long long t = tile0 + tid + h * kSwThreads;
        if (t < n_tiles) yd[(tid + h * kSwThreads) * M + p] = L::get(y, h);
      }
    } else if (CAREFUL) {
      float h0, h1, l0, l1;
      Stat32::split(yh[p], h0, h1);
      Stat32::split(yl[p], l0, l1);
      st.template add_careful<0>(L::get(y, 0), (double)h0 + (double)l0);
      st.template add_careful<1>(L::get(y, 1), (double)h1 + (double)l1);
    } else {
      st32.add(y, yh[p], yl[p]);
    }
  }
}

// Everything in registers; a CTA walks its tile blocks and, per block, its candidates.
// Each thread owns kKP1 pairs of tiles, so a candidate's coefficients (uniform registers)
// and its warp reduction are amortised over 2 * kKP1 tile evaluations.
constexpr int kKP1 = 4;

template <int M, int R, bool PAIR, bool NOFMA, bool DUMP, uint64_t ZA, uint64_t ZG, uint64_t ZB>
__global__ void __launch_bounds__(kSwThreads) sweep1d_kernel(SweepArgs a, const __grid_constant__ MatsParam P,
                                                             const __grid_constant__ IdxParam DI) {
  using L = Lane<PAIR, NOFMA>;
  using T = typename L::T;
  static_assert(PAIR, "sweep1d_kernel evaluates tile pairs");
  constexpr int W = L::W;
  constexpr int N = M + R - 1;
  constexpr int PER = M * N + N * R + N * N;
  constexpr int TPB = kSwThreads * W * kKP1;
  __shared__ double sacc[kMaxCpc * 4 * kPartial];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // persistent CTAs walk the (candidate group, tile group) work items round-robin
  const int n_items = a.n_cgroups * a.n_tgroups;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
  const int cg = item / a.n_tgroups, tg = item - cg * a.n_tgroups;
  const int c_begin = cg * a.cands_per_cta;
  const int c_end = min(a.n_cand, c_begin + a.cands_per_cta);
  __syncthreads();  // the previous item's accumulators are flushed
  if (!DUMP)
    for (int k = tid; k < kMaxCpc * 4 * kPartial; k += kSwThreads) sacc[k] = 0.0;
  __syncthreads();

  const int tb_begin = tg * a.tblk_per_cta;
  const int tb_end = min(a.n_tblk, tb_begin + a.tblk_per_cta);
  for (int tb = tb_begin; tb < tb_end; tb++) {
    T d[kKP1][N], g[kKP1][R];
    u64 yh[kKP1][M], yl[kKP1][M];   // y64 = hi + lo as fp32 pairs (tile A, tile B)
#pragma unroll
    for (int k = 0; k < kKP1; k++) {
      const long long tk0 = (long long)tb * TPB + k * kSwThreads * W;  // tile0 of sub-block k
      float dv[2][N], gv[2][R];
#pragma unroll
      for (int h = 0; h < W; h++) {
        const long long t = tk0 + tid + h * kSwThreads;
        const bool ok = t < a.n_tiles;
#pragma unroll
        for (int j = 0; j < N; j++) dv[h][j] = ok ? __ldg(a.d + t * N + j) : 0.0f;
#pragma unroll
        for (int j = 0; j < R; j++) gv[h][j] = ok ? __ldg(a.g + t * R + j) : 0.0f;
      }
#pragma unroll
      for (int j = 0; j < M; j++) {
        float hi[2] = {0.0f, 0.0f}, lo[2] = {0.0f, 0.0f};
#pragma unroll
        for (int h = 0; h < W; h++) {
          const long long t = tk0 + tid + h * kSwThreads;
          const double v = (t < a.n_tiles && !DUMP) ? __ldg(a.y64 + t * M + j) : 0.0;
          hi[h] = __double2float_rn(v);
          lo[h] = __double2float_rn(v - (double)hi[h]);
        }
        yh[k][j] = Stat32::join(hi[0], hi[1]);
        yl[k][j] = Stat32::join(lo[0], lo[1]);
      }
#pragma unroll
      for (int j = 0; j < N; j++) {
        if constexpr (PAIR) d[k][j] = L::pack(dv[0][j], dv[W - 1][j]);
        else d[k][j] = dv[0][j];
      }
#pragma unroll
      for (int j = 0; j < R; j++) {
        if constexpr (PAIR) g[k][j] = L::pack(gv[0][j], gv[W - 1][j]);
        else g[k][j] = gv[0][j];
      }
    }
    for (int s = c_begin; s < c_end; s++) {
      const float* cm = P.v + s * PER;
      Stat st;
      Stat32 st32;
#pragma unroll
      for (int k = 0; k < kKP1; k++) {
        const long long tk0 = (long long)tb * TPB + k * kSwThreads * W;
        float* yd = DUMP ? a.ydump + ((long long)DI.idx[s] * a.n_tiles + tk0) * M : nullptr;
        eval1d<M, R, PAIR, NOFMA, DUMP, false, ZA, ZG, ZB>(cm, d[k], g[k], yh[k], yl[k], st, st32, yd, tk0,
                                                           a.n_tiles, tid);
      }
      if (!DUMP) {
        double r0, r1, rm, rn = 0.0;
        if (__any_sync(0xffffffffu, !st32.finite())) {
#pragma unroll
          for (int k = 0; k < kKP1; k++)
            eval1d<M, R, PAIR, NOFMA, false, true, ZA, ZG, ZB>(cm, d[k], g[k], yh[k], yl[k], st, st32, nullptr, 0,
                                                               a.n_tiles, tid);
          st.warp_reduce();
          r0 = st.s0[0];
          r1 = st.s1[0];
          rm = st.m0[0];
          rn = (double)st.nonfin;
        } else {
          st32.warp_reduce_lane0(r0, r1, rm);
        }
        if (lane == 0) {
          double* acc = sacc + ((s - c_begin) * 4 + warp) * kPartial;
          acc[0] += r0;
          acc[1] += r1;
          acc[2] = rm > acc[2] ? rm : acc[2];
          acc[3] += rn;
        }
      }
    }
  }
  if (!DUMP) {
    __syncthreads();
    for (int s = c_begin + tid; s < c_end; s += kSwThreads) {
      double v[kPartial] = {0.0, 0.0, 0.0, 0.0};
      for (int w = 0; w < 4; w++) {
        const double* acc = sacc + ((s - c_begin) * 4 + w) * kPartial;
        v[0] += acc[0];
        v[1] += acc[1];
        v[2] = acc[2] > v[2] ? acc[2] : v[2];
        v[3] += acc[3];
      }
      double* pp = a.partial + ((long long)DI.idx[s] * a.n_tgroups + tg) * kPartial;
      for (int f = 0; f < kPartial; f++) pp[f] = v[f];
    }
  }
  }  // work items
}

typedef void (*SweepKernel)(SweepArgs, MatsParam, IdxParam);
typedef void (*RefsKernel)(const float*, const float*, double*, long long, double*);

// Kernel layouts: TPAIR = two tiles per thread (FFMA2 lanes = tiles, coefficients per
// candidate as uniform registers); TSINGLE = one tile per thread (FFMA), for large n;
// TPAIR_REG = tile pairs held in registers (sweep2d_reg_kernel), for small n.
enum Layout { TPAIR = 0, TSINGLE = 1, TPAIR_REG = 2 };

struct Variant {
  uint64_t za, zg, zb;   // structural-zero masks the kernel skips (0 = dense)
  SweepKernel k[2][2];   // [nofma][dump]
  Layout lay[2];         // layout of k[nofma][*]
};

struct SweepCfg {
  int dims, m, r;
  Layout fma_layout;     // layout of the FMA (parity-mode) kernels
  RefsKernel refs;
  std::vector<Variant> variants;   // most specialised first, dense last
};

template <int DIMS, int M, int R, Layout LAY, uint64_t ZA, uint64_t ZG, uint64_t ZB>
Variant make_variant() {
  Variant v;
  v.za = ZA;
  v.zg = ZG;
  v.zb = ZB;
  constexpr bool PAIR = LAY != TSINGLE;
  if constexpr (DIMS == 1) {
    v.k[0][0] = (SweepKernel)sweep1d_kernel<M, R, PAIR, false, false, ZA, ZG, ZB>;
    v.k[0][1] = (SweepKernel)sweep1d_kernel<M, R, PAIR, false, true, ZA, ZG, ZB>;
    v.k[1][0] = (SweepKernel)sweep1d_kernel<M, R, PAIR, true, false, ZA, ZG, ZB>;
    v.k[1][1] = (SweepKernel)sweep1d_kernel<M, R, PAIR, true, true, ZA, ZG, ZB>;
    v.lay[0] = v.lay[1] = PAIR ? TPAIR : TSINGLE;
  } else if constexpr (LAY == TPAIR_REG) {
    v.k[0][0] = (SweepKernel)sweep2d_reg_kernel<M, R, true, false, false, ZA, ZG, ZB>;
    v.k[0][1] = (SweepKernel)sweep2d_reg_kernel<M, R, true, false, true, ZA, ZG, ZB>;
    v.k[1][0] = (SweepKernel)sweep2d_reg_kernel<M, R, true, true, false, ZA, ZG, ZB>;
    v.k[1][1] = (SweepKernel)sweep2d_reg_kernel<M, R, true, true, true, ZA, ZG, ZB>;
    v.lay[0] = v.lay[1] = TPAIR_REG;
  } else {
    v.k[0][0] = (SweepKernel)sweep2d_kernel<M, R, PAIR, false, false, ZA, ZG, ZB>;
    v.k[0][1] = (SweepKernel)sweep2d_kernel<M, R, PAIR, false, true, ZA, ZG, ZB>;
    v.k[1][0] = (SweepKernel)sweep2d_kernel<M, R, PAIR, true, false, ZA, ZG, ZB>;
    v.k[1][1] = (SweepKernel)sweep2d_kernel<M, R, PAIR, true, true, ZA, ZG, ZB>;
    v.lay[0] = v.lay[1] = PAIR ? TPAIR : TSINGLE;
  }
  return v;
}

template <int DIMS, int M, int R, Layout LAY>
SweepCfg make_cfg(std::vector<Variant> specialised = {}) {
  SweepCfg c;
  c.dims = DIMS;
  c.m = M;
  c.r = R;
  c.fma_layout = LAY;
  c.refs = sweep_refs_kernel<DIMS, M, R>;
  c.variants = specialised;
  c.variants.push_back(make_variant<DIMS, M, R, LAY, 0, 0, 0>());
  return c;
}

// Structural-zero masks of the paper's families in canonical order (bit k = row-major
// entry k of Aᵀ / G / Bᵀ is exactly 0 for every c; generated from oracle R64 over the
// configs[1] grid, re-checked at run time per chunk and by tests/test_abi.py):
//   {0, ±c, ±1/c, ∞}, F(4,3):  Aᵀ 0x124920, G 0x18180, Bᵀ 0x56186a861   (570 of 834 FMAs)
//   {0, ±c, ∞},       F(2,3):  Aᵀ 0x28,     G 0x630,   Bᵀ 0x59a9
inline constexpr uint64_t kF43A = 0x124920ull, kF43G = 0x18180ull, kF43B = 0x56186a861ull;
inline constexpr uint64_t kF23A = 0x28ull, kF23G = 0x630ull, kF23B = 0x59a9ull;


// Huffman-order (sweep_huff.cuh) and mixed-precision (sweep_mixed.cuh) sweep kernels, [dump]
struct HuffCfg {
  int dims, m, r;
  SweepKernel k[2];
};

// per-translation-unit registries (sweep_inst_*.cu)
std::vector<SweepCfg> sweep_cfgs_1d();
std::vector<SweepCfg> sweep_cfgs_1d_large();
std::vector<SweepCfg> sweep_cfgs_2d_f43();
std::vector<SweepCfg> sweep_cfgs_2d_small();
std::vector<SweepCfg> sweep_cfgs_2d_large();
std::vector<HuffCfg> sweep_huff_cfgs();
std::vector<HuffCfg> sweep_mixed_cfgs();

}  // namespace wino
