// Sweep kernel templates (K6-K7) and their registry types; included by sweep.cu and the
// sweep_inst_*.cu translation units, which instantiate disjoint sets of kernels in
// parallel compilation units.  See sweep.cu for the design notes.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "wino_internal.h"
#include "zero_masks.h"
#include "sweep_dev.cuh"

namespace wino {
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

__device__ __forceinline__ u64 pack2(float a, float b) {
  u64 p;
  asm("mov.b64 %0, {%1,%2};" : "=l"(p) : "f"(a), "f"(b));
  return p;
}
__device__ __forceinline__ void split2(u64 p, float& a, float& b) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(p));
}

// fp32-pair scoring of the register-resident tile-pair kernels: per output pair (the two
// tiles of the thread) e = (y32 − hi) − lo with y64 = hi + lo split into fp32 (the first
// subtraction is exact whenever y32 and hi are within a factor 2, so e carries a relative
// error <= 2^-23), |e| by clearing the sign bits, Σ|e| and Σe² as FADD2 / FFMA2, max|e|
// per half.  Per thread the pair halves are folded once per candidate and tile block and
// accumulated in fp32 in shared memory (<= 32 x tile blocks per work item terms); the
// cross-thread reduction is fp64 in a fixed order.  The statistics stay within ~1e-6
// relative of the fp64 definition (tolerance of the north star: 1 %).  A non-finite sum
// sends the candidate's work item to the exact fp64 careful path.
struct Stat32 {
  // Σ|e| per half as scalars (FADD with an |.| operand modifier: no sign-mask LOP3), Σe² as
  // an FFMA2 pair, max|e| over both halves with one 3-input FMNMX -- the same sums as a
  // pair-wise accumulation, in fewer issue slots
  float s0a = 0.0f, s0b = 0.0f, m0 = 0.0f;
  u64 s1 = 0ull;
  __device__ __forceinline__ void add(u64 y, u64 hi, u64 lo) {
    u64 e, t;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(y), "l"(hi));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(e) : "l"(t), "l"(lo));
    float e0, e1;
    split2(e, e0, e1);
    s0a = __fadd_rn(s0a, fabsf(e0));
    s0b = __fadd_rn(s0b, fabsf(e1));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(s1) : "l"(e), "l"(s1));
    m0 = fmaxf(m0, fmaxf(fabsf(e0), fabsf(e1)));
  }
  // the two halves combined (fixed order)
  __device__ __forceinline__ void fold(float& v0, float& v1, float& vm) const {
    float a, b;
    v0 = s0a + s0b;
    split2(s1, a, b);
    v1 = a + b;
    vm = m0;
  }
};

// single-tile counterpart of Stat32 (large-n register kernels, one tile per thread)
struct Stat32S {
  float s0 = 0.0f, s1 = 0.0f, m0 = 0.0f;
  __device__ __forceinline__ void add(float y, float hi, float lo) {
    const float e = __fsub_rn(__fsub_rn(y, hi), lo);
    const float ae = fabsf(e);
    s0 = __fadd_rn(s0, ae);
    s1 = __fmaf_rn(e, e, s1);
    m0 = fmaxf(m0, ae);
  }
  __device__ __forceinline__ void fold(float& v0, float& v1, float& vm) const {
    v0 = s0;
    v1 = s1;
    vm = m0;
  }
};

template <bool PAIR>
struct StatF {
  typedef Stat32 type;
};
template <>
struct StatF<false> {
  typedef Stat32S type;
};

// Shared-memory statistics of the register kernels: per (candidate of the work item, thread)
// three fp32 accumulators [kMaxCpc][3][kSwThreads] (thread-private slots: no barrier, no
// warp reduction inside the candidate loop) and a per-candidate "needs the careful path"
// flag; scratch for the careful path's 4-warp combination.
__host__ __device__ constexpr size_t stat_smem_bytes(int cap) {
  return (size_t)cap * 3 * kSwThreads * 4 + (size_t)kMaxCpc * 4 + 4 * kPartial * 8;
}
// candidates per work item of the register kernels: the 2D tile-pair kernel caps them at 24
// so that its y64 staging + statistics fit three CTAs per SM (68 KB each)
__host__ __device__ constexpr int reg_cpc_cap(int dims, bool pair) { return dims == 2 && pair ? 24 : kMaxCpc; }

struct SmemStats {
  float* acc;    // [cap][3][kSwThreads]
  int* flag;     // [kMaxCpc]
  double* red;   // [4][kPartial]
  __device__ __forceinline__ static SmemStats at(unsigned char* p, int cap) {
    SmemStats s;
    s.acc = reinterpret_cast<float*>(p);
    s.flag = reinterpret_cast<int*>(s.acc + cap * 3 * kSwThreads);
    s.red = reinterpret_cast<double*>(s.flag + kMaxCpc);
    return s;
  }
  // accumulate one (candidate, tile block) contribution of this thread; `first`: the work
  // item's first tile block (initialise instead of reading)
  template <class ST>
  __device__ __forceinline__ void add(int k, bool first, const ST& st32) const {
    float* a = acc + k * 3 * kSwThreads + threadIdx.x;
    float o0 = 0.0f, o1 = 0.0f, o2 = 0.0f;
    if (!first) {
      o0 = a[0];
      o1 = a[kSwThreads];
      o2 = a[2 * kSwThreads];
    }
    float v0, v1, vm;
    st32.fold(v0, v1, vm);
    if (!(isfinite(v0) && isfinite(v1))) flag[k] = 1;   // idempotent: order-independent
    a[0] = o0 + v0;
    a[kSwThreads] = o1 + v1;
    a[2 * kSwThreads] = fmaxf(o2, vm);
  }
  // after a barrier: the flagged candidates of the work item as a bit mask, provably
  // warp-uniform (a ballot), so the loop over them keeps the item's candidate indices in
  // uniform registers (coefficients via LDCU, not per-thread LDC)
  __device__ __forceinline__ unsigned flagged(int ncand) const {
    const int lane = threadIdx.x & 31;
    return __ballot_sync(0xffffffffu, lane < ncand && flag[lane] != 0);
  }
  // after a barrier: per unflagged candidate k, fp64 fixed-order sum over the 128 threads
  // -> the (candidate, tile group) partial.  Warp w handles candidates w, w + 4, ...
  __device__ __forceinline__ void reduce(int ncand, int c_begin, const IdxParam& DI, double* partial, int n_tgroups,
                                         int tg) const {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int k = warp; k < ncand; k += 4) {
      const float* a = acc + k * 3 * kSwThreads;
      double v0 = 0.0, v1 = 0.0, vm = 0.0;
#pragma unroll
      for (int j = 0; j < kSwThreads / 32; j++) {
        v0 += (double)a[lane + 32 * j];
        v1 += (double)a[kSwThreads + lane + 32 * j];
        vm = fmax(vm, (double)a[2 * kSwThreads + lane + 32 * j]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        vm = fmax(vm, __shfl_xor_sync(0xffffffffu, vm, o));
      }
      if (lane == 0 && flag[k] == 0) {
        double* pp = partial + ((long long)DI.idx[c_begin + k] * n_tgroups + tg) * kPartial;
        pp[0] = v0;
        pp[1] = v1;
        pp[2] = vm;
        pp[3] = 0.0;
      }
    }
  }
  // careful path epilogue: per-thread exact Stat -> warp butterflies -> 4 warps in order
  // -> the partial (all threads call; contains barriers)
  __device__ __forceinline__ void write_careful(Stat& st, double* pp) const {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    st.warp_reduce();
    if (lane == 0) {
      red[warp * kPartial + 0] = st.s0[0];
      red[warp * kPartial + 1] = st.s1[0];
      red[warp * kPartial + 2] = st.m0[0];
      red[warp * kPartial + 3] = (double)st.nonfin;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double v[kPartial] = {0.0, 0.0, 0.0, 0.0};
      for (int w = 0; w < 4; w++) {
        v[0] += red[w * kPartial + 0];
        v[1] += red[w * kPartial + 1];
        v[2] = red[w * kPartial + 2] > v[2] ? red[w * kPartial + 2] : v[2];
        v[3] += red[w * kPartial + 3];
      }
      for (int f = 0; f < kPartial; f++) pp[f] = v[f];
    }
    __syncthreads();
  }
};

// ------------------------------------------------------------------ K6: fp64 references
// Generic layouts: y64 [n_tiles][m^dims] = fp64 direct valid correlation of every tile
// (c-independent, once per call) + per-block Σ|y64| / max|y64|; y64t = the same values
// tile-block-major [t / 128][m^dims][t % 128] (coalesced per-output reads of the generic 2D
// kernel; padding tiles of the last blocks are 0).
template <int DIMS, int M, int R>
__global__ void __launch_bounds__(256) sweep_refs_kernel(const float* __restrict__ d, const float* __restrict__ g,
                                                         double* __restrict__ y64, double* __restrict__ y64t,
                                                         long long n_tiles, double* __restrict__ ref_part) {
  constexpr int N = M + R - 1;
  constexpr int DN = DIMS == 1 ? N : N * N, DG = DIMS == 1 ? R : R * R, DY = DIMS == 1 ? M : M * M;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double* yt_t = y64t + (t >> 7) * DY * kSwThreads + (t & (kSwThreads - 1));
  if (t >= n_tiles)
    for (int o = 0; o < DY; o++) yt_t[o * kSwThreads] = 0.0;
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
        yt_t[p * kSwThreads] = acc;
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
          yt_t[(p * M + q) * kSwThreads] = acc;
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

// Register layouts: the same fp64 references, plus the tiles and references repacked into
// coalesced per-lane layouts.  PAIR: group G = tiles [256 G, 256 G + 256); element e of
// lane tid is the u64 (tile 256 G + tid, tile 256 G + 128 + tid).  Single: group G = tiles
// [128 G, 128 G + 128), element e of lane tid is the float of tile 128 G + tid.  y64 is split
// into fp32 hi = RN32(y64) and lo = RN32(y64 − hi).  Padding tiles (>= n_tiles) are zeros.
// One CTA per group; per-CTA Σ|y64|, max|y64| partials in the same fixed order for any
// candidate sharding.
template <int DIMS, int M, int R, bool PAIR>
__global__ void __launch_bounds__(kSwThreads) sweep_prep_kernel(const float* __restrict__ d,
                                                                const float* __restrict__ g, long long n_tiles,
                                                                u64* __restrict__ dp, u64* __restrict__ gp,
                                                                u64* __restrict__ yh, u64* __restrict__ yl,
                                                                double* __restrict__ ref_part) {
  constexpr int N = M + R - 1;
  constexpr int DN = DIMS == 1 ? N : N * N, DG = DIMS == 1 ? R : R * R, DY = DIMS == 1 ? M : M * M;
  constexpr int W = PAIR ? 2 : 1;
  const long long grp = blockIdx.x;
  const int tid = threadIdx.x;
  double s = 0.0, mx = 0.0;
  float y_hi[2][DY], y_lo[2][DY];
#pragma unroll 1
  for (int h = 0; h < W; h++) {
    const long long t = grp * (W * kSwThreads) + h * kSwThreads + tid;
    const bool ok = t < n_tiles;
    const float* dt = d + t * DN;
    const float* gt = g + t * DG;
#pragma unroll
    for (int o = 0; o < DY; o++) {
      const int p = DIMS == 1 ? o : o / M, q = DIMS == 1 ? 0 : o % M;
      double acc = 0.0;
      if (ok) {
        if (DIMS == 1) {
          for (int j = 0; j < R; j++) acc = __dadd_rn(acc, __dmul_rn((double)gt[j], (double)dt[p + j]));
        } else {
          for (int u = 0; u < R; u++)
            for (int v = 0; v < R; v++)
              acc = __dadd_rn(acc, __dmul_rn((double)gt[u * R + v], (double)dt[(p + u) * N + q + v]));
        }
      }
      s += fabs(acc);
      mx = fmax(mx, fabs(acc));
      y_hi[h][o] = __double2float_rn(acc);
      y_lo[h][o] = __double2float_rn(acc - (double)y_hi[h][o]);
    }
  }
  const long long t0 = grp * (W * kSwThreads) + tid, t1 = t0 + kSwThreads;
  const bool ok0 = t0 < n_tiles, ok1 = PAIR && t1 < n_tiles;
  if constexpr (PAIR) {
    for (int e = 0; e < DN; e++)
      dp[(grp * DN + e) * kSwThreads + tid] = pack2(ok0 ? __ldg(d + t0 * DN + e) : 0.0f, ok1 ? __ldg(d + t1 * DN + e) : 0.0f);
    for (int e = 0; e < DG; e++)
      gp[(grp * DG + e) * kSwThreads + tid] = pack2(ok0 ? __ldg(g + t0 * DG + e) : 0.0f, ok1 ? __ldg(g + t1 * DG + e) : 0.0f);
#pragma unroll
    for (int o = 0; o < DY; o++) {
      yh[(grp * DY + o) * kSwThreads + tid] = pack2(y_hi[0][o], y_hi[1][o]);
      yl[(grp * DY + o) * kSwThreads + tid] = pack2(y_lo[0][o], y_lo[1][o]);
    }
  } else {
    float* dpf = reinterpret_cast<float*>(dp);
    float* gpf = reinterpret_cast<float*>(gp);
    float* yhf = reinterpret_cast<float*>(yh);
    float* ylf = reinterpret_cast<float*>(yl);
    for (int e = 0; e < DN; e++) dpf[(grp * DN + e) * kSwThreads + tid] = ok0 ? __ldg(d + t0 * DN + e) : 0.0f;
    for (int e = 0; e < DG; e++) gpf[(grp * DG + e) * kSwThreads + tid] = ok0 ? __ldg(g + t0 * DG + e) : 0.0f;
#pragma unroll
    for (int o = 0; o < DY; o++) {
      yhf[(grp * DY + o) * kSwThreads + tid] = y_hi[0][o];
      ylf[(grp * DY + o) * kSwThreads + tid] = y_lo[0][o];
    }
  }
  __shared__ double red[2][4];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = s;
    red[1][tid >> 5] = mx;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < 4; w++) {
      a += red[0][w];
      b = fmax(b, red[1][w]);
    }
    ref_part[grp * 2] = a;
    ref_part[grp * 2 + 1] = b;
  }
}

// ------------------------------------------------------------------ K7 (2D, generic)
// One candidate on this thread's tile(s); tiles d in shared memory (reused by the CTA's
// candidates), T2 staged in shared memory.  Scores (fast: add_fast; careful: exact with
// per-output finiteness, padding tiles excluded) and, if yd != NULL, writes the outputs.
template <int M, int R, bool PAIR, bool NOFMA, bool CAREFUL, int Z>
__device__ __forceinline__ void eval2d(const float* __restrict__ cm, const typename Lane<PAIR, NOFMA>::T* sd,
                                       typename Lane<PAIR, NOFMA>::T* st2, const double* const (&yt)[2],
                                       const typename Lane<PAIR, NOFMA>::T (&g)[R * R], int tid, Stat& st,
                                       float* yd, long long tile0, long long n_tiles) {
  using L = Lane<PAIR, NOFMA>;
  using T = typename L::T;
  constexpr int W = L::W;
  constexpr int N = M + R - 1, MM = M * M;
  constexpr int OFF_G = M * N, OFF_B = M * N + N * R;
  // COMPACT (n >= 9): the column loop of T2 and the row loop of U / V / T3 are NOT unrolled.
  // Fully unrolled, one F(6x6,5x5) evaluation is ~3000 FFMAs (150 KB of SASS with the careful
  // path) and the warps stall on instruction fetch (ncu: "no instructions" the top stall).
  // Rolled, the hot code shrinks ~10x.  The structural zeros of Bᵀ (T2, V) and G (U) depend
  // only on the unrolled indices and stay compile-time skipped; T1 = G g and the T3 update
  // (whose zeros depend on the rolled row i) run dense -- the canonical chains themselves
  // (parity semantics: skipping a zero term is the optimisation, not the definition).
  constexpr bool COMPACT = N >= 9;
  // T2 = Bᵀ d, column by column (d column q from smem), staged to smem
#pragma unroll (COMPACT ? 1 : N)
  for (int q = 0; q < N; q++) {
    T dc[N];
#pragma unroll
    for (int j = 0; j < N; j++) dc[j] = sd[(j * N + q) * kSwThreads + tid];
#pragma unroll
    for (int i = 0; i < N; i++) {
      T acc = L::zero();
#pragma unroll
      for (int j = 0; j < N; j++)
        if (nzB<Z>(i * N + j)) acc = L::fma(dc[j], cm[OFF_B + i * N + j], acc);
      st2[(i * N + q) * kSwThreads + tid] = acc;
    }
  }
  T t3[M][N];
#pragma unroll
  for (int p = 0; p < M; p++)
#pragma unroll
    for (int l = 0; l < N; l++) t3[p][l] = L::zero();
#pragma unroll (COMPACT ? 1 : N)
  for (int i = 0; i < N; i++) {
    // U row i = (G g Gᵀ)[i,:]:  T1[i][q] = Σ_j G[i][j] g[j][q];  U[i][l] = Σ_q T1[i][q] G[l][q]
    T t1[R];
#pragma unroll
    for (int q = 0; q < R; q++) {
      T acc = L::zero();
#pragma unroll
      for (int j = 0; j < R; j++)
        if (COMPACT || nzG<Z>(i * R + j)) acc = L::fma(g[j * R + q], cm[OFF_G + i * R + j], acc);
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
        if (nzG<Z>(l * R + q)) u = L::fma(t1[q], cm[OFF_G + l * R + q], u);
      // V[i][l] = Σ_q T2[i][q] Bᵀ[l][q]
      T v = L::zero();
#pragma unroll
      for (int q = 0; q < N; q++)
        if (nzB<Z>(l * N + q)) v = L::fma(t2r[q], cm[OFF_B + l * N + q], v);
      const T mw = L::mul(u, v);
      // T3[p][l] += Aᵀ[p][i] Mw[i][l]  (ascending i, from +0)
#pragma unroll
      for (int p = 0; p < M; p++)
        if (COMPACT || nzA<Z>(p * N + i)) t3[p][l] = L::fma(mw, cm[p * N + i], t3[p][l]);
    }
  }
  // Y[p][q] = Σ_l T3[p][l] Aᵀ[q][l]; score (and write)
#pragma unroll
  for (int p = 0; p < M; p++) {
#pragma unroll
    for (int q = 0; q < M; q++) {
      T y = L::zero();
#pragma unroll
      for (int l = 0; l < N; l++)
        if (nzA<Z>(q * N + l)) y = L::fma(t3[p][l], cm[q * N + l], y);
      const int o = p * M + q;
#pragma unroll
      for (int h = 0; h < W; h++) {
        const bool ok = tile0 + tid + h * kSwThreads < n_tiles;
        if (yd != nullptr && ok) yd[(tid + h * kSwThreads) * MM + o] = L::get(y, h);
        const double yref = __ldg(yt[h] + o * kSwThreads);   // coalesced, L1/L2-resident
        if (CAREFUL) {
          if (ok) {
            if (h == 0) st.template add_careful<0>(L::get(y, h), yref);
            else st.template add_careful<1>(L::get(y, h), yref);
          }
        } else {
          if (h == 0) st.template add_fast<0>(L::get(y, h), yref);
          else st.template add_fast<1>(L::get(y, h), yref);
        }
      }
    }
  }
}

// smem: sd [NN][128] T (tiles), st2 [NN][128] T (T2 staging), sacc [kMaxCpc][4 warps][kPartial]
// double; the fp64 references are read per output from y64t (no shared-memory copy: the
// large-n tiles need the capacity for occupancy)
template <int M, int R, bool PAIR, bool NOFMA, int Z>
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
  double* sacc = reinterpret_cast<double*>(st2 + NN * kSwThreads);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_launch_dependents();
  // persistent CTAs walk the (candidate group, tile group) work items round-robin
  const int n_items = a.n_cgroups * a.n_tgroups;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int cg = item / a.n_tgroups, tg = item - cg * a.n_tgroups;
    const int c_begin = cg * a.cands_per_cta;
    const int c_end = min(a.n_cand, c_begin + a.cands_per_cta);
    __syncthreads();  // the previous item's accumulators are flushed
    for (int k = tid; k < kMaxCpc * 4 * kPartial; k += kSwThreads) sacc[k] = 0.0;
    __syncthreads();  // zeroed before any warp accumulates (lane 0 of another warp)

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

      const double* yt[2];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const long long t = tile0 + tid + (W == 2 ? h : 0) * kSwThreads;
        yt[h] = a.y64t + (t >> 7) * MM * kSwThreads + (t & (kSwThreads - 1));
      }
      for (int s = c_begin; s < c_end; s++) {
        const float* cm = P.v + s * PER;
        Stat st;
        float* yd = a.ydump ? a.ydump + ((long long)DI.idx[s] * a.n_tiles + tile0) * MM : nullptr;
        eval2d<M, R, PAIR, NOFMA, false, Z>(cm, sd, st2, yt, g, tid, st, yd, tile0, a.n_tiles);
        if (__any_sync(0xffffffffu, !st.finite())) {
          // exact per-output path with the dense chains (the oracle's; a skipped zero term
          // can hide an inf * 0 = NaN of the dense chain), padding tiles excluded
          st = Stat();
          eval2d<M, R, PAIR, NOFMA, true, 0>(cm, sd, st2, yt, g, tid, st, yd, tile0, a.n_tiles);
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
  }  // work items
  pdl_wait();
}

// ------------------------------------------------------------------ K7 (2D, tiles in registers)
// For small n (PAIR: the thread's two tiles) or large n (single: one tile): the tiles d stay
// in registers and T2 is formed row by row from them (T2[i][q] = Σ_j Bᵀ[i][j] d[j][q],
// ascending j), so no candidate-dependent data touches shared memory; only y64 (hi, lo) is
// staged.  Same chains as eval2d.
template <int M, int R, bool PAIR, bool NOFMA, bool CAREFUL, int Z>
__device__ __forceinline__ void eval2d_r(const float* __restrict__ cm,
                                         const typename Lane<PAIR, NOFMA>::T (&d)[(M + R - 1) * (M + R - 1)],
                                         const typename Lane<PAIR, NOFMA>::T (&g)[R * R],
                                         const typename Lane<PAIR, NOFMA>::T* syh,
                                         const typename Lane<PAIR, NOFMA>::T* syl, int tid, Stat& st,
                                         typename StatF<PAIR>::type& st32, float* yd, long long tile0,
                                         long long n_tiles) {
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
        if (nzG<Z>(i * R + j)) acc = L::fma(g[j * R + q], cm[OFF_G + i * R + j], acc);
      t1[q] = acc;
    }
    T t2r[N];
#pragma unroll
    for (int q = 0; q < N; q++) {
      T acc = L::zero();
#pragma unroll
      for (int j = 0; j < N; j++)
        if (nzB<Z>(i * N + j)) acc = L::fma(d[j * N + q], cm[OFF_B + i * N + j], acc);
      t2r[q] = acc;
    }
#pragma unroll
    for (int l = 0; l < N; l++) {
      T u = L::zero();
#pragma unroll
      for (int q = 0; q < R; q++)
        if (nzG<Z>(l * R + q)) u = L::fma(t1[q], cm[OFF_G + l * R + q], u);
      T v = L::zero();
#pragma unroll
      for (int q = 0; q < N; q++)
        if (nzB<Z>(l * N + q)) v = L::fma(t2r[q], cm[OFF_B + l * N + q], v);
      const T mw = L::mul(u, v);
#pragma unroll
      for (int p = 0; p < M; p++)
        if (nzA<Z>(p * N + i)) t3[p][l] = L::fma(mw, cm[p * N + i], t3[p][l]);
    }
  }
  // this thread's own y64 slots, staged by cp.async at the tile block's start, have landed
  if (!CAREFUL) cp_async_wait_all();
#pragma unroll
  for (int p = 0; p < M; p++) {
#pragma unroll
    for (int q = 0; q < M; q++) {
      T y = L::zero();
#pragma unroll
      for (int l = 0; l < N; l++)
        if (nzA<Z>(q * N + l)) y = L::fma(t3[p][l], cm[q * N + l], y);
      const int o = p * M + q;
      if (yd != nullptr) {
#pragma unroll
        for (int h = 0; h < W; h++)
          if (tile0 + tid + h * kSwThreads < n_tiles) yd[(tid + h * kSwThreads) * MM + o] = L::get(y, h);
      }
      if (CAREFUL) {
        // exact fp64 path on y64 = hi + lo (the split is exact in fp64 to 2^-48 relative)
        const T hp = syh[o * kSwThreads + tid], lp = syl[o * kSwThreads + tid];
        if (tile0 + tid < n_tiles)
          st.template add_careful<0>(L::get(y, 0), (double)L::get(hp, 0) + (double)L::get(lp, 0));
        if (W == 2 && tile0 + tid + kSwThreads < n_tiles)
          st.template add_careful<1>(L::get(y, 1), (double)L::get(hp, 1) + (double)L::get(lp, 1));
      } else {
        st32.add(y, syh[o * kSwThreads + tid], syl[o * kSwThreads + tid]);
      }
    }
  }
}

// Coalesced loads of the thread's packed tile(s) (group grp).
template <class T, int NN, int RR>
__device__ __forceinline__ void load_tiles2d(const SweepArgs& a, long long grp, int tid, T (&d)[NN], T (&g)[RR]) {
  const T* dp = reinterpret_cast<const T*>(a.dp);
  const T* gp = reinterpret_cast<const T*>(a.gp);
#pragma unroll
  for (int e = 0; e < NN; e++) d[e] = __ldg(dp + (grp * NN + e) * kSwThreads + tid);
#pragma unroll
  for (int e = 0; e < RR; e++) g[e] = __ldg(gp + (grp * RR + e) * kSwThreads + tid);
}

// smem: syh [MM][128] T, syl [MM][128] T, then SmemStats
template <int M, int R, bool PAIR, bool NOFMA, int Z>
__global__ void __launch_bounds__(kSwThreads, PAIR ? 3 : 1) sweep2d_reg_kernel(SweepArgs a, const __grid_constant__ MatsParam P,
                                                                 const __grid_constant__ IdxParam DI) {
  using L = Lane<PAIR, NOFMA>;
  using T = typename L::T;
  constexpr int N = M + R - 1, NN = N * N, MM = M * M, RR = R * R;
  constexpr int PER = M * N + N * R + N * N;
  constexpr int TPB = L::W * kSwThreads;
  extern __shared__ __align__(16) unsigned char smem[];
  T* syh = reinterpret_cast<T*>(smem);            // [MM][128] (hi_A, hi_B) / hi
  T* syl = syh + MM * kSwThreads;                  // [MM][128] (lo_A, lo_B) / lo
  const SmemStats ss = SmemStats::at(reinterpret_cast<unsigned char*>(syl + MM * kSwThreads), reg_cpc_cap(2, PAIR));
  const T* gyh = reinterpret_cast<const T*>(a.yh);
  const T* gyl = reinterpret_cast<const T*>(a.yl);

  const int tid = threadIdx.x;
  pdl_launch_dependents();
  const int n_items = a.n_cgroups * a.n_tgroups;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int cg = item / a.n_tgroups, tg = item - cg * a.n_tgroups;
    const int c_begin = cg * a.cands_per_cta;
    const int c_end = min(a.n_cand, c_begin + a.cands_per_cta);
    const int ncand = c_end - c_begin;
    const int tb_begin = tg * a.tblk_per_cta;
    const int tb_end = min(a.n_tblk, tb_begin + a.tblk_per_cta);
    __syncthreads();  // the previous item's statistics have been read
    if (tid < kMaxCpc) ss.flag[tid] = 0;
    __syncthreads();
    for (int tb = tb_begin; tb < tb_end; tb++) {
      const long long tile0 = (long long)tb * TPB;
      // each thread stages (and later reads) only its own y64 slots: no barrier needed.  The
      // copies are asynchronous (waited for before the first scoring) and issued before the
      // tile loads, so their latency hides behind the first candidate's transforms; the
      // previous block's reads of these slots were consumed before this point (program order)
#pragma unroll 4
      for (int o = 0; o < MM; o++) {
        cp_async_word(syh + o * kSwThreads + tid, gyh + ((long long)tb * MM + o) * kSwThreads + tid);
        cp_async_word(syl + o * kSwThreads + tid, gyl + ((long long)tb * MM + o) * kSwThreads + tid);
      }
      cp_async_commit();
      T d[NN], g[RR];
      load_tiles2d<T, NN, RR>(a, tb, tid, d, g);
      for (int s = c_begin; s < c_end; s++) {
        const float* cm = P.v + s * PER;
        Stat st;
        typename StatF<PAIR>::type st32;
        float* yd = a.ydump ? a.ydump + ((long long)DI.idx[s] * a.n_tiles + tile0) * MM : nullptr;
        eval2d_r<M, R, PAIR, NOFMA, false, Z>(cm, d, g, syh, syl, tid, st, st32, yd, tile0, a.n_tiles);
        ss.add(s - c_begin, tb == tb_begin, st32);
      }
    }
    __syncthreads();
    ss.reduce(ncand, c_begin, DI, a.partial, a.n_tgroups, tg);
    // Rare: a candidate whose fp32 sums went non-finite in this work item is re-evaluated
    // exactly (fp64 statistics per output, dense chains, padding tiles excluded).
    for (unsigned fl = ss.flagged(ncand); fl != 0u; fl &= fl - 1u) {
      const int k = __ffs(fl) - 1;
      const int s = c_begin + k;
      const float* cm = P.v + s * PER;
      Stat st;
      typename StatF<PAIR>::type st32;
      for (int tb = tb_begin; tb < tb_end; tb++) {
        const long long tile0 = (long long)tb * TPB;
        T d[NN], g[RR];
        load_tiles2d<T, NN, RR>(a, tb, tid, d, g);
        float* yd = a.ydump ? a.ydump + ((long long)DI.idx[s] * a.n_tiles + tile0) * MM : nullptr;
        eval2d_r<M, R, PAIR, NOFMA, true, 0>(cm, d, g, gyh + (long long)tb * MM * kSwThreads,
                                             gyl + (long long)tb * MM * kSwThreads, tid, st, st32, yd, tile0,
                                             a.n_tiles);
      }
      ss.write_careful(st, a.partial + ((long long)DI.idx[s] * a.n_tgroups + tg) * kPartial);
    }
  }
  cp_async_wait_all();
  pdl_wait();
}

// ------------------------------------------------------------------ K7 (1D)
// Tile pairs in registers; scoring as in the register-resident 2D kernel.
template <int M, int R, bool NOFMA, bool CAREFUL, int Z>
__device__ __forceinline__ void eval1d(const float* __restrict__ cm, const u64 (&d)[M + R - 1], const u64 (&g)[R],
                                       const u64 (&yh)[M], const u64 (&yl)[M], Stat& st, Stat32& st32, float* yd,
                                       long long tile0, long long n_tiles, int tid) {
  using L = Lane<true, NOFMA>;
  using T = u64;
  constexpr int N = M + R - 1;
  constexpr int OFF_G = M * N, OFF_B = M * N + N * R;
  T mw[N];
#pragma unroll
  for (int i = 0; i < N; i++) {
    T u = L::zero(), v = L::zero();
#pragma unroll
    for (int j = 0; j < R; j++)
      if (nzG<Z>(i * R + j)) u = L::fma(g[j], cm[OFF_G + i * R + j], u);
#pragma unroll
    for (int j = 0; j < N; j++)
      if (nzB<Z>(i * N + j)) v = L::fma(d[j], cm[OFF_B + i * N + j], v);
    mw[i] = L::mul(u, v);
  }
#pragma unroll
  for (int p = 0; p < M; p++) {
    T y = L::zero();
#pragma unroll
    for (int i = 0; i < N; i++)
      if (nzA<Z>(p * N + i)) y = L::fma(mw[i], cm[p * N + i], y);
    if (yd != nullptr) {
#pragma unroll
      for (int h = 0; h < 2; h++)
        if (tile0 + tid + h * kSwThreads < n_tiles) yd[(tid + h * kSwThreads) * M + p] = L::get(y, h);
    }
    if (CAREFUL) {
      float h0, h1, l0, l1;
      split2(yh[p], h0, h1);
      split2(yl[p], l0, l1);
      if (tile0 + tid < n_tiles) st.template add_careful<0>(L::get(y, 0), (double)h0 + (double)l0);
      if (tile0 + tid + kSwThreads < n_tiles) st.template add_careful<1>(L::get(y, 1), (double)h1 + (double)l1);
    } else {
      st32.add(y, yh[p], yl[p]);
    }
  }
}

// Packed data of sub-block k of tile block tb (group tb * kKP1 + k).
template <int M, int R>
__device__ __forceinline__ void load_pair1d(const SweepArgs& a, long long grp, int tid, u64 (&d)[M + R - 1],
                                            u64 (&g)[R], u64 (&yh)[M], u64 (&yl)[M]) {
  constexpr int N = M + R - 1;
#pragma unroll
  for (int j = 0; j < N; j++) d[j] = __ldg(a.dp + (grp * N + j) * kSwThreads + tid);
#pragma unroll
  for (int j = 0; j < R; j++) g[j] = __ldg(a.gp + (grp * R + j) * kSwThreads + tid);
#pragma unroll
  for (int j = 0; j < M; j++) {
    yh[j] = __ldg(a.yh + (grp * M + j) * kSwThreads + tid);
    yl[j] = __ldg(a.yl + (grp * M + j) * kSwThreads + tid);
  }
}

// Everything in registers; a CTA walks its tile blocks and, per block, its candidates.
// Each thread owns kKP1 pairs of tiles, so a candidate's coefficients (uniform registers)
// are amortised over 2 * kKP1 tile evaluations.  smem: SmemStats.  No min-blocks launch
// bound: capping the registers (2-3 CTAs/SM) made ptxas move the coefficients from uniform
// registers (LDCU) to per-thread LDC loads and re-load the tiles per candidate (measured
// 1.7x slower).
template <int M, int R, bool NOFMA, int Z>
__global__ void __launch_bounds__(kSwThreads) sweep1d_kernel(SweepArgs a, const __grid_constant__ MatsParam P,
                                                             const __grid_constant__ IdxParam DI) {
  constexpr int N = M + R - 1;
  constexpr int PER = M * N + N * R + N * N;
  constexpr int TPB = kGroupTiles * kKP1;
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemStats ss = SmemStats::at(smem, reg_cpc_cap(1, true));

  const int tid = threadIdx.x;
  pdl_launch_dependents();
  const int n_items = a.n_cgroups * a.n_tgroups;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int cg = item / a.n_tgroups, tg = item - cg * a.n_tgroups;
    const int c_begin = cg * a.cands_per_cta;
    const int c_end = min(a.n_cand, c_begin + a.cands_per_cta);
    const int ncand = c_end - c_begin;
    const int tb_begin = tg * a.tblk_per_cta;
    const int tb_end = min(a.n_tblk, tb_begin + a.tblk_per_cta);
    __syncthreads();
    if (tid < kMaxCpc) ss.flag[tid] = 0;
    __syncthreads();
    for (int tb = tb_begin; tb < tb_end; tb++) {
      u64 d[kKP1][N], g[kKP1][R], yh[kKP1][M], yl[kKP1][M];
#pragma unroll
      for (int k = 0; k < kKP1; k++) load_pair1d<M, R>(a, (long long)tb * kKP1 + k, tid, d[k], g[k], yh[k], yl[k]);
      for (int s = c_begin; s < c_end; s++) {
        const float* cm = P.v + s * PER;
        Stat st;
        Stat32 st32;
#pragma unroll
        for (int k = 0; k < kKP1; k++) {
          const long long tk0 = (long long)tb * TPB + k * kGroupTiles;
          float* yd = a.ydump ? a.ydump + ((long long)DI.idx[s] * a.n_tiles + tk0) * M : nullptr;
          eval1d<M, R, NOFMA, false, Z>(cm, d[k], g[k], yh[k], yl[k], st, st32, yd, tk0, a.n_tiles, tid);
        }
        ss.add(s - c_begin, tb == tb_begin, st32);
      }
    }
    __syncthreads();
    ss.reduce(ncand, c_begin, DI, a.partial, a.n_tgroups, tg);
    for (unsigned fl = ss.flagged(ncand); fl != 0u; fl &= fl - 1u) {
      const int kc = __ffs(fl) - 1;
      const int s = c_begin + kc;
      const float* cm = P.v + s * PER;
      Stat st;
      Stat32 st32;
      for (int tb = tb_begin; tb < tb_end; tb++) {
#pragma unroll 1
        for (int k = 0; k < kKP1; k++) {
          u64 d[N], g[R], yh[M], yl[M];
          load_pair1d<M, R>(a, (long long)tb * kKP1 + k, tid, d, g, yh, yl);
          const long long tk0 = (long long)tb * TPB + k * kGroupTiles;
          float* yd = a.ydump ? a.ydump + ((long long)DI.idx[s] * a.n_tiles + tk0) * M : nullptr;
          eval1d<M, R, NOFMA, true, 0>(cm, d, g, yh, yl, st, st32, yd, tk0, a.n_tiles, tid);
        }
      }
      ss.write_careful(st, a.partial + ((long long)DI.idx[s] * a.n_tgroups + tg) * kPartial);
    }
  }
  pdl_wait();
}

typedef void (*SweepKernel)(SweepArgs, MatsParam, IdxParam);
typedef void (*RefsKernel)(const float*, const float*, double*, double*, long long, double*);
typedef void (*PrepKernel)(const float*, const float*, long long, u64*, u64*, u64*, u64*, double*);

// Kernel layouts: TPAIR = two tiles per thread (FFMA2 lanes = tiles, coefficients per
// candidate as uniform registers), tiles in shared memory; TSINGLE = one tile per thread
// (FFMA), for large n; TPAIR_REG = tile pairs held in registers, packed inputs (K6 prep):
// the 2D small-n kernels and every 1D kernel; TSINGLE_REG = one tile per thread held in
// registers (2D large n).
enum Layout { TPAIR = 0, TSINGLE = 1, TPAIR_REG = 2, TSINGLE_REG = 3 };

struct Variant {
  int z;                         // structural-zero family (zero_masks.h; 0 = dense)
  uint64_t za[2], zg[2], zb[2];  // its 128-bit masks (bit k: entry k skipped)
  SweepKernel k[2];              // [nofma]
  Layout lay;
};

struct SweepCfg {
  int dims, m, r;
  Layout lay;
  RefsKernel refs;               // generic layouts, Huffman, mixed
  PrepKernel prep;               // TPAIR_REG, TSINGLE_REG
  std::vector<Variant> variants; // most specialised first, dense last
};

template <int DIMS, int M, int R, Layout LAY, int Z>
Variant make_variant() {
  Variant v;
  v.z = Z;
  for (int w = 0; w < 2; w++) {
    v.za[w] = ZM<Z>::A(w);
    v.zg[w] = ZM<Z>::G(w);
    v.zb[w] = ZM<Z>::B(w);
  }
  if constexpr (Z != 0) static_assert(ZM<Z>::m == M && ZM<Z>::r == R, "zero-mask family of another shape");
  if constexpr (DIMS == 1) {
    static_assert(LAY == TPAIR_REG, "1D kernels are register-resident");
    v.k[0] = (SweepKernel)sweep1d_kernel<M, R, false, Z>;
    v.k[1] = (SweepKernel)sweep1d_kernel<M, R, true, Z>;
  } else if constexpr (LAY == TPAIR_REG || LAY == TSINGLE_REG) {
    constexpr bool PAIR = LAY == TPAIR_REG;
    v.k[0] = (SweepKernel)sweep2d_reg_kernel<M, R, PAIR, false, Z>;
    v.k[1] = (SweepKernel)sweep2d_reg_kernel<M, R, PAIR, true, Z>;
  } else {
    constexpr bool PAIR = LAY == TPAIR;
    v.k[0] = (SweepKernel)sweep2d_kernel<M, R, PAIR, false, Z>;
    v.k[1] = (SweepKernel)sweep2d_kernel<M, R, PAIR, true, Z>;
  }
  v.lay = LAY;
  return v;
}

template <int DIMS, int M, int R, Layout LAY>
SweepCfg make_cfg(std::vector<Variant> specialised = {}) {
  SweepCfg c;
  c.dims = DIMS;
  c.m = M;
  c.r = R;
  c.lay = LAY;
  c.refs = nullptr;
  c.prep = nullptr;
  // refs: the generic layouts and the Huffman / mixed-precision kernels of every shape
  c.refs = sweep_refs_kernel<DIMS, M, R>;
  if constexpr (LAY == TPAIR_REG || LAY == TSINGLE_REG) c.prep = sweep_prep_kernel<DIMS, M, R, LAY == TPAIR_REG>;
  c.variants = specialised;
  c.variants.push_back(make_variant<DIMS, M, R, LAY, 0>());
  return c;
}

// Huffman-order (sweep_huff.cuh) and mixed-precision (sweep_mixed.cuh) sweep kernels
// (generic layout: raw tiles + fp64 references; always score, write outputs if ydump)
struct HuffCfg {
  int dims, m, r;
  SweepKernel k;
};

// per-translation-unit registries (sweep_inst_*.cu)
std::vector<SweepCfg> sweep_cfgs_1d();
std::vector<SweepCfg> sweep_cfgs_1d_large();
std::vector<SweepCfg> sweep_cfgs_2d_f43();
std::vector<SweepCfg> sweep_cfgs_2d_small();
std::vector<SweepCfg> sweep_cfgs_2d_large();
std::vector<SweepCfg> sweep_cfgs_2d_mid();
std::vector<HuffCfg> sweep_huff_cfgs();
std::vector<HuffCfg> sweep_mixed_cfgs();

}  // namespace wino
