// fp32 Winograd convolution layer F(m x m, r x r) (PAPER.md eq:conv_2d P:181; the channel
// sum "implemented using matrix multiplication"), sm_100a.  Kernels:
//   K1 filter_kernel : U_p[c][k] = (G w_kc Gᵀ)[p]                     -> U [NN][Cp][Kp]
//   K2 input_kernel  : V_p[c][t] = (Bᵀ d_ct B)[p], zero padding        -> V [NN][Cp][Tp]
//   K3 gemm_kernel   : M_p[k][t] = Σ_c U_p[c][k] V_p[c][t]  (NN batched fp32 GEMMs,
//                      FFMA2 register tiles, ascending-c chain, no split-K, no TF32)
//   K4 output_kernel : y tile = Aᵀ M_t A, cropped                      -> y [N][K][Ho][Wo]
//   K5 score_kernel  : y64 = fp64 direct correlation (eq:conv P:112), e = y - y64,
//                      per-warp statistics (warp shuffles), fixed grid
//   K8 finalize      : fixed-order reduction into d_sums/d_maxs
// Cp = C rounded up to 16, Kp = K rounded up to 128 (64 when K <= 64), Tp = T rounded up to
// 128; padding is zero-filled
// by K1/K2, so K3 needs no bounds checks (an fma(0, 0, acc) leaves acc unchanged up to
// the sign of a zero).  Parity semantics: every dot product is an
// fmaf chain from +0 in ascending index order, 2D transforms left product first.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "tc_gemm.cuh"
#include "wino_internal.h"
#include "zero_masks.h"

namespace wino {

namespace {

typedef unsigned long long u64;

constexpr int kMaxN = 10;   // layer kernels compiled for n <= 10

struct LayerMats {
  float AT[kMaxN * kMaxN];  // [m][n]
  float G[kMaxN * kMaxN];   // [n][r]
  float BT[kMaxN * kMaxN];  // [n][n]
};

struct Geo {
  int N, C, H, W, K, r, pad, m;
  int Ho, Wo, th, tw;
  long long T;     // tiles = N * th * tw
  int Cp, Kp;
  long long Tp;
  int tf32;        // 1: U / V rounded to TF32 (nearest, ties away) for the tcgen05 variant;
                   // 2: 3xTF32 -- hi = tf32(x) in plane p, lo = tf32(x - hi) in plane NN + p
  int bn;          // t-width of the FFMA GEMM's CTA tile (128, or 64: see make_geo)
};

// round-to-nearest fp32 -> TF32 (10 explicit mantissa bits); the tensor core would otherwise
// drop the low 13 bits (measured: truncation)
__device__ __forceinline__ float round_tf32(float v) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// Programmatic dependent launch (the unfused fp32 layer is the chain K1 -> K2 -> K3 -> K4 on
// one stream): a kernel launched with the attribute may become resident while its
// predecessor drains (after every CTA of the predecessor executed launch_dependents) and
// must execute `wait` before it touches the predecessor's output.  K2 does not depend on K1,
// so it runs beside it and waits only at its END -- its completion then implies K1's, which
// is what K3's wait (on K2) relies on for U.  Without the launch attribute both instructions
// are no-ops.
__device__ __forceinline__ void lpdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void lpdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, bool pdl,
                     Args&&... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = stream;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = la;
  lc.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&lc, kern, KArgs(args)...);
}

Geo make_geo(int N, int C, int H, int W, int K, int r, int pad, int m, int tf32 = 0) {
  Geo g;
  g.N = N; g.C = C; g.H = H; g.W = W; g.K = K; g.r = r; g.pad = pad; g.m = m;
  g.Ho = H + 2 * pad - r + 1;
  g.Wo = W + 2 * pad - r + 1;
  g.th = (g.Ho + m - 1) / m;
  g.tw = (g.Wo + m - 1) / m;
  g.T = (long long)N * g.th * g.tw;
  // FFMA GEMM: BK = 16, BN = 128 or 64; tcgen05 variant: BK = 32, N = 256
  const int ca = tf32 ? 32 : 16;
  g.Cp = (C + ca - 1) / ca * ca;
  // FFMA GEMM: 64-row tiles when K <= 64 (VGG's 64-channel layers), else 128; tcgen05: 128
  g.Kp = (!tf32 && K <= 64) ? 64 : (K + 127) / 128 * 128;
  // FFMA GEMM CTA tile: 128 (k) x 128 (t) at 2 CTAs per SM, or 128 x 64 at 4 per SM (the
  // same 8 x 8 register tile per thread, the same work per SM and wave): the narrow tile
  // pads T to 64 instead of 128 and quantises the grid in half-size steps, so it is chosen
  // when it needs fewer waves (VGG's 14 x 14 layers: T = 576 -> 5 waves of 128-wide tiles,
  // 4 of 64-wide ones).  Fixed SM count (B200: 148) so the workspace query and the launch
  // agree on Tp.
  g.bn = 128;
  if (!tf32 && g.Kp >= 128) {
    const long long per = (long long)(g.Kp / 128) * (m + r - 1) * (m + r - 1);
    const long long w128 = ((g.T + 127) / 128 * per + 2 * 148 - 1) / (2 * 148);
    const long long w64 = ((g.T + 63) / 64 * per + 4 * 148 - 1) / (4 * 148);
    if (w64 < w128) g.bn = 64;
  }
  const int ta = tf32 ? 256 : g.bn;
  g.Tp = (g.T + ta - 1) / ta * ta;
  g.tf32 = tf32;
  return g;
}


// ------------------------------------------------------------------ K1
template <int M, int R>
__global__ void filter_kernel(const float* __restrict__ w, float* __restrict__ U, int C, int K, int Cp, int Kp, int tf32,
                              const __grid_constant__ LayerMats mt) {
  constexpr int N = M + R - 1;
  lpdl_launch_dependents();
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // over Cp * Kp, k fastest
  if (idx >= (long long)Cp * Kp) return;
  const int k = (int)(idx % Kp), c = (int)(idx / Kp);
  const long long plane = (long long)Cp * Kp;
  if (k >= K || c >= C) {
#pragma unroll
    for (int p = 0; p < (tf32 == 2 ? 2 : 1) * N * N; p++) U[p * plane + idx] = 0.0f;
    return;
  }
  float g[R * R];
  const float* wk = w + ((long long)k * C + c) * R * R;
#pragma unroll
  for (int e = 0; e < R * R; e++) g[e] = wk[e];
  float t1[N][R];
#pragma unroll
  for (int i = 0; i < N; i++)
#pragma unroll
    for (int q = 0; q < R; q++) {
      float acc = 0.0f;
#pragma unroll
      for (int j = 0; j < R; j++) acc = __fmaf_rn(mt.G[i * R + j], g[j * R + q], acc);
      t1[i][q] = acc;
    }
#pragma unroll
  for (int i = 0; i < N; i++)
#pragma unroll
    for (int l = 0; l < N; l++) {
      float acc = 0.0f;
#pragma unroll
      for (int q = 0; q < R; q++) acc = __fmaf_rn(t1[i][q], mt.G[l * R + q], acc);
      if (tf32 == 2) {
        const float hi = round_tf32(acc);
        U[(i * N + l) * plane + idx] = hi;
        U[(N * N + i * N + l) * plane + idx] = round_tf32(acc - hi);
      } else {
        U[(i * N + l) * plane + idx] = tf32 ? round_tf32(acc) : acc;
      }
    }
}

// ------------------------------------------------------------------ K2
// Z: structural-zero family of the point set (zero_masks.h; 0 = dense): the Bᵀ entries it
// marks are skipped at compile time -- the launcher picks Z only when they are exactly 0 in
// this call's matrices, and a skipped fma(0, v, acc) = acc for finite v, so every element is
// the canonical chain's (22 % fewer FMAs for the F(6x6,3x3) family).
// one thread per (kInCpt channels, t); t fastest -> coalesced V stores per Winograd
// position.  The tile geometry, padding predicates and patch offsets are computed once and
// reused for the thread's kInCpt channels (the kernel is issue-bound on that arithmetic).
// channels per thread: 4 for the large n = 10 tiles (where the per-tile arithmetic
// dominates), 1 otherwise (more threads in flight); always divides Cp (a multiple of 16)
template <int N>
constexpr int in_cpt() { return N > 8 ? 4 : 1; }
// TF: the rounding of V compiled in (Geo::tf32: 0 fp32, 1 TF32, 2 3xTF32 hi / lo planes)
template <int M, int R, int Z, int TF>
__global__ void __launch_bounds__(256, M + R - 1 <= 8 ? 3 : 1) input_kernel(const float* __restrict__ x, float* __restrict__ V, Geo geo,
                                                       const __grid_constant__ LayerMats mt) {
  constexpr int N = M + R - 1;
  constexpr int kInCpt = in_cpt<N>();
  static_assert(N <= 16, "row / column masks are 16 bits");
  lpdl_launch_dependents();
  const long long gidx = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // over Cp / kInCpt * Tp
  if (gidx >= (long long)(geo.Cp / kInCpt) * geo.Tp) {
    lpdl_wait();
    return;
  }
  const long long t = gidx % geo.Tp;
  const int c0 = (int)(gidx / geo.Tp) * kInCpt;
  const long long plane = (long long)geo.Cp * geo.Tp;
  const long long lo_off = (long long)N * N * plane;   // 3xTF32 lo planes
  const bool tile_ok = t < geo.T;
  int img = 0, h0 = 0, w0 = 0;
  unsigned rowm = 0, colm = 0;
  if (tile_ok) {
    const int per_img = geo.th * geo.tw;
    img = (int)(t / per_img);
    const int rem = (int)(t - (long long)img * per_img);
    const int ty = rem / geo.tw, tx = rem - ty * geo.tw;
    h0 = ty * M - geo.pad;
    w0 = tx * M - geo.pad;
#pragma unroll
    for (int a = 0; a < N; a++) rowm |= (h0 + a >= 0 && h0 + a < geo.H) ? 1u << a : 0u;
#pragma unroll
    for (int b = 0; b < N; b++) colm |= (w0 + b >= 0 && w0 + b < geo.W) ? 1u << b : 0u;
  }
  const long long off0 = (long long)h0 * geo.W + w0;   // patch origin (may lie outside)
#pragma unroll 1
  for (int cc = 0; cc < kInCpt; cc++) {
    const int c = c0 + cc;
    float* dst = V + (long long)c * geo.Tp + t;
    if (!tile_ok || c >= geo.C) {
#pragma unroll
      for (int p = 0; p < N * N; p++) {
        dst[(long long)p * plane] = 0.0f;
        if (TF == 2) dst[lo_off + (long long)p * plane] = 0.0f;
      }
      continue;
    }
    const float* xc = x + ((long long)img * geo.C + c) * geo.H * geo.W + off0;
    float d[N][N];
#pragma unroll
    for (int a = 0; a < N; a++)
#pragma unroll
      for (int b = 0; b < N; b++)
        d[a][b] = ((rowm >> a) & (colm >> b) & 1u) ? __ldg(xc + (long long)a * geo.W + b) : 0.0f;
    // T2[i][q] = Σ_j Bᵀ[i][j] d[j][q]
    float t2[N][N];
#pragma unroll
    for (int q = 0; q < N; q++)
#pragma unroll
      for (int i = 0; i < N; i++) {
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < N; j++)
          if (nzB<Z>(i * N + j)) acc = __fmaf_rn(mt.BT[i * N + j], d[j][q], acc);
        t2[i][q] = acc;
      }
    // V[i][l] = Σ_q T2[i][q] Bᵀ[l][q]; positions p = i N + l stored in ascending order
#pragma unroll
    for (int i = 0; i < N; i++)
#pragma unroll
      for (int l = 0; l < N; l++) {
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < N; q++)
          if (nzB<Z>(l * N + q)) acc = __fmaf_rn(t2[i][q], mt.BT[l * N + q], acc);
        if (TF == 2) {
          const float hi = round_tf32(acc);
          dst[0] = hi;
          dst[lo_off] = round_tf32(acc - hi);
        } else {
          dst[0] = TF ? round_tf32(acc) : acc;
        }
        dst += plane;
      }
  }
  lpdl_wait();   // K2 completes after K1 (see lpdl_wait above)
}

// ------------------------------------------------------------------ K3
// Batched SGEMM  M_p[k][t] = Σ_c U_p[c][k] V_p[c][t], BMT x BNT CTA tile (128 x 128;
// 64 x 128 when K <= 64 so the GEMM neither computes nor writes padded k rows; 128 x 64
// when that needs fewer waves, make_geo), BK = 16, BMT * BNT / 64 threads x (8 x 8) register
// tile, accumulators as FFMA2 pairs along t.
// cp.async 3-stage shared-memory ring; every accumulator is one ascending-c fmaf chain.
constexpr int BK = 16;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NW>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NW)); }

__device__ __forceinline__ u64 ffma2_bcast(u64 a, float c, u64 acc) {
  u64 d, cc;
  asm("mov.b64 %0, {%1,%1};" : "=l"(cc) : "f"(c));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(cc), "l"(acc));
  return d;
}

constexpr int kStages = 3;
template <int BMT, int BNT>
constexpr size_t gemm_smem() { return (size_t)kStages * BK * (BMT + BNT) * sizeof(float); }

template <int BMT, int BNT>
__global__ void __launch_bounds__(BMT * BNT / 64, 32768 / (BMT * BNT)) gemm_kernel(const float* __restrict__ U,
                                                                 const float* __restrict__ V, float* __restrict__ Mo,
                                                                 int Cp, int Kp, long long Tp) {
  constexpr int BN = BNT;
  constexpr int NT = BMT * BNT / 64;          // threads
  constexpr int AV = BK * BMT / 4 / NT;       // float4 per thread per stage (A)
  constexpr int BV = BK * BN / 4 / NT;        // (B)
  extern __shared__ __align__(16) float gsm[];
  float (*As)[BK][BMT] = reinterpret_cast<float (*)[BK][BMT]>(gsm);
  float (*Bs)[BK][BN] = reinterpret_cast<float (*)[BK][BN]>(gsm + kStages * BK * BMT);
  const int tid = threadIdx.x;
  lpdl_launch_dependents();
  lpdl_wait();   // U (K1, via K2's completion) and V (K2) are complete and visible
  const int tx = tid % (BN / 8), ty = tid / (BN / 8);     // tx < BN / 8, ty < BMT / 8
  const long long t0 = (long long)blockIdx.x * BN;
  const int k0 = blockIdx.y * BMT;
  const int p = blockIdx.z;
  const float* Ap = U + (long long)p * Cp * Kp + k0;
  const float* Bp = V + (long long)p * Cp * Tp + t0;

  u64 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0ull;

  const int nk = Cp / BK;
  auto load = [&](int stage, int kt) {
#pragma unroll
    for (int h = 0; h < AV; h++) {
      const int f = tid + h * NT;               // float4 index in the BK x BMT tile
      const int row = f / (BMT / 4), col = (f % (BMT / 4)) * 4;
      cp_async16(&As[stage][row][col], Ap + ((long long)kt * BK + row) * Kp + col);
    }
#pragma unroll
    for (int h = 0; h < BV; h++) {
      const int f = tid + h * NT;
      const int row = f / (BN / 4), col = (f % (BN / 4)) * 4;
      cp_async16(&Bs[stage][row][col], Bp + ((long long)kt * BK + row) * Tp + col);
    }
  };
#pragma unroll
  for (int st = 0; st < kStages - 1; st++) {
    if (st < nk) load(st, st);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; kt++) {
    cp_async_wait<kStages - 2>();   // stage kt has landed (only the newest kStages - 2 groups may be pending)
    __syncthreads();                // ... for every thread; stage (kt - 1) % kStages was consumed at kt - 1
    if (kt + kStages - 1 < nk) load((kt + kStages - 1) % kStages, kt + kStages - 1);
    cp_async_commit();
    const int cur = kt % kStages;
#pragma unroll
    for (int kk = 0; kk < BK; kk++) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[cur][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[cur][kk][BMT / 2 + ty * 4]);
      const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(&Bs[cur][kk][tx * 4]);
      const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(&Bs[cur][kk][BN / 2 + tx * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const u64 bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = ffma2_bcast(bv[j], av[i], acc[i][j]);
    }
  }
  float* Mp = Mo + (long long)p * Kp * Tp;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const int k = k0 + (i < 4 ? ty * 4 + i : BMT / 2 + ty * 4 + (i - 4));
    float* row = Mp + (long long)k * Tp + t0;
    *reinterpret_cast<ulonglong2*>(row + tx * 4) = make_ulonglong2(acc[i][0], acc[i][1]);
    *reinterpret_cast<ulonglong2*>(row + BN / 2 + tx * 4) = make_ulonglong2(acc[i][2], acc[i][3]);
  }
}

// ------------------------------------------------------------------ K3 variant (NEXT row N3)
// tcgen05 kind::tf32 contraction: tc::gemm_tf32_kernel in tc_gemm.cuh.  NOT the parity path.
using tc::gemm_tf32_kernel;

// ------------------------------------------------------------------ K4
// one thread per (k, t); t fastest -> coalesced M loads per Winograd position.
// Epilogue (network glue of configs[4], fused): with act != NULL the thread also writes
// act = maxpool_pool(ReLU(y)) of its tile (pool 1: ReLU; pool 2: 2 x 2 / 2 max pool, which
// needs an even tile size so no window straddles two tiles -- the launcher only fuses then);
// y itself is written only when y != NULL (the scorer and the caller's `keep` need it).
// ReLU and max are exact, so the fused output equals relu_pool(y) bit for bit.
// EP: the epilogue compiled in -- 0: y only; 1: ReLU activation (y optional); 2: ReLU +
// 2 x 2 max pool (y optional).  One kernel with run-time epilogue branches cost the y-only
// and pooled paths registers / issue slots (measured when the 8-byte ReLU stores were added).
template <int M, int R, int Z, int EP>
__global__ void __launch_bounds__(256, M + R - 1 <= 8 ? 3 : 2) output_kernel(const float* __restrict__ Mw,
                                                                           float* __restrict__ y, Geo geo,
                                                                           const __grid_constant__ LayerMats mt,
                                                                           float* __restrict__ act_in, int) {
  constexpr int N = M + R - 1;
  constexpr int pool = EP == 2 ? 2 : 1;
  float* const act = EP == 0 ? nullptr : act_in;
  lpdl_wait();   // M (K3) is complete and visible
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // over K * T
  if (idx >= (long long)geo.K * geo.T) return;
  const long long t = idx % geo.T;
  const int k = (int)(idx / geo.T);
  const long long plane = (long long)geo.Kp * geo.Tp;
  const float* src = Mw + (long long)k * geo.Tp + t;
  // T3[p][l] = Σ_i Aᵀ[p][i] Mw[i][l]: rows of Mw streamed in ascending i (each (p, l) is
  // still one ascending fmaf chain from +0)
  float t3[M][N];
#pragma unroll
  for (int p = 0; p < M; p++)
#pragma unroll
    for (int l = 0; l < N; l++) t3[p][l] = 0.0f;
#pragma unroll
  for (int i = 0; i < N; i++) {
    float mw[N];
#pragma unroll
    for (int l = 0; l < N; l++) mw[l] = src[(i * N + l) * plane];
#pragma unroll
    for (int p = 0; p < M; p++)
      if (nzA<Z>(p * N + i))
#pragma unroll
        for (int l = 0; l < N; l++) t3[p][l] = __fmaf_rn(mt.AT[p * N + i], mw[l], t3[p][l]);
  }
  const int per_img = geo.th * geo.tw;
  const int img = (int)(t / per_img);
  const int rem = (int)(t - (long long)img * per_img);
  const int ty = rem / geo.tw, tx = rem - ty * geo.tw;
  float* yk = y ? y + ((long long)img * geo.K + k) * geo.Ho * geo.Wo : nullptr;
  const int Hp = geo.Ho / 2, Wp = geo.Wo / 2;   // pool 2 (floor)
  float* ak = act ? act + ((long long)img * geo.K + k) * (pool == 2 ? (long long)Hp * Wp : (long long)geo.Ho * geo.Wo)
                  : nullptr;
  // rows of the output tile; even M with an even row length -> 8-byte pair stores (the
  // lanes of a warp cover consecutive tiles, so a pair store fills 1/3 of a 768 B span
  // instead of 1/6)
  const bool pairs = (M % 2 == 0) && (geo.Wo % 2 == 0) && (reinterpret_cast<uintptr_t>(y) % 8 == 0) &&
                     (reinterpret_cast<uintptr_t>(act) % 8 == 0);
  float prev[M];
#pragma unroll
  for (int p = 0; p < M; p++) {
    const int h = ty * M + p;
    float yr[M];
#pragma unroll
    for (int s = 0; s < M; s++) {
      float acc = 0.0f;
#pragma unroll
      for (int l = 0; l < N; l++)
        if (nzA<Z>(s * N + l)) acc = __fmaf_rn(t3[p][l], mt.AT[s * N + l], acc);
      yr[s] = acc;
    }
    const int wmax = geo.Wo - tx * M;   // valid columns in this tile row
    if (yk != nullptr && h < geo.Ho) {
      float* row = yk + (long long)h * geo.Wo + tx * M;
      if (pairs) {
#pragma unroll
        for (int s = 0; s + 1 < M; s += 2)
          if (s < wmax) *reinterpret_cast<float2*>(row + s) = make_float2(yr[s], yr[s + 1]);
      } else {
#pragma unroll
        for (int s = 0; s < M; s++)
          if (s < wmax) row[s] = yr[s];
      }
    }
    if (EP != 0 && ak != nullptr) {
      if (EP == 1) {
        if (h < geo.Ho) {
          float* row = ak + (long long)h * geo.Wo + tx * M;
          if (pairs) {
#pragma unroll
            for (int s = 0; s + 1 < M; s += 2)
              if (s < wmax)
                *reinterpret_cast<float2*>(row + s) = make_float2(fmaxf(yr[s], 0.0f), fmaxf(yr[s + 1], 0.0f));
          } else {
#pragma unroll
            for (int s = 0; s < M; s++)
              if (s < wmax) row[s] = fmaxf(yr[s], 0.0f);
          }
        }
      } else if (M % 2 == 0) {
        if (p % 2 == 0) {
#pragma unroll
          for (int s = 0; s < M; s++) prev[s] = yr[s];
        } else if (h / 2 < Hp) {
          float* row = ak + (long long)(h / 2) * Wp + tx * (M / 2);
#pragma unroll
          for (int s = 0; s + 1 < M; s += 2)
            if (tx * (M / 2) + s / 2 < Wp)
              row[s / 2] = fmaxf(fmaxf(fmaxf(prev[s], prev[s + 1]), fmaxf(yr[s], yr[s + 1])), 0.0f);
        }
      }
    }
  }
}

// ------------------------------------------------------------------ K2+K3+K4 fused, C <= 4
// First layers (VGG's / CIFAR stacks' RGB input, C = 3): the unfused pipeline pads C to 16
// and round-trips V and M (n² K T floats: 1.5 GB each way for VGG conv1_1 x64) through HBM
// for a 3-term contraction.  Here one thread owns a tile: it transforms its C input patches
// into shared memory (sV [C][n²][128 tiles], conflict-free), then for every PAIR of output
// channels (k, k+1) of the CTA's 16 forms Mw = Σ_c U ⊙ V (ascending c from +0, the
// canonical chain) and the output transform in registers as FFMA2 with the two channels in
// the halves of each register pair, and runs the same crop / ReLU / pool epilogue as K4.
// U pairs of the CTA's channels are staged once ([k pair][c][n² padded to even] u64, read
// as 16-byte broadcasts).  HBM traffic = x + U slice + outputs.  Per element the operations
// and their order are exactly K2 / K3 / K4's (padding channels of K3 add fma(0, 0, acc) =
// acc), so the result is bit-identical to the unfused path and the oracle.
constexpr int kSmcC = 4;     // max input channels
constexpr int kSmcKG = 16;   // output channels per CTA (multiple of 2; divides Kp)
constexpr int kSmcT = 128;   // tiles = threads per CTA

__device__ __forceinline__ void unpack2(u64 v, float& lo, float& hi) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

// one row (P of the tile, image row h) of one output channel: y and / or the fused
// activation; identical to K4's epilogue
template <int M, int P, int EP>
__device__ __forceinline__ void smc_emit_row(const float (&yr)[M], float (&prev)[M], int h, int tx, float* yk, float* ak,
                                             bool pairs, const Geo& geo, int Hp, int Wp) {
  const int wmax = geo.Wo - tx * M;
  if (yk != nullptr && h < geo.Ho) {
    float* row = yk + (long long)h * geo.Wo + tx * M;
    if (pairs) {
#pragma unroll
      for (int s = 0; s + 1 < M; s += 2)
        if (s < wmax) *reinterpret_cast<float2*>(row + s) = make_float2(yr[s], yr[s + 1]);
    } else {
#pragma unroll
      for (int s = 0; s < M; s++)
        if (s < wmax) row[s] = yr[s];
    }
  }
  if (EP != 0 && ak != nullptr) {
    if (EP == 1) {
      if (h < geo.Ho) {
        float* row = ak + (long long)h * geo.Wo + tx * M;
        if (pairs) {   // Wo even and both base pointers 8-byte aligned (checked by the kernel)
#pragma unroll
          for (int s = 0; s + 1 < M; s += 2)
            if (s < wmax) *reinterpret_cast<float2*>(row + s) = make_float2(fmaxf(yr[s], 0.0f), fmaxf(yr[s + 1], 0.0f));
        } else {
#pragma unroll
          for (int s = 0; s < M; s++)
            if (s < wmax) row[s] = fmaxf(yr[s], 0.0f);
        }
      }
    } else if (M % 2 == 0) {
      if (P % 2 == 0) {
#pragma unroll
        for (int s = 0; s < M; s++) prev[s] = yr[s];
      } else if (h / 2 < Hp) {
        float* row = ak + (long long)(h / 2) * Wp + tx * (M / 2);
#pragma unroll
        for (int s = 0; s + 1 < M; s += 2)
          if (tx * (M / 2) + s / 2 < Wp)
            row[s / 2] = fmaxf(fmaxf(fmaxf(prev[s], prev[s + 1]), fmaxf(yr[s], yr[s + 1])), 0.0f);
      }
    }
  }
}

template <int M, int N, int Z, int P, int EP>
__device__ __forceinline__ void smc_rows(const u64 (&t3)[M][N], const LayerMats& mt, float (&prev0)[M], float (&prev1)[M],
                                         int ty, int tx, float* yk0, float* yk1, float* ak0, float* ak1, bool has1,
                                         bool pairs, const Geo& geo, int Hp, int Wp) {
  if constexpr (P < M) {
    float y0[M], y1[M];
#pragma unroll
    for (int s = 0; s < M; s++) {
      u64 acc = 0ull;
#pragma unroll
      for (int l = 0; l < N; l++)
        if (nzA<Z>(s * N + l)) acc = ffma2_bcast(t3[P][l], mt.AT[s * N + l], acc);
      unpack2(acc, y0[s], y1[s]);
    }
    const int h = ty * M + P;
    smc_emit_row<M, P, EP>(y0, prev0, h, tx, yk0, ak0, pairs, geo, Hp, Wp);
    if (has1) smc_emit_row<M, P, EP>(y1, prev1, h, tx, yk1, ak1, pairs, geo, Hp, Wp);
    smc_rows<M, N, Z, P + 1, EP>(t3, mt, prev0, prev1, ty, tx, yk0, yk1, ak0, ak1, has1, pairs, geo, Hp, Wp);
  }
}

template <int N>
constexpr int smc_nnp() { return (N * N + 1) / 2 * 2; }
template <int N>
size_t smc_smem(int C) {
  return (size_t)C * N * N * kSmcT * sizeof(float) + (size_t)(kSmcKG / 2) * C * smc_nnp<N>() * sizeof(u64);
}

template <int M, int R, int Z, int EP>   // EP: K4's epilogue modes (y only / ReLU / ReLU + pool)
__global__ void __launch_bounds__(kSmcT, 2) smallc_kernel(const float* __restrict__ x, const float* __restrict__ U,
                                                         float* __restrict__ y, Geo geo,
                                                         const __grid_constant__ LayerMats mt, float* __restrict__ act_in,
                                                         int) {
  constexpr int N = M + R - 1, NN = N * N, NNP = smc_nnp<N>();
  constexpr int pool = EP == 2 ? 2 : 1;
  float* const act = EP == 0 ? nullptr : act_in;
  extern __shared__ __align__(16) float smc_sm[];
  float* sV = smc_sm;                                                       // [C][NN][kSmcT]
  u64* sU = reinterpret_cast<u64*>(smc_sm + (size_t)geo.C * NN * kSmcT);    // [kSmcKG/2][C][NNP]
  const int tid = threadIdx.x;
  const long long t = (long long)blockIdx.x * kSmcT + tid;
  const int k0 = blockIdx.y * kSmcKG;
  {
    // U [NN][Cp][Kp] -> (k, k+1) pairs; k0 + 2 kp is even and Kp is a multiple of 64, so the
    // 8-byte reads are aligned and stay inside the (zero-filled) padded rows
    const long long uplane = (long long)geo.Cp * geo.Kp;
    for (int idx = tid; idx < (kSmcKG / 2) * geo.C * NNP; idx += kSmcT) {
      const int p = idx % NNP, c = (idx / NNP) % geo.C, kp = idx / (NNP * geo.C);
      sU[idx] = p < NN ? *reinterpret_cast<const u64*>(U + (long long)p * uplane + (long long)c * geo.Kp + k0 + 2 * kp)
                       : 0ull;
    }
  }
  const bool tile_ok = t < geo.T;
  int ty = 0, tx = 0, img = 0;
  if (tile_ok) {
    const int per_img = geo.th * geo.tw;
    img = (int)(t / per_img);
    const int rem = (int)(t - (long long)img * per_img);
    ty = rem / geo.tw;
    tx = rem - ty * geo.tw;
    const int h0 = ty * M - geo.pad, w0 = tx * M - geo.pad;
    unsigned rowm = 0, colm = 0;
#pragma unroll
    for (int a = 0; a < N; a++) rowm |= (h0 + a >= 0 && h0 + a < geo.H) ? 1u << a : 0u;
#pragma unroll
    for (int b = 0; b < N; b++) colm |= (w0 + b >= 0 && w0 + b < geo.W) ? 1u << b : 0u;
    const long long off0 = (long long)h0 * geo.W + w0;
#pragma unroll 1
    for (int c = 0; c < geo.C; c++) {
      const float* xc = x + ((long long)img * geo.C + c) * geo.H * geo.W + off0;
      float d[N][N];
#pragma unroll
      for (int a = 0; a < N; a++)
#pragma unroll
        for (int b = 0; b < N; b++)
          d[a][b] = ((rowm >> a) & (colm >> b) & 1u) ? __ldg(xc + (long long)a * geo.W + b) : 0.0f;
      float t2[N][N];
#pragma unroll
      for (int q = 0; q < N; q++)
#pragma unroll
        for (int i = 0; i < N; i++) {
          float acc = 0.0f;
#pragma unroll
          for (int j = 0; j < N; j++)
            if (nzB<Z>(i * N + j)) acc = __fmaf_rn(mt.BT[i * N + j], d[j][q], acc);
          t2[i][q] = acc;
        }
      float* dst = sV + (size_t)c * NN * kSmcT + tid;
#pragma unroll
      for (int i = 0; i < N; i++)
#pragma unroll
        for (int l = 0; l < N; l++) {
          float acc = 0.0f;
#pragma unroll
          for (int q = 0; q < N; q++)
            if (nzB<Z>(l * N + q)) acc = __fmaf_rn(t2[i][q], mt.BT[l * N + q], acc);
          dst[(i * N + l) * kSmcT] = acc;
        }
    }
  }
  __syncthreads();
  if (!tile_ok) return;
  const int Hp = geo.Ho / 2, Wp = geo.Wo / 2;
  const bool pairs = (M % 2 == 0) && (geo.Wo % 2 == 0) && (reinterpret_cast<uintptr_t>(y) % 8 == 0) &&
                     (reinterpret_cast<uintptr_t>(act) % 8 == 0);
  const long long ysz = (long long)geo.Ho * geo.Wo, asz = pool == 2 ? (long long)Hp * Wp : ysz;
  const float* sv = sV + tid;
#pragma unroll 1
  for (int kp = 0; kp < kSmcKG / 2; kp++) {
    const int k = k0 + 2 * kp;
    if (k >= geo.K) break;
    const u64* su = sU + (size_t)kp * geo.C * NNP;
    u64 t3[M][N];
#pragma unroll
    for (int p = 0; p < M; p++)
#pragma unroll
      for (int l = 0; l < N; l++) t3[p][l] = 0ull;
#pragma unroll
    for (int i = 0; i < N; i++) {
      u64 mw[N];
#pragma unroll
      for (int l = 0; l < N; l++) mw[l] = 0ull;
#pragma unroll
      for (int c = 0; c < kSmcC; c++) {
        if (c < geo.C) {
          // U pairs of positions i N .. i N + N - 1 as 16-byte broadcast loads (even position
          // pairs; NNP is even, so every channel row starts 16-byte aligned)
          const u64* suc = su + c * NNP;
          const float* svc = sv + (size_t)c * NN * kSmcT;
#pragma unroll
          for (int j = (i * N) / 2; j <= (i * N + N - 1) / 2; j++) {
            const ulonglong2 u2 = *reinterpret_cast<const ulonglong2*>(suc + 2 * j);
            const int q0 = 2 * j, q1 = 2 * j + 1;
            if (q0 >= i * N && q0 < i * N + N) {
              const float v = svc[q0 * kSmcT];
              mw[q0 - i * N] = ffma2_bcast(u2.x, v, mw[q0 - i * N]);
            }
            if (q1 >= i * N && q1 < i * N + N) {
              const float v = svc[q1 * kSmcT];
              mw[q1 - i * N] = ffma2_bcast(u2.y, v, mw[q1 - i * N]);
            }
          }
        }
      }
#pragma unroll
      for (int p = 0; p < M; p++)
        if (nzA<Z>(p * N + i))
#pragma unroll
          for (int l = 0; l < N; l++) t3[p][l] = ffma2_bcast(mw[l], mt.AT[p * N + i], t3[p][l]);
    }
    const bool k1 = k + 1 < geo.K;
    float* yk0 = y ? y + ((long long)img * geo.K + k) * ysz : nullptr;
    float* yk1 = (y && k1) ? yk0 + ysz : nullptr;
    float* ak0 = act ? act + ((long long)img * geo.K + k) * asz : nullptr;
    float* ak1 = (act && k1) ? ak0 + asz : nullptr;
    float prev0[M], prev1[M];
    smc_rows<M, N, Z, 0, EP>(t3, mt, prev0, prev1, ty, tx, yk0, yk1, ak0, ak1, k1, pairs, geo, Hp, Wp);
  }
}

// ------------------------------------------------------------------ K5 scoring
// fp64 direct valid correlation of the same fp32 x, w (eq:conv P:112, O7), compared with
// the Winograd output y.  Each thread owns a 2 x 2 block of output positions for
// 16 output channels (64 fp64 accumulators): per (channel, filter row u) it reads its
// 2 x (R + 1) input values once and reuses them for the R filter columns, and every weight
// (a shared-memory broadcast) feeds 4 DFMAs -- about 1 shared-memory load per 6 DFMA.  A CTA
// covers BR x BC such blocks, with BC = min(ceil(Wo / 2), 32) and BR = min(128 / BC,
// ceil(Ho / 2)) chosen at launch so the CTA region tiles the image with little waste
// (56 x 56: 28 x 4 blocks, no waste).  Per input channel the x patch (converted to fp64) and
// the 16 filters are staged in double-buffered shared memory, channel c + 1 fetched into
// registers while channel c is accumulated.  Every accumulator is one chain in the oracle's
// order (Σ_c Σ_u Σ_v ascending).  Statistics: warp butterflies, then a fixed-order
// combination of the warps -> one partial per CTA (deterministic; CTAs ordered image-major).
constexpr int kScK = 16;        // output channels per CTA
constexpr int kScThreads = 128;

struct ScoreTile {
  int BR, BC, tiles_h, tiles_w;
};
int score_threads(const ScoreTile& t) { return std::max(64, (t.BR * t.BC + 31) / 32 * 32); }
ScoreTile score_tile(const Geo& g) {
  ScoreTile t;
  const int bh = (g.Ho + 1) / 2, bw = (g.Wo + 1) / 2;
  t.BC = std::min(bw, 32);
  t.BR = std::max(1, std::min(kScThreads / t.BC, bh));
  // the staging registers hold <= 8 patch values per thread
  while (t.BR > 1 && (2 * t.BR + g.r - 1) * (2 * t.BC + g.r - 1) > 8 * score_threads(t)) t.BR--;
  t.tiles_h = (bh + t.BR - 1) / t.BR;
  t.tiles_w = (bw + t.BC - 1) / t.BC;
  return t;
}
size_t score_smem(const ScoreTile& t, int r) {
  const int PH = 2 * t.BR + r - 1, PW = 2 * t.BC + r - 1;
  return (size_t)2 * (PH * PW + r * r * kScK) * sizeof(double) + 4 * 8 * sizeof(double);
}

template <int R>
__global__ void __launch_bounds__(kScThreads, 2) score_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                                            const float* __restrict__ y, Geo geo, ScoreTile st,
                                                            double* __restrict__ partial) {
  const int BR = st.BR, BC = st.BC;
  const int PH = 2 * BR + R - 1, PW = 2 * BC + R - 1, PATCH = PH * PW;
  extern __shared__ __align__(16) double ssm[];
  double* sx = ssm;                        // [2][PATCH]
  double* sw = sx + 2 * PATCH;             // [2][R*R][kScK]
  double* red = sw + 2 * R * R * kScK;     // [4 warps][8]
  const int tid = threadIdx.x;
  const int nthr = blockDim.x;
  const bool active = tid < BR * BC;
  const int br = active ? tid / BC : 0, bc = active ? tid - (tid / BC) * BC : 0;
  const int h0 = (blockIdx.x / st.tiles_w) * 2 * BR, w0 = (blockIdx.x % st.tiles_w) * 2 * BC;
  const int k0 = blockIdx.y * kScK, img = blockIdx.z;
  constexpr int XMAX = 8, WMAX = (kScK * R * R + 63) / 64;   // staged values per thread (<= PATCH / 64)
  // channel-independent staging geometry, computed once (no integer divisions per channel):
  // x: offset inside the channel plane (-1 = zero padding / beyond the patch); w: offset
  // relative to channel 0 (-1 = beyond the CTA's channels) and the shared-memory slot
  int xoff[XMAX], woff[WMAX], wslot[WMAX];
#pragma unroll
  for (int q = 0; q < XMAX; q++) {
    const int idx = tid + q * nthr;
    const int a = idx / PW, b = idx - a * PW;
    const int hh = h0 - geo.pad + a, wx = w0 - geo.pad + b;
    xoff[q] = (idx < PATCH && hh >= 0 && hh < geo.H && wx >= 0 && wx < geo.W) ? hh * geo.W + wx : -1;
  }
#pragma unroll
  for (int q = 0; q < WMAX; q++) {
    const int idx = tid + q * nthr;
    const int kk = idx / (R * R), e = idx - kk * (R * R);
    woff[q] = (idx < kScK * R * R && k0 + kk < geo.K) ? (k0 + kk) * geo.C * R * R + e : -1;
    wslot[q] = idx < kScK * R * R ? e * kScK + kk : -1;
  }
  float xr[XMAX], wr[WMAX];
  auto fetch = [&](int c) {
    const float* xc = x + ((long long)img * geo.C + c) * geo.H * geo.W;
#pragma unroll
    for (int q = 0; q < XMAX; q++) xr[q] = xoff[q] >= 0 ? __ldg(xc + xoff[q]) : 0.0f;
#pragma unroll
    for (int q = 0; q < WMAX; q++) wr[q] = woff[q] >= 0 ? __ldg(w + woff[q] + (long long)c * R * R) : 0.0f;
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < XMAX; q++) {
      const int idx = tid + q * nthr;
      if (idx < PATCH) sx[buf * PATCH + idx] = (double)xr[q];
    }
#pragma unroll
    for (int q = 0; q < WMAX; q++)
      if (wslot[q] >= 0) sw[buf * R * R * kScK + wslot[q]] = (double)wr[q];
  };
  double acc[kScK][4];   // [k][2 * rho + j]: output (h0 + 2 br + rho, w0 + 2 bc + j)
#pragma unroll
  for (int k = 0; k < kScK; k++)
#pragma unroll
    for (int p = 0; p < 4; p++) acc[k][p] = 0.0;
  if (geo.C > 0) {
    fetch(0);
    store(0);
  }
  __syncthreads();
  for (int c = 0; c < geo.C; c++) {
    const int buf = c & 1;
    if (c + 1 < geo.C) fetch(c + 1);
    if (active) {
      const double* px = sx + buf * PATCH + (2 * br) * PW + 2 * bc;
      const double* pw = sw + buf * R * R * kScK;
#pragma unroll
      for (int u = 0; u < R; u++) {
        double xv[2][R + 1];
#pragma unroll
        for (int rho = 0; rho < 2; rho++)
#pragma unroll
          for (int j = 0; j <= R; j++) xv[rho][j] = px[(rho + u) * PW + j];
#pragma unroll
        for (int v = 0; v < R; v++) {
#pragma unroll
          for (int k2 = 0; k2 < kScK / 2; k2++) {
            const double2 wv = *reinterpret_cast<const double2*>(pw + (u * R + v) * kScK + 2 * k2);
#pragma unroll
            for (int rho = 0; rho < 2; rho++)
#pragma unroll
              for (int j = 0; j < 2; j++) {
                acc[2 * k2][2 * rho + j] = __fma_rn(wv.x, xv[rho][j + v], acc[2 * k2][2 * rho + j]);
                acc[2 * k2 + 1][2 * rho + j] = __fma_rn(wv.y, xv[rho][j + v], acc[2 * k2 + 1][2 * rho + j]);
              }
          }
        }
      }
    }
    if (c + 1 < geo.C) store(buf ^ 1);
    __syncthreads();
  }
  double s0 = 0, s1 = 0, s2 = 0, m0 = 0, m1 = 0, n = 0, nf = 0;
  if (active) {
#pragma unroll
    for (int rho = 0; rho < 2; rho++)
#pragma unroll
      for (int j = 0; j < 2; j++) {
        const int h = h0 + 2 * br + rho, ww = w0 + 2 * bc + j;
        if (h >= geo.Ho || ww >= geo.Wo) continue;
#pragma unroll
        for (int k = 0; k < kScK; k++) {
          if (k0 + k >= geo.K) break;
          const double r = acc[k][2 * rho + j];
          const double e = (double)y[(((long long)img * geo.K + k0 + k) * geo.Ho + h) * geo.Wo + ww] - r;
          s2 += fabs(r);
          m1 = fmax(m1, fabs(r));
          if (isfinite(e)) {
            s0 += fabs(e);
            s1 = __fma_rn(e, e, s1);
            m0 = fmax(m0, fabs(e));
            n += 1.0;
          } else {
            nf += 1.0;
          }
        }
      }
  }
  double v[7] = {s0, s1, s2, n, nf, m0, m1};
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int f = 0; f < 5; f++) v[f] += __shfl_xor_sync(0xffffffffu, v[f], off);
    v[5] = fmax(v[5], __shfl_xor_sync(0xffffffffu, v[5], off));
    v[6] = fmax(v[6], __shfl_xor_sync(0xffffffffu, v[6], off));
  }
  if ((tid & 31) == 0)
    for (int f = 0; f < 7; f++) red[(tid >> 5) * 8 + f] = v[f];
  __syncthreads();
  if (tid == 0) {
    double t[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int wi = 0; wi < nthr / 32; wi++) {
      for (int f = 0; f < 5; f++) t[f] += red[wi * 8 + f];
      t[5] = fmax(t[5], red[wi * 8 + 5]);
      t[6] = fmax(t[6], red[wi * 8 + 6]);
    }
    const long long blk = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    double* p = partial + blk * 8;
    for (int f = 0; f < 7; f++) p[f] = t[f];
    p[7] = 0.0;
  }
}

__global__ void score_finalize_kernel(const double* __restrict__ partial, int n_entries, double* d_sums,
                                      double* d_maxs) {
  const int lane = threadIdx.x;
  partial += (long long)blockIdx.x * n_entries * 8;
  d_sums += (long long)blockIdx.x * WINO_SUMS;
  d_maxs += (long long)blockIdx.x * WINO_MAXS;
  double v[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int e = lane; e < n_entries; e += 32) {
#pragma unroll
    for (int f = 0; f < 5; f++) v[f] += partial[e * 8 + f];
    v[5] = fmax(v[5], partial[e * 8 + 5]);
    v[6] = fmax(v[6], partial[e * 8 + 6]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int f = 0; f < 5; f++) v[f] += __shfl_xor_sync(0xffffffffu, v[f], off);
    v[5] = fmax(v[5], __shfl_xor_sync(0xffffffffu, v[5], off));
    v[6] = fmax(v[6], __shfl_xor_sync(0xffffffffu, v[6], off));
  }
  if (lane == 0) {
    for (int f = 0; f < 5; f++) d_sums[f] += v[f];
    d_maxs[0] = fmax(d_maxs[0], v[5]);
    d_maxs[1] = fmax(d_maxs[1], v[6]);
  }
}

// ------------------------------------------------------------------ K9 ReLU (+ 2x2/2 max pool)
// Network glue of BASELINE.json configs[4] (VGG-16: "ReLU + 2x2 maxpool").  Both are exact
// operations (max, and the sign test), so they add no rounding.  pool = 1: ReLU only.
// pool = 1: flat ReLU, float4 grid-stride; pool = 2: one warp per output row (n, c, h),
// index arithmetic once per row, lanes over the row's columns (float2 loads of the two
// input rows).
__global__ void relu_kernel(const float4* __restrict__ x, float4* __restrict__ y, long long n4) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = __ldg(x + i);
    y[i] = make_float4(fmaxf(v.x, 0.0f), fmaxf(v.y, 0.0f), fmaxf(v.z, 0.0f), fmaxf(v.w, 0.0f));
  }
}

__global__ void relu_pool1_scalar_kernel(const float* __restrict__ x, float* __restrict__ y, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = fmaxf(__ldg(x + i), 0.0f);
}

__global__ void relu_pool2_kernel(const float* __restrict__ x, float* __restrict__ y, long long rows, int H, int W) {
  const int Ho = H / 2, Wo = W / 2;
  const long long row = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const long long nc = row / Ho;
  const int h = (int)(row - nc * Ho);
  const float* r0 = x + (nc * H + 2 * h) * W;
  const float* r1 = r0 + W;
  float* dst = y + row * Wo;
  for (int w = threadIdx.x & 31; w < Wo; w += 32) {
    const float a = fmaxf(__ldg(r0 + 2 * w), __ldg(r0 + 2 * w + 1));
    const float b = fmaxf(__ldg(r1 + 2 * w), __ldg(r1 + 2 * w + 1));
    dst[w] = fmaxf(fmaxf(a, b), 0.0f);   // ReLU then max == max then ReLU (monotone)
  }
}

// ------------------------------------------------------------------ dispatch
typedef void (*FilterK)(const float*, float*, int, int, int, int, int, LayerMats);
typedef void (*InputK)(const float*, float*, Geo, LayerMats);
typedef void (*OutputK)(const float*, float*, Geo, LayerMats, float*, int);
typedef void (*ScoreK)(const float*, const float*, const float*, Geo, ScoreTile, double*);
typedef void (*SmallCK)(const float*, const float*, float*, Geo, LayerMats, float*, int);
typedef size_t (*SmallCSmem)(int);

// transform kernels of one structural-zero family Z (0 = dense)
struct XformK {
  int z;
  uint64_t za[2], zb[2];   // skipped entries of Aᵀ / Bᵀ (zero_masks.h)
  InputK ik[3];           // by Geo::tf32
  OutputK ok[3];          // by epilogue: y only / ReLU / ReLU + pool
  SmallCK sck[3];         // fused C <= kSmcC kernel by epilogue (NULL: not compiled for this shape)
  SmallCSmem sck_smem;
};

struct LayerCfg {
  int m, r;
  FilterK fk;
  ScoreK sk;
  XformK xk[2];   // most specialised first, dense last
  int nxk;
};

template <int M, int R, int Z>
XformK make_xform_k() {
  static_assert(Z == 0 || (ZM<Z>::m == M && ZM<Z>::r == R), "zero-mask family of another shape");
  XformK v;
  v.z = Z;
  for (int w = 0; w < 2; w++) {
    v.za[w] = ZM<Z>::A(w);
    v.zb[w] = ZM<Z>::B(w);
  }
  v.ik[0] = input_kernel<M, R, Z, 0>;
  v.ik[1] = input_kernel<M, R, Z, 1>;
  v.ik[2] = input_kernel<M, R, Z, 2>;
  v.ok[0] = output_kernel<M, R, Z, 0>;
  v.ok[1] = output_kernel<M, R, Z, 1>;
  v.ok[2] = output_kernel<M, R, Z, 2>;
  v.sck[0] = v.sck[1] = v.sck[2] = nullptr;
  v.sck_smem = nullptr;
  if constexpr (R == 3 && M + R - 1 <= 8) {   // the first layers of the 3 x 3 stacks
    v.sck[0] = smallc_kernel<M, R, Z, 0>;
    v.sck[1] = smallc_kernel<M, R, Z, 1>;
    v.sck[2] = smallc_kernel<M, R, Z, 2>;
    v.sck_smem = smc_smem<M + R - 1>;
  }
  return v;
}

// ZF: the structural-zero family compiled for this shape (0: dense only)
template <int M, int R, int ZF = 0>
LayerCfg make_layer_cfg() {
  LayerCfg c{M, R, filter_kernel<M, R>, score_kernel<R>, {}, 0};
  if constexpr (ZF != 0) c.xk[c.nxk++] = make_xform_k<M, R, ZF>();
  c.xk[c.nxk++] = make_xform_k<M, R, 0>();
  return c;
}

dim3 score_grid(const Geo& g) {
  const ScoreTile t = score_tile(g);
  return dim3((unsigned)(t.tiles_h * t.tiles_w), (unsigned)((g.K + kScK - 1) / kScK), (unsigned)g.N);
}

// F(m x m, 3 x 3) for m = 2..8 (n = 4..10: the paper's T7-T9 sizes) and the
// 5 x 5 kernels of configs[3]
const LayerCfg kLayerCfgs[] = {
    make_layer_cfg<2, 3, kZ_F23_C>(), make_layer_cfg<3, 3>(), make_layer_cfg<4, 3, kZ_F43_C>(),
    make_layer_cfg<5, 3>(), make_layer_cfg<6, 3, kZ_N8_CD>(), make_layer_cfg<7, 3>(), make_layer_cfg<8, 3, kZ_N10_C1C2>(),
    make_layer_cfg<2, 5>(), make_layer_cfg<4, 5, kZ_N8_C1C2_R5>(), make_layer_cfg<6, 5, kZ_N10_C1C2_R5>(),
};

// The transform kernels for these fp32 matrices: the first variant whose skipped Aᵀ / Bᵀ
// entries are all exactly zero.  Families are used only for moderate coefficients
// (|a| < 2^32): skipping a zero term equals the dense chain while no intermediate overflows
// (finite x, w), and huge coefficients are the likely overflow source; the dense variant
// takes the rest.
const XformK& pick_xform(const LayerCfg& cfg, const LayerMats& mt, int m, int n) {
  uint64_t nzA[2] = {0, 0}, nzB[2] = {0, 0};
  bool moderate = true;
  for (int t = 0; t < m * n; t++) {
    if (mt.AT[t] != 0.0f) nzA[t >> 6] |= 1ull << (t & 63);
    moderate = moderate && std::fabs(mt.AT[t]) < 4294967296.0f;
  }
  for (int t = 0; t < n * n; t++) {
    if (mt.BT[t] != 0.0f) nzB[t >> 6] |= 1ull << (t & 63);
    moderate = moderate && std::fabs(mt.BT[t]) < 4294967296.0f;
  }
  for (int v = 0; v + 1 < cfg.nxk; v++) {
    const XformK& k = cfg.xk[v];
    if (moderate && (k.za[0] & nzA[0]) == 0 && (k.za[1] & nzA[1]) == 0 && (k.zb[0] & nzB[0]) == 0 &&
        (k.zb[1] & nzB[1]) == 0)
      return k;
  }
  return cfg.xk[cfg.nxk - 1];
}

const LayerCfg* find_layer(int m, int r) {
  for (const auto& c : kLayerCfgs)
    if (c.m == m && c.r == r) return &c;
  return nullptr;
}

struct WsLayout {
  size_t u_off, v_off, m_off, p_off, total;
};

// per-thread, per-device side stream + fork/join events for layer_launch
struct SideStream {
  bool ok = false;
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_stream() {
  thread_local SideStream per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& ss = per_dev[dev & 63];
  if (!ss.ok && ss.s == nullptr) {
    ss.ok = cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) == cudaSuccess;
  }
  return ss;
}

WsLayout ws_layout(const Geo& g) {
  const int n = g.m + g.r - 1, nn = n * n;
  WsLayout L;
  L.u_off = 0;
  const size_t planes = g.tf32 == 2 ? 2 : 1;   // 3xTF32: hi and lo planes of U and V
  L.v_off = L.u_off + align_up(planes * nn * g.Cp * g.Kp * sizeof(float), 256);
  L.m_off = L.v_off + align_up(planes * nn * g.Cp * g.Tp * sizeof(float), 256);
  L.p_off = L.m_off + align_up((size_t)nn * g.Kp * g.Tp * sizeof(float), 256);
  const dim3 sg = score_grid(g);
  L.total = L.p_off + align_up((size_t)sg.x * sg.y * sg.z * 8 * sizeof(double), 256);
  return L;
}

}  // namespace

int relu_pool_launch(const float* x, float* y, int N, int C, int H, int W, int pool, cudaStream_t stream) {
  const long long total = (long long)N * C * (H / pool) * (W / pool);
  int launches = 0;
  if (total > 0) {
    if (pool == 1 && total % 4 == 0 && ((uintptr_t)x % 16) == 0 && ((uintptr_t)y % 16) == 0) {
      timed_launch("relu_pool", stream, [&] {
        relu_kernel<<<148 * 16, 256, 0, stream>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y),
                                                  total / 4);
      });
    } else if (pool == 1) {
      // unaligned or ragged: treat as pool-1 rows through the row kernel's scalar path
      timed_launch("relu_pool", stream, [&] {
        relu_pool1_scalar_kernel<<<148 * 16, 256, 0, stream>>>(x, y, total);
      });
    } else {
      const long long rows = (long long)N * C * (H / 2);
      timed_launch("relu_pool", stream, [&] {
        relu_pool2_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, stream>>>(x, y, rows, H, W);
      });
    }
    launches = 1;
  }
  count_launches(launches);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(WINO_E_CUDA, "relu_pool launch: %s", cudaGetErrorString(e));
  return WINO_OK;
}

int layer_supported(int m, int r) { return find_layer(m, r) != nullptr; }

size_t layer_workspace_bytes(int N, int C, int H, int W, int K, int r, int pad, int m) {
  // large enough for the FFMA path and the tcgen05 variant's alignments
  return std::max(ws_layout(make_geo(N, C, H, W, K, r, pad, m, 0)).total,
                  ws_layout(make_geo(N, C, H, W, K, r, pad, m, 2)).total);
}

// which kernel layer_launch picks for the parity path (wino_conv2d_gemm_tile)
int layer_gemm_tile(int N, int C, int H, int W, int K, int r, int pad, int m) {
  const LayerCfg* cfg = find_layer(m, r);
  if (!cfg) return 0;
  const bool no_smallc = std::getenv("WINO_LAYER_NO_SMALLC") != nullptr;
  if (!no_smallc && C <= kSmcC && cfg->xk[0].sck[0] != nullptr && cfg->xk[0].sck_smem(C) <= 200 * 1024) return 1;
  const Geo g = make_geo(N, C, H, W, K, r, pad, m, 0);
  return g.Kp == 64 ? 64128 : 128000 + g.bn;
}

int layer_launch(const float* x, const float* w, float* y, int N, int C, int H, int W, int K, int r, int pad,
                 int m, const float* AT, const float* G, const float* BT, void* workspace, size_t ws_bytes,
                 double* d_sums, double* d_maxs, unsigned flags, cudaStream_t stream, float* act, int pool) {
  const LayerCfg* cfg = find_layer(m, r);
  if (!cfg) return set_error(WINO_E_UNSUPPORTED, "no layer kernel for m=%d r=%d", m, r);
  const int tf32 = (flags & WINO_CONV_3XTF32) ? 2 : (flags & WINO_CONV_TF32) ? 1 : 0;
  const Geo g = make_geo(N, C, H, W, K, r, pad, m, tf32);
  const WsLayout L = ws_layout(g);
  if (!workspace || ws_bytes < L.total)
    return set_error(WINO_E_WORKSPACE, "layer workspace %zu < %zu bytes", ws_bytes, L.total);
  const int n = m + r - 1;
  LayerMats mt;
  std::fill(mt.AT, mt.AT + kMaxN * kMaxN, 0.0f);
  std::fill(mt.G, mt.G + kMaxN * kMaxN, 0.0f);
  std::fill(mt.BT, mt.BT + kMaxN * kMaxN, 0.0f);
  std::copy(AT, AT + m * n, mt.AT);
  std::copy(G, G + n * r, mt.G);
  std::copy(BT, BT + n * n, mt.BT);
  const XformK& xk = pick_xform(*cfg, mt, m, n);
  char* ws = reinterpret_cast<char*>(workspace);
  float* U = reinterpret_cast<float*>(ws + L.u_off);
  float* V = reinterpret_cast<float*>(ws + L.v_off);
  float* Mw = reinterpret_cast<float*>(ws + L.m_off);
  double* partial = reinterpret_cast<double*>(ws + L.p_off);
  const int tpb = 256;
  int launches = 0;
  // K1 (filter) and K2 (input) are independent: K1 runs on a per-thread, per-device side
  // stream forked from / joined to `stream` with events (graph-capture compatible), so the
  // small filter transform hides under the input transform.
  // C <= 4 (RGB first layers): K2 + K3 + K4 fused in one kernel after K1 (smallc_kernel);
  // WINO_LAYER_NO_SMALLC=1 forces the unfused pipeline (A/B measurements, parity tests)
  const bool no_smallc = std::getenv("WINO_LAYER_NO_SMALLC") != nullptr;
  const bool smallc = !tf32 && !no_smallc && C <= kSmcC && xk.sck[0] != nullptr && xk.sck_smem(C) <= 200 * 1024;
  // Unfused fp32 path: K1 -> K2 -> K3 -> K4 as a programmatic-dependent-launch chain on
  // `stream` (lpdl_wait above; K2 runs beside K1 without a side stream, K3 / K4 become
  // resident while their predecessor drains).  The timing hook records events between the
  // launches, which would serialise them, so with the hook on (and for the TF32 variants,
  // whose GEMM has no wait) the kernels are launched plainly with K1 on the side stream.
  // n > 8: the input transform runs one 256-thread CTA per SM in < 2 waves; started behind
  // K1's CTAs instead of racing them from another stream it takes an extra wave (configs[3]
  // n = 10: 0.205 ms plain, 0.215 ms chained), so those shapes keep the side stream.
  const bool pdl = !tf32 && !smallc && !timing_enabled() && (m + r - 1) <= 8 &&
                   std::getenv("WINO_LAYER_NO_PDL") == nullptr;
  SideStream& side = side_stream();
  bool forked = !smallc && !pdl && side.ok && cudaEventRecord(side.fork, stream) == cudaSuccess &&
                cudaStreamWaitEvent(side.s, side.fork, 0) == cudaSuccess;
  cudaStream_t fs = forked ? side.s : stream;
  {
    const long long tot = (long long)g.Cp * g.Kp;
    const auto fk = cfg->fk;
    timed_launch("layer_filter", fs,
                 [&] { fk<<<(unsigned)((tot + tpb - 1) / tpb), tpb, 0, fs>>>(w, U, C, K, g.Cp, g.Kp, g.tf32, mt); });
    launches++;
  }
  if (forked) cudaEventRecord(side.join, fs);
  if (smallc) {
    const size_t smem = xk.sck_smem(C);
    const bool fuse = act != nullptr && (pool == 1 || m % 2 == 0);
    const auto sck = xk.sck[fuse ? (pool == 2 ? 2 : 1) : 0];
    cudaFuncSetAttribute((const void*)sck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)((g.T + kSmcT - 1) / kSmcT), (unsigned)((K + kSmcKG - 1) / kSmcKG));
    timed_launch("layer_smallc", stream,
                 [&] { sck<<<grid, kSmcT, smem, stream>>>(x, U, y, g, mt, fuse ? act : nullptr, pool); });
    launches++;
  }
  if (!smallc) {
    const int cpt = (m + r - 1) > 8 ? 4 : 1;   // = in_cpt<N>() of the kernel
    const long long tot = (long long)(g.Cp / cpt) * g.Tp;
    const auto ik = xk.ik[g.tf32];
    const dim3 igrid((unsigned)((tot + tpb - 1) / tpb));
    timed_launch("layer_input", stream, [&] {
      if (pdl)
        launch_k(ik, igrid, dim3(tpb), 0, stream, true, x, V, g, mt);
      else
        ik<<<igrid, tpb, 0, stream>>>(x, V, g, mt);
    });
    launches++;
  }
  if (forked) cudaStreamWaitEvent(stream, side.join, 0);
  if (!smallc) {
    if (tf32) {
      // per call (cheap), so several devices / host threads in one process stay correct
      const auto kern = tf32 == 2 ? gemm_tf32_kernel<3> : gemm_tf32_kernel<1>;
      const int smem = tf32 == 2 ? tc::Cfg<3>::kSmem : tc::Cfg<1>::kSmem;
      cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int dev = 0, n_sm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
      const long long tiles = (long long)(n * n) * (g.Kp / tc::kM) * (g.Tp / tc::kN);
      const unsigned grid = (unsigned)std::min<long long>(tiles, n_sm);
      CUtensorMap tmU, tmV, tmUl, tmVl, tmM;
      const unsigned long long pc = (unsigned long long)(n * n) * g.Cp, pk = (unsigned long long)(n * n) * g.Kp;
      const float* Ul = U + (size_t)(n * n) * g.Cp * g.Kp;   // lo planes (3xTF32)
      const float* Vl = V + (size_t)(n * n) * g.Cp * g.Tp;
      bool enc = tc::encode_map_2d(&tmU, U, (unsigned long long)g.Kp, pc, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) &&
                 tc::encode_map_2d(&tmV, V, (unsigned long long)g.Tp, pc, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) &&
                 tc::encode_map_2d(&tmM, Mw, (unsigned long long)g.Tp, pk, CU_TENSOR_MAP_SWIZZLE_128B);
      if (tf32 == 2)
        enc = enc && tc::encode_map_2d(&tmUl, Ul, (unsigned long long)g.Kp, pc, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) &&
              tc::encode_map_2d(&tmVl, Vl, (unsigned long long)g.Tp, pc, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
      else
        tmUl = tmU, tmVl = tmV;
      if (!enc) return set_error(WINO_E_CUDA, "cuTensorMapEncodeTiled failed for the tf32 contraction");
      timed_launch(tf32 == 2 ? "layer_gemm_3xtf32" : "layer_gemm_tf32", stream, [&] {
        kern<<<grid, tc::kThreads, smem, stream>>>(tmU, tmV, tmUl, tmVl, tmM, g.Cp, g.Kp, g.Tp, n * n);
      });
    } else {
      auto run_gemm = [&](auto kern, int threads, size_t smem, unsigned kblocks, int bn) {
        dim3 grid((unsigned)(g.Tp / bn), kblocks, (unsigned)(n * n));
        cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        timed_launch("layer_gemm", stream, [&] {
          if (pdl)
            launch_k(kern, grid, dim3(threads), smem, stream, true, U, V, Mw, g.Cp, g.Kp, g.Tp);
          else
            kern<<<grid, threads, smem, stream>>>(U, V, Mw, g.Cp, g.Kp, g.Tp);
        });
      };
      if (g.Kp == 64)
        run_gemm(gemm_kernel<64, 128>, 128, gemm_smem<64, 128>(), 1u, 128);
      else if (g.bn == 64)
        run_gemm(gemm_kernel<128, 64>, 128, gemm_smem<128, 64>(), (unsigned)(g.Kp / 128), 64);
      else
        run_gemm(gemm_kernel<128, 128>, 256, gemm_smem<128, 128>(), (unsigned)(g.Kp / 128), 128);
    }
    launches++;
  }
  if (!smallc) {
    const long long tot = (long long)g.K * g.T;
    // fused ReLU (+ 2 x 2 pool for even m) epilogue; odd m with pool 2 runs the separate
    // ReLU / pool kernel on y after the layer
    const bool fuse = act != nullptr && (pool == 1 || m % 2 == 0);
    const auto ok = xk.ok[fuse ? (pool == 2 ? 2 : 1) : 0];
    const dim3 ogrid((unsigned)((tot + tpb - 1) / tpb));
    timed_launch("layer_output", stream, [&] {
      if (pdl)
        launch_k(ok, ogrid, dim3(tpb), 0, stream, true, Mw, y, g, mt, fuse ? act : nullptr, pool);
      else
        ok<<<ogrid, tpb, 0, stream>>>(Mw, y, g, mt, fuse ? act : nullptr, pool);
    });
    launches++;
  }
  if (d_sums) {
    const dim3 sg = score_grid(g);
    const auto sk = cfg->sk;
    const ScoreTile st = score_tile(g);
    const size_t ssm = score_smem(st, r);
    timed_launch("layer_score", stream,
                 [&] { sk<<<sg, score_threads(st), ssm, stream>>>(x, w, y, g, st, partial); });
    // partials are ordered image-major (blockIdx.z = image), so per-image rows are contiguous
    const bool per_image = (flags & WINO_CONV_SCORE_PER_IMAGE) != 0;
    const unsigned rows = per_image ? sg.z : 1u;
    const int entries = (int)(per_image ? sg.x * sg.y : sg.x * sg.y * sg.z);
    timed_launch("layer_score_finalize", stream, [&] {
      score_finalize_kernel<<<rows, 32, 0, stream>>>(partial, entries, d_sums, d_maxs);
    });
    launches += 2;
  }
  count_launches(launches);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(WINO_E_CUDA, "layer launch: %s", cudaGetErrorString(e));
  if (act != nullptr && !(pool == 1 || m % 2 == 0)) return relu_pool_launch(y, act, N, K, g.Ho, g.Wo, pool, stream);
  return WINO_OK;
}

}  // namespace wino
