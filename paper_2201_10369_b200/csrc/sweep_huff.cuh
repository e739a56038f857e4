// NEXT row N2: the error sweep with Huffman-ordered transforms (WINO_SWEEP_HUFFMAN).
// PAPER.md P:465 ("Huffman tree evaluation order ... We also use the same evaluation order
// and present results based on it"); reading R21: every dot product of a
// transform row with data is the sum of the products RN(coef_j * x_j) of the non-zero
// coefficients along a Huffman tree over |coef_j| (ties: leaves in index order, then older
// nodes); the Hadamard product is RN(u * v).
//
// The tree depends on the candidate's coefficients, so it cannot be unrolled at compile
// time.  The host builds, per candidate and matrix row, a small program (huffman_program in
// sweep.cu): `nops` additions (a, b) over slots 0..len-1 (the products, by coefficient
// index) and len.. (the internal nodes in creation order), plus the result slot (255: no
// term, +0).  The programs ride in the kernel parameter space after the candidate's
// matrices; the kernel forms the products with FMUL2 (two tiles per thread), keeps them in
// a per-thread column of shared memory ([slot][thread], conflict-free) and executes the
// additions with FADD2 in program order.  Scoring as in the fp64 paths (Stat, careful).
// Kernel and host agree on the record layout below; outputs are bit-identical to the
// oracle's Huffman mode (tests/test_gpu_huffman.py).
#pragma once
#include "sweep_kernels.cuh"

namespace wino {

// per-row program record: [nops][result][a0 b0][a1 b1]...  (2 + 2 * (len - 1) bytes)
__host__ __device__ constexpr int huff_rec_bytes(int len) { return 2 + 2 * (len - 1); }
// per-candidate program bytes: n rows of G (len r), n rows of Bᵀ (len n), m rows of Aᵀ (len n)
__host__ __device__ constexpr int huff_prog_bytes(int m, int r) {
  return (m + r - 1) * huff_rec_bytes(r) + (m + r - 1) * huff_rec_bytes(m + r - 1) + m * huff_rec_bytes(m + r - 1);
}
__host__ __device__ constexpr int huff_prog_words(int m, int r) { return (huff_prog_bytes(m, r) + 3) / 4; }
constexpr unsigned char kHuffNone = 255;
// dots evaluated together per row program in 2D (shared memory bounds it for n > 8)
__host__ __device__ constexpr int huff_group(int n) { return n <= 8 ? n : 3; }
// per-thread slot columns: one dot at a time in 1D, huff_group(n) dots sharing a program in 2D
__host__ __device__ constexpr int huff_slot_columns(int dims, int n) {
  return dims == 1 ? 2 * n - 1 : huff_group(n) * (2 * n - 1);
}

__device__ __forceinline__ u64 hmul2(u64 a, float c) {
  u64 d, cc;
  asm("mov.b64 %0, {%1,%1};" : "=l"(cc) : "f"(c));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(cc));
  return d;
}
__device__ __forceinline__ u64 hmulv2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 hadd2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// Σ_j coef[j * cs] * x[j] in the row's Huffman order.  `slot` = this thread's column
// (stride kSwThreads u64); `rec` = the row's program record (parameter space).
template <int LEN>
__device__ __forceinline__ u64 huff_dot(const float* coef, int cs, const u64 (&x)[LEN], const unsigned char* rec,
                                        u64* slot) {
#pragma unroll
  for (int j = 0; j < LEN; j++) slot[j * kSwThreads] = hmul2(x[j], coef[j * cs]);
  const int nops = rec[0];
#pragma unroll
  for (int k = 0; k < LEN - 1; k++) {
    if (k < nops) {
      const int a = rec[2 + 2 * k], b = rec[3 + 2 * k];
      slot[(LEN + k) * kSwThreads] = hadd2(slot[a * kSwThreads], slot[b * kSwThreads]);
    }
  }
  const int res = rec[1];
  return res == kHuffNone ? 0ull : slot[res * kSwThreads];
}

// ND dot products sharing one row program: Σ_j coef[j] * x[d][j] for d < ND, in groups of
// G dots.  Each dot of a group has its own slot column (slot + d * (2 LEN - 1) * kSwThreads),
// so the G addition chains are independent (ILP) and the program decode is shared.
template <int LEN, int ND, int G>
__device__ __forceinline__ void huff_dot_multi(const float* coef, const u64 (&x)[ND][LEN], const unsigned char* rec,
                                               u64* slot, u64 (&out)[ND]) {
  constexpr int S = (2 * LEN - 1) * kSwThreads;   // slot column stride per dot
  const int nops = rec[0], res = rec[1];
#pragma unroll
  for (int d0 = 0; d0 < ND; d0 += G) {
#pragma unroll
    for (int j = 0; j < LEN; j++) {
      const float c = coef[j];
#pragma unroll
      for (int dd = 0; dd < G; dd++)
        if (d0 + dd < ND) slot[dd * S + j * kSwThreads] = hmul2(x[d0 + dd][j], c);
    }
#pragma unroll
    for (int k = 0; k < LEN - 1; k++) {
      if (k < nops) {
        const int a = rec[2 + 2 * k] * kSwThreads, b = rec[3 + 2 * k] * kSwThreads;
#pragma unroll
        for (int dd = 0; dd < G; dd++)
          if (d0 + dd < ND) slot[dd * S + (LEN + k) * kSwThreads] = hadd2(slot[dd * S + a], slot[dd * S + b]);
      }
    }
#pragma unroll
    for (int dd = 0; dd < G; dd++)
      if (d0 + dd < ND) out[d0 + dd] = res == kHuffNone ? 0ull : slot[dd * S + res * kSwThreads];
  }
}

// Out-of-line wrapper for n > 8: the fully inlined 2D kernels for F(7,3) / F(8,3) take
// minutes to compile; calls keep the code size linear (the variant is not the hot path).
template <int LEN, int ND, int G>
__device__ __noinline__ void huff_dot_multi_ool(const float* coef, const u64 (&x)[ND][LEN], const unsigned char* rec,
                                                u64* slot, u64 (&out)[ND]) {
  huff_dot_multi<LEN, ND, G>(coef, x, rec, slot, out);
}

template <int LEN, int ND, int G, bool OOL>
__device__ __forceinline__ void huff_dot_rows(const float* coef, const u64 (&x)[ND][LEN], const unsigned char* rec,
                                              u64* slot, u64 (&out)[ND]) {
  if constexpr (OOL) huff_dot_multi_ool<LEN, ND, G>(coef, x, rec, slot, out);
  else huff_dot_multi<LEN, ND, G>(coef, x, rec, slot, out);
}

// smem: slots [huff_slot_columns][kSwThreads] u64, y64 [MM][2][kSwThreads] double, sacc
template <int DIMS, int M, int R>
__global__ void __launch_bounds__(kSwThreads) sweep_huff_kernel(SweepArgs a, const __grid_constant__ MatsParam P,
                                                                const __grid_constant__ IdxParam DI) {
  constexpr int N = M + R - 1;
  constexpr int DN = DIMS == 1 ? N : N * N, DG = DIMS == 1 ? R : R * R, DY = DIMS == 1 ? M : M * M;
  constexpr int PER = M * N + N * R + N * N;
  constexpr int STRIDE = PER + huff_prog_words(M, R);
  constexpr int TPB = kSwThreads * 2;
  constexpr int RG = huff_rec_bytes(R), RB = huff_rec_bytes(N);
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int SLOTS = huff_slot_columns(DIMS, N);
  constexpr int HG = huff_group(N);
  u64* slots = reinterpret_cast<u64*>(smem);                        // [SLOTS][kSwThreads]
  double* sy = reinterpret_cast<double*>(slots + SLOTS * kSwThreads);   // [DY][2][kSwThreads]
  double* sacc = sy + DY * 2 * kSwThreads;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  u64* slot = slots + tid;

  pdl_launch_dependents();
  const int n_items = a.n_cgroups * a.n_tgroups;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int cg = item / a.n_tgroups, tg = item - cg * a.n_tgroups;
    const int c_begin = cg * a.cands_per_cta;
    const int c_end = min(a.n_cand, c_begin + a.cands_per_cta);
    __syncthreads();
    for (int k = tid; k < kMaxCpc * 4 * kPartial; k += kSwThreads) sacc[k] = 0.0;
    __syncthreads();   // zeroed before lane 0 of any warp accumulates
    const int tb_begin = tg * a.tblk_per_cta;
    const int tb_end = min(a.n_tblk, tb_begin + a.tblk_per_cta);
    for (int tb = tb_begin; tb < tb_end; tb++) {
      const long long tile0 = (long long)tb * TPB;
      bool ok[2];
#pragma unroll
      for (int h = 0; h < 2; h++) ok[h] = tile0 + tid + h * kSwThreads < a.n_tiles;
      u64 d[DN], g[DG];
#pragma unroll
      for (int e = 0; e < DN; e++) {
        float v[2];
#pragma unroll
        for (int h = 0; h < 2; h++) v[h] = ok[h] ? __ldg(a.d + (tile0 + tid + h * kSwThreads) * DN + e) : 0.0f;
        d[e] = Lane<true, true>::pack(v[0], v[1]);
      }
#pragma unroll
      for (int e = 0; e < DG; e++) {
        float v[2];
#pragma unroll
        for (int h = 0; h < 2; h++) v[h] = ok[h] ? __ldg(a.g + (tile0 + tid + h * kSwThreads) * DG + e) : 0.0f;
        g[e] = Lane<true, true>::pack(v[0], v[1]);
      }
#pragma unroll
      for (int o = 0; o < DY; o++)
#pragma unroll
          for (int h = 0; h < 2; h++)
            sy[(o * 2 + h) * kSwThreads + tid] = ok[h] ? __ldg(a.y64 + (tile0 + tid + h * kSwThreads) * DY + o) : 0.0;

      for (int s = c_begin; s < c_end; s++) {
        const float* cm = P.v + s * STRIDE;
        const float* AT = cm;
        const float* G = cm + M * N;
        const float* BT = cm + M * N + N * R;
        const unsigned char* pg = reinterpret_cast<const unsigned char*>(cm + PER);   // G rows
        const unsigned char* pb = pg + N * RG;                                        // Bᵀ rows
        const unsigned char* pa = pb + N * RB;                                        // Aᵀ rows
        u64 y[DY];
        if constexpr (DIMS == 1) {
          u64 mw[N];
#pragma unroll
          for (int i = 0; i < N; i++) {
            const u64 u = huff_dot<R>(G + i * R, 1, g, pg + i * RG, slot);
            const u64 v = huff_dot<N>(BT + i * N, 1, d, pb + i * RB, slot);
            mw[i] = hmulv2(u, v);
          }
#pragma unroll
          for (int p = 0; p < M; p++) y[p] = huff_dot<N>(AT + p * N, 1, mw, pa + p * RB, slot);
        } else {
          // Every pass evaluates the dots that share a row program together (huff_dot_multi).
          // U = G g Gᵀ: T1[i][q] = dot(G row i, g[.][q]); U[i][l] = dot(G row l, T1[i][.])
          u64 T1[N][R];
#pragma unroll
          for (int i = 0; i < N; i++) {
            u64 cols[R][R];
#pragma unroll
            for (int q = 0; q < R; q++)
#pragma unroll
              for (int j = 0; j < R; j++) cols[q][j] = g[j * R + q];
            huff_dot_rows<R, R, (R < HG ? R : HG), (N > 8)>(G + i * R, cols, pg + i * RG, slot, T1[i]);
          }
          u64 U[N][N];
#pragma unroll
          for (int l = 0; l < N; l++) {
            u64 o[N];
            huff_dot_rows<R, N, HG, (N > 8)>(G + l * R, T1, pg + l * RG, slot, o);
#pragma unroll
            for (int i = 0; i < N; i++) U[i][l] = o[i];
          }
          // T2[i][q] = dot(Bᵀ row i, d[.][q]); V[i][l] = dot(Bᵀ row l, T2[i][.]); Mw = U ⊙ V
          u64 T2[N][N];
#pragma unroll
          for (int i = 0; i < N; i++) {
            u64 cols[N][N];
#pragma unroll
            for (int q = 0; q < N; q++)
#pragma unroll
              for (int j = 0; j < N; j++) cols[q][j] = d[j * N + q];
            huff_dot_rows<N, N, HG, (N > 8)>(BT + i * N, cols, pb + i * RB, slot, T2[i]);
          }
#pragma unroll
          for (int l = 0; l < N; l++) {
            u64 o[N];
            huff_dot_rows<N, N, HG, (N > 8)>(BT + l * N, T2, pb + l * RB, slot, o);
#pragma unroll
            for (int i = 0; i < N; i++) U[i][l] = hmulv2(U[i][l], o[i]);
          }
          // T3[p][l] = dot(Aᵀ row p, Mw[.][l]); Y[p][q] = dot(Aᵀ row q, T3[p][.])
          u64 T3[M][N];
#pragma unroll
          for (int p = 0; p < M; p++) {
            u64 cols[N][N];
#pragma unroll
            for (int l = 0; l < N; l++)
#pragma unroll
              for (int i = 0; i < N; i++) cols[l][i] = U[i][l];
            huff_dot_rows<N, N, HG, (N > 8)>(AT + p * N, cols, pa + p * RB, slot, T3[p]);
          }
#pragma unroll
          for (int q = 0; q < M; q++) {
            u64 o[M];
            huff_dot_rows<N, M, (M < HG ? M : HG), (N > 8)>(AT + q * N, T3, pa + q * RB, slot, o);
#pragma unroll
            for (int p = 0; p < M; p++) y[p * M + q] = o[p];
          }
        }
        if (a.ydump != nullptr) {
          float* yd = a.ydump + ((long long)DI.idx[s] * a.n_tiles + tile0) * DY;
#pragma unroll
          for (int h = 0; h < 2; h++)
            if (ok[h])
#pragma unroll
              for (int o = 0; o < DY; o++) yd[(tid + h * kSwThreads) * DY + o] = Lane<true, true>::get(y[o], h);
        }
        {
          Stat st;
#pragma unroll
          for (int o = 0; o < DY; o++) {
            if (ok[0]) st.add_careful<0>(Lane<true, true>::get(y[o], 0), sy[(o * 2) * kSwThreads + tid]);
            if (ok[1]) st.add_careful<1>(Lane<true, true>::get(y[o], 1), sy[(o * 2 + 1) * kSwThreads + tid]);
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
    {
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
  pdl_wait();
}

template <int DIMS, int M, int R>
HuffCfg make_huff_cfg() {
  HuffCfg h;
  h.dims = DIMS;
  h.m = M;
  h.r = R;
  h.k = (SweepKernel)sweep_huff_kernel<DIMS, M, R>;
  return h;
}

}  // namespace wino
