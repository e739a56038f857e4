// NEXT row N2: the mixed-precision error sweep (WINO_SWEEP_MIXED).
// ("double precision floating point for the transforms and single precision for Hadamard
// product"); reading R22: the three transforms in fp64 with the fp64 (R64)
// matrices, each dot product an ascending DFMA chain from +0, 2D left product first;
// U and V rounded to fp32; M = RN32(u * v); the output transform in fp64 on M, rounded to
// fp32.  One tile per thread (the FP64 pipe has no paired form); the candidates' fp64
// matrices ride in the kernel parameter space (as pairs of floats); y64 is staged in shared
// memory per tile block; fp64 scoring (Stat).  Bit-identical to the oracle's
// oref_sweep_mixed (tests/test_gpu_mixed.py).
#pragma once
#include "sweep_kernels.cuh"

namespace wino {

// smem: y64 [DY][kSwThreads] double, sacc
template <int DIMS, int M, int R>
__global__ void __launch_bounds__(kSwThreads) sweep_mixed_kernel(SweepArgs a, const __grid_constant__ MatsParam P,
                                                                 const __grid_constant__ IdxParam DI) {
  constexpr int N = M + R - 1;
  constexpr int DN = DIMS == 1 ? N : N * N, DG = DIMS == 1 ? R : R * R, DY = DIMS == 1 ? M : M * M;
  constexpr int PER = M * N + N * R + N * N;   // doubles per candidate
  extern __shared__ __align__(16) unsigned char smem[];
  double* sy = reinterpret_cast<double*>(smem);   // [DY][kSwThreads]
  double* sacc = sy + DY * kSwThreads;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* PV = reinterpret_cast<const double*>(P.v);

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
      const long long t = (long long)tb * kSwThreads + tid;
      const bool ok = t < a.n_tiles;
      double d[DN], g[DG];
#pragma unroll
      for (int e = 0; e < DN; e++) d[e] = ok ? (double)__ldg(a.d + t * DN + e) : 0.0;
#pragma unroll
      for (int e = 0; e < DG; e++) g[e] = ok ? (double)__ldg(a.g + t * DG + e) : 0.0;
#pragma unroll
      for (int o = 0; o < DY; o++) sy[o * kSwThreads + tid] = ok ? __ldg(a.y64 + t * DY + o) : 0.0;

      for (int s = c_begin; s < c_end; s++) {
        const double* AT = PV + s * PER;
        const double* G = AT + M * N;
        const double* BT = G + N * R;
        float y[DY];
        if constexpr (DIMS == 1) {
          double mw[N];
#pragma unroll
          for (int i = 0; i < N; i++) {
            double u = 0.0, v = 0.0;
#pragma unroll
            for (int j = 0; j < R; j++) u = __fma_rn(G[i * R + j], g[j], u);
#pragma unroll
            for (int j = 0; j < N; j++) v = __fma_rn(BT[i * N + j], d[j], v);
            mw[i] = (double)__fmul_rn(__double2float_rn(u), __double2float_rn(v));
          }
#pragma unroll
          for (int p = 0; p < M; p++) {
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < N; i++) acc = __fma_rn(AT[p * N + i], mw[i], acc);
            y[p] = __double2float_rn(acc);
          }
        } else {
          // U = RN32(G g Gᵀ), kept in fp32
          float U[N][N];
#pragma unroll
          for (int i = 0; i < N; i++) {
            double t1[R];
#pragma unroll
            for (int q = 0; q < R; q++) {
              double acc = 0.0;
#pragma unroll
              for (int j = 0; j < R; j++) acc = __fma_rn(G[i * R + j], g[j * R + q], acc);
              t1[q] = acc;
            }
#pragma unroll
            for (int l = 0; l < N; l++) {
              double acc = 0.0;
#pragma unroll
              for (int q = 0; q < R; q++) acc = __fma_rn(G[l * R + q], t1[q], acc);
              U[i][l] = __double2float_rn(acc);
            }
          }
          // rows of V; M = RN32(U V); T3[p][l] = Σ_i Aᵀ[p][i] M[i][l] (ascending i)
          double t3[M][N];
#pragma unroll
          for (int p = 0; p < M; p++)
#pragma unroll
            for (int l = 0; l < N; l++) t3[p][l] = 0.0;
#pragma unroll
          for (int i = 0; i < N; i++) {
            double t2[N];
#pragma unroll
            for (int q = 0; q < N; q++) {
              double acc = 0.0;
#pragma unroll
              for (int j = 0; j < N; j++) acc = __fma_rn(BT[i * N + j], d[j * N + q], acc);
              t2[q] = acc;
            }
#pragma unroll
            for (int l = 0; l < N; l++) {
              double acc = 0.0;
#pragma unroll
              for (int q = 0; q < N; q++) acc = __fma_rn(BT[l * N + q], t2[q], acc);
              const double mw = (double)__fmul_rn(U[i][l], __double2float_rn(acc));
#pragma unroll
              for (int p = 0; p < M; p++) t3[p][l] = __fma_rn(AT[p * N + i], mw, t3[p][l]);
            }
          }
#pragma unroll
          for (int p = 0; p < M; p++)
#pragma unroll
            for (int q = 0; q < M; q++) {
              double acc = 0.0;
#pragma unroll
              for (int l = 0; l < N; l++) acc = __fma_rn(AT[q * N + l], t3[p][l], acc);
              y[p * M + q] = __double2float_rn(acc);
            }
        }
        if (a.ydump != nullptr && ok) {
          float* yd = a.ydump + ((long long)DI.idx[s] * a.n_tiles + t) * DY;
#pragma unroll
          for (int o = 0; o < DY; o++) yd[o] = y[o];
        }
        {
          Stat st;
          if (ok)
#pragma unroll
            for (int o = 0; o < DY; o++) st.add_careful<0>(y[o], sy[o * kSwThreads + tid]);
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
HuffCfg make_mixed_cfg() {
  HuffCfg h;
  h.dims = DIMS;
  h.m = M;
  h.r = R;
  h.k = (SweepKernel)sweep_mixed_kernel<DIMS, M, R>;
  return h;
}

}  // namespace wino
