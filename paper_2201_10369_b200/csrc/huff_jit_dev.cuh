// NEXT row N2, Huffman order, register-resident form: the skeleton of the run-time
// specialised Huffman-order sweep kernels.  PAPER.md P:465 ("Huffman tree evaluation
// order"); reading R21.
//
// The Huffman tree of a transform row depends on the candidate's coefficient MAGNITUDES
// only through their order, so across a c-sweep the candidates fall into a handful of
// classes with identical per-row programs (8 classes for the 4096 configs[1] F(4,3)
// candidates).  huff_jit.cpp emits, per class, an `eval` functor whose every dot product
// is its Huffman tree written out as straight-line code -- leaves RN(x_j * c_j), internal
// nodes RN(v_a + v_b), coefficients read from the kernel parameters (uniform registers),
// all operands in registers -- and compiles it with NVRTC against this header (embedded in
// libwino.so).  The interpreter kernel (sweep_huff.cuh) keeps every node in a shared-memory
// slot (3 shared-memory operations per addition); here the additions are plain FADDs.
//
// Scalar __fmul_rn / __fadd_rn, one tile per thread: their rounding modifiers forbid
// contraction (ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2, sweep_kernels.cuh),
// and one tile per thread halves the registers of the pair layout at the same FP32-pipe
// throughput.  Scoring: exact fp64 statistics per output (Stat::add_careful, padding tiles
// excluded), the interpreter's semantics.  Compiled by NVRTC only (no host includes).
#pragma once
#include "sweep_dev.cuh"

namespace wino {

// E::eval(cm, sd, d, g, tid, y): cm = the candidate's fp32 matrices [AT | G | BT] (kernel
// parameters), sd = this CTA's staged 2D tiles [n*n][kSwThreads] (2D), d = the 1D tile in
// registers (1D), g = the filter, y = the m^dims outputs.
template <int DIMS, int M, int R, class E>
__device__ __forceinline__ void huff_jit_run(const SweepArgs& a, const MatsParam& P, const IdxParam& DI) {
  constexpr int N = M + R - 1;
  constexpr int DN = DIMS == 1 ? N : N * N, DG = DIMS == 1 ? R : R * R, DY = DIMS == 1 ? M : M * M;
  constexpr int PER = M * N + N * R + N * N;
  extern __shared__ __align__(16) unsigned char smem[];
  float* sd = reinterpret_cast<float*>(smem);   // [DN][kSwThreads] (2D)
  double* sacc = reinterpret_cast<double*>(smem + (DIMS == 2 ? DN * kSwThreads * 4 : 0));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_launch_dependents();

  const int n_items = a.n_cgroups * a.n_tgroups;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int cg = item / a.n_tgroups, tg = item - cg * a.n_tgroups;
    const int c_begin = cg * a.cands_per_cta;
    const int c_end = min(a.n_cand, c_begin + a.cands_per_cta);
    __syncthreads();   // the previous item's accumulators have been read
    for (int k = tid; k < kMaxCpc * 4 * kPartial; k += kSwThreads) sacc[k] = 0.0;
    __syncthreads();   // zeroed before lane 0 of any warp accumulates
    const int tb_begin = tg * a.tblk_per_cta;
    const int tb_end = min(a.n_tblk, tb_begin + a.tblk_per_cta);
    for (int tb = tb_begin; tb < tb_end; tb++) {
      const long long t = (long long)tb * kSwThreads + tid;
      const bool ok = t < a.n_tiles;
      // the thread's own tile; 2D: staged to its own shared-memory column (read back one
      // tile column at a time by eval), no barrier needed
      float d[DIMS == 1 ? DN : 1];
      if constexpr (DIMS == 1) {
#pragma unroll
        for (int e = 0; e < DN; e++) d[e] = ok ? __ldg(a.d + t * DN + e) : 0.0f;
      } else if constexpr (DN % 4 == 0) {
        d[0] = 0.0f;
#pragma unroll 4
        for (int e4 = 0; e4 < DN / 4; e4++) {
          const float4 v = ok ? __ldg(reinterpret_cast<const float4*>(a.d + t * DN) + e4) : make_float4(0.f, 0.f, 0.f, 0.f);
          sd[(4 * e4 + 0) * kSwThreads + tid] = v.x;
          sd[(4 * e4 + 1) * kSwThreads + tid] = v.y;
          sd[(4 * e4 + 2) * kSwThreads + tid] = v.z;
          sd[(4 * e4 + 3) * kSwThreads + tid] = v.w;
        }
      } else {
        d[0] = 0.0f;
#pragma unroll 4
        for (int e = 0; e < DN; e++) sd[e * kSwThreads + tid] = ok ? __ldg(a.d + t * DN + e) : 0.0f;
      }
      float g[DG];
#pragma unroll
      for (int e = 0; e < DG; e++) g[e] = ok ? __ldg(a.g + t * DG + e) : 0.0f;
      // fp64 references, tile-block-major [t / 128][DY][128]: coalesced, L1/L2-resident
      const double* yt = a.y64t + (long long)tb * DY * kSwThreads + tid;

      for (int s = c_begin; s < c_end; s++) {
        const float* cm = P.v + s * PER;
        float y[DY];
        E::eval(cm, sd, d, g, tid, y);
        if (a.ydump != nullptr && ok) {
          float* yd = a.ydump + ((long long)DI.idx[s] * a.n_tiles + t) * DY;
#pragma unroll
          for (int o = 0; o < DY; o++) yd[o] = y[o];
        }
        // fast path: unconditional fp64 scoring (a padding tile has y = y64 = 0: no effect);
        // if any sum of the warp went non-finite, the same outputs are re-scored exactly with
        // per-output finiteness and padding tiles excluded (Stat::add_careful)
        Stat st;
#pragma unroll
        for (int o = 0; o < DY; o++) {
          if (o & 1) st.add_fast<1>(y[o], __ldg(yt + o * kSwThreads));
          else st.add_fast<0>(y[o], __ldg(yt + o * kSwThreads));
        }
        if (__any_sync(0xffffffffu, !st.finite())) {
          st = Stat();
          if (ok) {
#pragma unroll
            for (int o = 0; o < DY; o++) {
              if (o & 1) st.add_careful<1>(y[o], __ldg(yt + o * kSwThreads));
              else st.add_careful<0>(y[o], __ldg(yt + o * kSwThreads));
            }
          }
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
  }
  pdl_wait();
}

}  // namespace wino
