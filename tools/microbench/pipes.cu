// Pipe-throughput microbenchmark for the sweep/layer design decisions.
// Measures, per SM and per clock, the warp-instruction throughput of:
//   FFMA (3 vector-register operands), FFMA with a uniform-register operand,
//   FFMA2 (fma.rn.f32x2) with register / uniform-broadcast operands, DFMA, DADD,
//   and FFMA2 interleaved with DADD (do the FP32 and FP64 pipes overlap?).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu -lnvidia-ml
// Output: one JSON line per test: lane-ops per SM per cycle, and ops/s at the measured clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 p; asm("mov.b64 %0, {%1,%2};" : "=l"(p) : "f"(a), "f"(b)); return p; }
__device__ __forceinline__ void ffma2(u64& d, u64 a, u64 b) { asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b)); }
__device__ __forceinline__ float lo(u64 p) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(p)); return a + b; }

struct Coef { float c[64]; };

// Each kernel: 8 independent chains per thread, ITER iterations of an unrolled body.
// cycles[blockIdx] = clock64 span of thread 0 of the block.
#define ITER 4096

__global__ void k_ffma_reg(float* out, long long* cyc, float a, float b) {
  float x[8]; for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  float av = a + threadIdx.x * 1e-30f, bv = b + threadIdx.x * 1e-30f;  // vector registers
  long long t0 = clock64();
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __fmaf_rn(x[i], av, bv);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma_ur(float* out, long long* cyc, const __grid_constant__ Coef cf) {
  float x[8]; for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < ITER; it++) {
    int base = (it & 3) * 16;
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __fmaf_rn(x[i], cf.c[base + i], x[i]);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2_reg(float* out, long long* cyc, float a, float b) {
  u64 x[8]; for (int i = 0; i < 8; i++) x[i] = pk(threadIdx.x + i, i);
  u64 av = pk(a + threadIdx.x * 1e-30f, a), bv = pk(b, b + threadIdx.x * 1e-30f);
  long long t0 = clock64();
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) ffma2(x[i], x[i], av);
    av ^= 1ull; bv ^= 1ull;
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += lo(x[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + lo(bv);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2_ur(float* out, long long* cyc, const __grid_constant__ Coef cf) {
  u64 x[8]; for (int i = 0; i < 8; i++) x[i] = pk(threadIdx.x + i, i);
  long long t0 = clock64();
  for (int it = 0; it < ITER; it++) {
    int base = (it & 3) * 16;
#pragma unroll
    for (int i = 0; i < 8; i++) { float c = cf.c[base + i]; ffma2(x[i], x[i], pk(c, c)); }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += lo(x[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dfma(float* out, long long* cyc, double a, double b) {
  double x[8]; for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  double av = a + threadIdx.x * 1e-300, bv = b;
  long long t0 = clock64();
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __fma_rn(x[i], av, bv);
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; i++) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dadd(float* out, long long* cyc, double a, double b) {
  double x[8]; for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  double av = a + threadIdx.x * 1e-300;
  long long t0 = clock64();
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __dadd_rn(x[i], av);
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; i++) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s + (float)b;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// 8 FFMA2 (UR operand) + 4 DADD per body: do the FP64 ops hide under the FP32 pipe?
__global__ void k_mix(float* out, long long* cyc, const __grid_constant__ Coef cf) {
  u64 x[8]; for (int i = 0; i < 8; i++) x[i] = pk(threadIdx.x + i, i);
  double y[4]; for (int i = 0; i < 4; i++) y[i] = threadIdx.x * 0.5 + i;
  double dv = 1e-7 + threadIdx.x * 1e-300;
  long long t0 = clock64();
  for (int it = 0; it < ITER; it++) {
    int base = (it & 3) * 16;
#pragma unroll
    for (int i = 0; i < 8; i++) { float c = cf.c[base + i]; ffma2(x[i], x[i], pk(c, c)); }
#pragma unroll
    for (int i = 0; i < 4; i++) y[i] = __dadd_rn(y[i], dv);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += lo(x[i]);
  for (int i = 0; i < 4; i++) s += (float)y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// The layer GEMM's inner-loop operand pattern, registers only: 32 accumulator pairs,
// acc[i][j] = fma2(b[j], bcast(a[i]), acc[i][j]) with 8 scalar a (regular registers) and 4
// vector b -- FFMA2 R, R.F32x2, R.F32, R.F32x2 with three distinct vector registers per
// instruction (k_ffma2_reg repeats one).  Its rate is the FMA-pipe ceiling of that kernel.
__global__ void __launch_bounds__(256, 2) k_ffma2_gemm(float* out, long long* cyc, float a0, float b0) {
  u64 acc[8][4];
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) acc[i][j] = pk(threadIdx.x + i, j);
  float a[8]; u64 b[4];
  for (int i = 0; i < 8; i++) a[i] = a0 + (threadIdx.x + i) * 1e-30f;
  for (int j = 0; j < 4; j++) b[j] = pk(b0 + threadIdx.x * 1e-30f, b0 + j * 1e-30f);
  long long t0 = clock64();
  for (int it = 0; it < ITER * 2; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        u64 cc = pk(a[i], a[i]), d;   // the layer's ffma2_bcast: ptxas is free to rotate the accumulators
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(b[j]), "l"(cc), "l"(acc[i][j]));
        acc[i][j] = d;
      }
#pragma unroll
    for (int j = 0; j < 4; j++) b[j] ^= 1ull;
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) s += lo(acc[i][j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// The GEMM pattern ordered b-major: one vector operand b[j] held for 8 consecutive FFMA2
// (operand-reuse cache), the scalar a[i] and the accumulator change every instruction.
template <bool PIN>
__global__ void __launch_bounds__(256, 2) k_ffma2_gemm_bmajor(float* out, long long* cyc, float a0, float b0) {
  u64 acc[8][4];
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) acc[i][j] = pk(threadIdx.x + i, j);
  float a[8]; u64 b[4];
  for (int i = 0; i < 8; i++) a[i] = a0 + (threadIdx.x + i) * 1e-30f;
  for (int j = 0; j < 4; j++) b[j] = pk(b0 + threadIdx.x * 1e-30f, b0 + j * 1e-30f);
  long long t0 = clock64();
  for (int it = 0; it < ITER * 2; it++) {
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int i = 0; i < 8; i++) {
        u64 cc = pk(a[i], a[i]);
        if (PIN) {
          asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][j]) : "l"(b[j]), "l"(cc));
        } else {
          u64 d;
          asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(b[j]), "l"(cc), "l"(acc[i][j]));
          acc[i][j] = d;
        }
      }
#pragma unroll
    for (int j = 0; j < 4; j++) b[j] ^= 1ull;
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) s += lo(acc[i][j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// The GEMM outer product with scalar FFMA: acc[i][j] = fma(a[i], b[j], acc[i][j]), 8 x 8.
__global__ void __launch_bounds__(256, 2) k_ffma_gemm(float* out, long long* cyc, float a0, float b0) {
  float acc[8][8];
  for (int i = 0; i < 8; i++) for (int j = 0; j < 8; j++) acc[i][j] = threadIdx.x + i + 8 * j;
  float a[8], b[8];
  for (int i = 0; i < 8; i++) a[i] = a0 + (threadIdx.x + i) * 1e-30f;
  for (int j = 0; j < 8; j++) b[j] = b0 + (threadIdx.x + 3 * j) * 1e-30f;
  long long t0 = clock64();
  for (int it = 0; it < ITER * 2; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 8; j++) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
#pragma unroll
    for (int j = 0; j < 8; j++) b[j] = __int_as_float(__float_as_int(b[j]) ^ 1);
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; i++) for (int j = 0; j < 8; j++) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// The same outer product with the scalar operand pre-duplicated into a 64-bit pair (a, a):
// FFMA2 R, R.F32x2, R.F32x2, R.F32x2 (no .F32 broadcast operand).
__global__ void __launch_bounds__(256, 2) k_ffma2_gemm_pairs(float* out, long long* cyc, float a0, float b0) {
  u64 acc[8][4];
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) acc[i][j] = pk(threadIdx.x + i, j);
  u64 a[8], b[4];
  for (int i = 0; i < 8; i++) a[i] = pk(a0 + (threadIdx.x + i) * 1e-30f, a0 + (threadIdx.x + 2 * i) * 1e-30f);
  for (int j = 0; j < 4; j++) b[j] = pk(b0 + threadIdx.x * 1e-30f, b0 + j * 1e-30f);
  long long t0 = clock64();
  for (int it = 0; it < ITER * 2; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        u64 d;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(b[j]), "l"(a[i]), "l"(acc[i][j]));
        acc[i][j] = d;
      }
#pragma unroll
    for (int j = 0; j < 4; j++) b[j] ^= 1ull;
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) s += lo(acc[i][j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0, nsm = 0, clk_khz = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  const int threads = 256, per_sm = 4, blocks = nsm * per_sm;
  float* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(float) * blocks * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * blocks));
  Coef cf; for (int i = 0; i < 64; i++) cf.c[i] = 1.0f - 1e-7f * i;
  long long hc[4096];
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct T { const char* name; double lane_ops_per_instr; double instr_per_iter; int flops_per_op; };
  // lane-ops per thread per iteration, per test
  for (int test = 0; test < 12; test++) {
    const char* name = nullptr; double ops_per_thread_iter = 0; int flops_per_op = 2;
    int nblk = blocks, psm = per_sm;
    for (int rep = 0; rep < 3; rep++) {
      CK(cudaEventRecord(e0));
      switch (test) {
        case 0: k_ffma_reg<<<blocks, threads>>>(out, cyc, 1.0000001f, 1e-9f); name = "ffma_reg"; ops_per_thread_iter = 8; break;
        case 1: k_ffma_ur<<<blocks, threads>>>(out, cyc, cf); name = "ffma_ur"; ops_per_thread_iter = 8; break;
        case 2: k_ffma2_reg<<<blocks, threads>>>(out, cyc, 1.0000001f, 1e-9f); name = "ffma2_reg"; ops_per_thread_iter = 16; break;
        case 3: k_ffma2_ur<<<blocks, threads>>>(out, cyc, cf); name = "ffma2_ur"; ops_per_thread_iter = 16; break;
        case 4: k_dfma<<<blocks, threads>>>(out, cyc, 1.0000001, 1e-9); name = "dfma"; ops_per_thread_iter = 8; break;
        case 5: k_dadd<<<blocks, threads>>>(out, cyc, 1e-9, 0.0); name = "dadd"; ops_per_thread_iter = 8; flops_per_op = 1; break;
        case 6: k_mix<<<blocks, threads>>>(out, cyc, cf); name = "ffma2_ur+dadd(2:1 fp32:fp64 instr)"; ops_per_thread_iter = 16; break;
        // 2 CTAs of 256 threads per SM like the GEMM; 32 FFMA2 = 64 lane-ops per body, 2 ITER bodies
        case 8: nblk = nsm * 2; psm = 2; k_ffma2_gemm_pairs<<<nblk, threads>>>(out, cyc, 1.0000001f, 1e-9f); name = "ffma2_gemm_pattern_pairs(scalar pre-duplicated)"; ops_per_thread_iter = 128; break;
        case 9: nblk = nsm * 2; psm = 2; k_ffma2_gemm_bmajor<false><<<nblk, threads>>>(out, cyc, 1.0000001f, 1e-9f); name = "ffma2_gemm_pattern_bmajor"; ops_per_thread_iter = 128; break;
        case 10: nblk = nsm * 2; psm = 2; k_ffma2_gemm_bmajor<true><<<nblk, threads>>>(out, cyc, 1.0000001f, 1e-9f); name = "ffma2_gemm_pattern_bmajor_pinned_order"; ops_per_thread_iter = 128; break;
        case 11: nblk = nsm * 2; psm = 2; k_ffma_gemm<<<nblk, threads>>>(out, cyc, 1.0000001f, 1e-9f); name = "ffma_gemm_pattern(scalar FFMA 8x8)"; ops_per_thread_iter = 128; break;
        case 7: nblk = nsm * 2; psm = 2; k_ffma2_gemm<<<nblk, threads>>>(out, cyc, 1.0000001f, 1e-9f); name = "ffma2_gemm_pattern(3 vector regs, 16 warps/SM)"; ops_per_thread_iter = 128; break;
      }
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
    }
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(hc, cyc, sizeof(long long) * nblk, cudaMemcpyDeviceToHost));
    double cmax = 0, csum = 0; for (int b = 0; b < nblk; b++) { csum += hc[b]; if (hc[b] > cmax) cmax = hc[b]; }
    double lane_ops = (double)nblk * threads * ITER * ops_per_thread_iter;
    // per SM per cycle, using the mean per-block cycle span (blocks on one SM run concurrently: per_sm * threads)
    double per_sm_cycle = (double)psm * threads * ITER * ops_per_thread_iter / (csum / nblk);
    double eff_clock_mhz = (csum / nblk) / (ms * 1e3);
    printf("{\"test\": \"%s\", \"sms\": %d, \"ms\": %.4f, \"lane_ops_per_sm_per_cycle\": %.2f, \"lane_ops_per_s\": %.4e, "
           "\"flops_per_s\": %.4e, \"implied_clock_mhz\": %.0f, \"rated_clock_mhz\": %d}\n",
           name, nsm, ms, per_sm_cycle, lane_ops / (ms * 1e-3), flops_per_op * lane_ops / (ms * 1e-3), eff_clock_mhz, clk_khz / 1000);
  }
  return 0;
}
