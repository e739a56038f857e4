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
  for (int test = 0; test < 7; test++) {
    const char* name = nullptr; double ops_per_thread_iter = 0; int flops_per_op = 2;
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
      }
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
    }
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(hc, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
    double cmax = 0, csum = 0; for (int b = 0; b < blocks; b++) { csum += hc[b]; if (hc[b] > cmax) cmax = hc[b]; }
    double lane_ops = (double)blocks * threads * ITER * ops_per_thread_iter;
    // per SM per cycle, using the mean per-block cycle span (blocks on one SM run concurrently: per_sm * threads)
    double per_sm_cycle = (double)per_sm * threads * ITER * ops_per_thread_iter / (csum / blocks);
    double eff_clock_mhz = (csum / blocks) / (ms * 1e3);
    printf("{\"test\": \"%s\", \"sms\": %d, \"ms\": %.4f, \"lane_ops_per_sm_per_cycle\": %.2f, \"lane_ops_per_s\": %.4e, "
           "\"flops_per_s\": %.4e, \"implied_clock_mhz\": %.0f, \"rated_clock_mhz\": %d}\n",
           name, nsm, ms, per_sm_cycle, lane_ops / (ms * 1e-3), flops_per_op * lane_ops / (ms * 1e-3), eff_clock_mhz, clk_khz / 1000);
  }
  return 0;
}
