// Standalone probe of tc::gemm_tf32_kernel (tcgen05 kind::tf32) against a host fp64 GEMM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2201_10369_b200/csrc tools/probe/tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "tc_gemm.cuh"

int main(int argc, char** argv) {
  const int Cp = argc > 1 ? atoi(argv[1]) : 32, Kp = argc > 2 ? atoi(argv[2]) : 128;
  const long long Tp = argc > 3 ? atoll(argv[3]) : 256;
  const int mode = argc > 4 ? atoi(argv[4]) : 0;   // 0 random ints, 1 A = identity-ish
  std::vector<float> U((size_t)Cp * Kp), V((size_t)Cp * Tp), M((size_t)Kp * Tp);
  srand(1);
  for (int c = 0; c < Cp; c++)
    for (int k = 0; k < Kp; k++) U[(size_t)c * Kp + k] = mode == 1 ? (c == (k % Cp) ? 1.f : 0.f) : (float)(rand() % 7 - 3);
  for (int c = 0; c < Cp; c++)
    for (long long t = 0; t < Tp; t++) V[(size_t)c * Tp + t] = mode == 1 ? (float)(c * 1000 + t) : (float)(rand() % 7 - 3);
  float *dU, *dV, *dM;
  cudaMalloc(&dU, U.size() * 4); cudaMalloc(&dV, V.size() * 4); cudaMalloc(&dM, M.size() * 4);
  cudaMemcpy(dU, U.data(), U.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dM, 0xff, M.size() * 4);
  cudaFuncSetAttribute((const void*)wino::tc::gemm_tf32_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, wino::tc::Cfg<1>::kSmem);
  const int grid = argc > 5 ? atoi(argv[5]) : 148;   // persistent CTAs (fewer -> several tiles each)
  CUtensorMap tmU, tmV, tmM;
  const char* sw = getenv("TC_SWZ");
  const CUtensorMapSwizzle swz = (!sw || !*sw) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                     : (atoi(sw) == 1 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!wino::tc::encode_map_2d(&tmU, dU, Kp, Cp, swz) || !wino::tc::encode_map_2d(&tmV, dV, Tp, Cp, swz) ||
      !wino::tc::encode_map_2d(&tmM, dM, Tp, Kp, CU_TENSOR_MAP_SWIZZLE_128B)) {
    printf("encode failed\n");
    return 2;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 4; rep++) {
    cudaEventRecord(e0);
    wino::tc::gemm_tf32_kernel<1><<<grid, wino::tc::kThreads, wino::tc::Cfg<1>::kSmem>>>(tmU, tmV, tmU, tmV, tmM, Cp, Kp, Tp, 1);
    cudaEventRecord(e1);
  }
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("kernel: %s  %.3f ms\n", cudaGetErrorString(e), ms);
  cudaMemcpy(M.data(), dM, M.size() * 4, cudaMemcpyDeviceToHost);
  long long bad = 0, nan = 0, zero = 0;
  if (getenv("TC_NOCHECK")) return 0;
  for (int k = 0; k < Kp; k++)
    for (long long t = 0; t < Tp; t++) {
      double ref = 0;
      for (int c = 0; c < Cp; c++) ref += (double)U[(size_t)c * Kp + k] * V[(size_t)c * Tp + t];
      float got = M[(size_t)k * Tp + t];
      if (std::isnan(got)) nan++;
      if (got == 0.f) zero++;
      if ((double)got != ref) {
        if (bad < 12) printf("k=%d t=%lld got %g ref %g\n", k, t, got, ref);
        bad++;
      }
    }
  printf("Cp=%d Kp=%d Tp=%lld mode=%d: bad %lld / %lld (nan %lld zero %lld)\n", Cp, Kp, Tp, mode, bad,
         (long long)Kp * Tp, nan, zero);
  for (int k = 0; k < 3; k++) {
    printf("row %d:", k);
    for (int t = 0; t < 12; t++) printf(" %g", M[(size_t)k * Tp + t]);
    printf("\n");
  }
  return bad != 0;
}
