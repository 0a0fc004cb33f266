// DGEMM rate of the library's DMMA GEMM (gemm.cu) on the shapes the sweeps
// use, next to cuBLAS-free ceilings (37 TFLOP/s DMMA issue rate).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude
//   -Ipaper_1707_07803_b200/csrc tools/ubench/gemm_rate.cu
//   paper_1707_07803_b200/csrc/gemm.cu paper_1707_07803_b200/csrc/core_ops.cu
//   -o tools/ubench/gemm_rate
#include <cstdio>
#include "kernels.cuh"
namespace mpob { unsigned long long g_launches = 0; }
int main() {
  using namespace mpob;
  cudaStream_t st;
  cudaStreamCreate(&st);
  struct S { bool ta, tb; int64_t m, n, k; };
  S shapes[] = {{false, false, 4096, 4096, 4096}, {true, false, 4096, 4096, 4096},
                {false, true, 4096, 4096, 4096}, {false, false, 7680, 4083, 4096},
                {true, false, 128, 3840, 3840}, {false, false, 3840, 3840, 128},
                {false, true, 6144, 8192, 4096}, {false, false, 3072, 8192, 49152}};
  for (auto& s : shapes) {
    const int64_t lda = s.ta ? s.k : s.m, ldb = s.tb ? s.n : s.k;
    double *A, *B, *C;
    cudaMalloc(&A, sizeof(double) * s.m * s.k);
    cudaMalloc(&B, sizeof(double) * s.k * s.n);
    cudaMalloc(&C, sizeof(double) * s.m * s.n);
    cudaMemset(A, 0, sizeof(double) * s.m * s.k);
    cudaMemset(B, 0, sizeof(double) * s.k * s.n);
    dgemm(st, s.ta, s.tb, s.m, s.n, s.k, 1.0, A, lda, B, ldb, 0.0, C, s.m);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 5;
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) dgemm(st, s.ta, s.tb, s.m, s.n, s.k, 1.0, A, lda, B, ldb, 0.0, C, s.m);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%c%c m=%6lld n=%6lld k=%6lld: %8.3f ms %6.2f TFLOP/s\n", s.ta ? 'T' : 'N', s.tb ? 'T' : 'N',
           (long long)s.m, (long long)s.n, (long long)s.k, ms, 2.0 * s.m * s.n * s.k / ms / 1e9);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
