// FP64 tensor-core issue-rate microbenchmark for the mma.sync f64 shapes on
// sm_100a: independent accumulator chains per warp, all SMs, no memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_rate dmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void kern(double* out, int iters) {
  // SHAPE 0: m8n8k4 (acc 2, a 1, b 1)   1: m16n8k4 (acc 4, a 2, b 1)
  //       2: m16n8k8 (acc 4, a 4, b 2)   3: m16n8k16 (acc 4, a 8, b 4)
  constexpr int CH = 4;   // independent accumulators per warp
  double acc[CH][4];
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - 1e-9 * (threadIdx.x + i);
  for (int c = 0; c < CH; ++c)
    for (int e = 0; e < 4; ++e) acc[c][e] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a[0]), "d"(b[0]));
      else if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int c = 0; c < CH; ++c)
    for (int e = 0; e < 4; ++e) s += acc[c][e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SHAPE>
void run(const char* name, double fma_per_inst, int warps) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * nsm * warps * 32);
  const int iters = 20000;
  kern<SHAPE><<<nsm, warps * 32>>>(out, 100);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<SHAPE><<<nsm, warps * 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * fma_per_inst * 4 * (double)iters * warps * nsm;
  printf("%-10s warps/SM %2d: %.2f TFLOP/s\n", name, warps, fl / ms / 1e9);
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16, 32}) {
    run<0>("m8n8k4", 8 * 8 * 4, w);
    run<1>("m16n8k4", 16 * 8 * 4, w);
    run<2>("m16n8k8", 16 * 8 * 8, w);
    run<3>("m16n8k16", 16 * 8 * 16, w);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
