// Legacy (mma.sync) TF32 / BF16 tensor-core and FP32 FFMA issue rates on
// sm_100a, all SMs, no memory: does a low-precision Jacobi preconditioning
// phase have headroom over the FP64 DMMA pipe (37 TFLOP/s)?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tf32_rate tf32_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void kern(float* out, int iters) {
  constexpr int CH = 4;
  float acc[CH][4];
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3f800000u + threadIdx.x + i;
  for (int i = 0; i < 2; ++i) b[i] = 0x3f800000u + threadIdx.x * 3 + i;
  for (int c = 0; c < CH; ++c)
    for (int e = 0; e < 4; ++e) acc[c][e] = 0.f;
  float x = 1.0f + threadIdx.x * 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else if (KIND == 1)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else {
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[c][e] = fmaf(acc[c][e], x, 1.0f);
      }
    }
  }
  float s = 0;
  for (int c = 0; c < CH; ++c)
    for (int e = 0; e < 4; ++e) s += acc[c][e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND>
void run(const char* name, double flop_per_inst_warp, int warps) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * nsm * warps * 32);
  const int iters = 20000;
  kern<KIND><<<nsm, warps * 32>>>(out, 100);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<KIND><<<nsm, warps * 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = flop_per_inst_warp * 4 * (double)iters * warps * nsm;
  printf("%-22s warps/SM %2d: %.1f TFLOP/s\n", name, warps, fl / ms / 1e9);
  cudaFree(out);
}

int main() {
  for (int w : {8, 16, 32}) {
    run<0>("tf32 m16n8k8", 2.0 * 16 * 8 * 8, w);
    run<1>("bf16 m16n8k16", 2.0 * 16 * 8 * 16, w);
    run<2>("fp32 ffma (x4/thread)", 2.0 * 4 * 32, w);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
