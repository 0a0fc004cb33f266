// Microbenchmark: dependent-chain latency (cycles/op) of FP64 and related
// instructions on the B200 (one warp), and __syncthreads cost with 16 warps.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, double x0, int iters) {
  double x = x0 + threadIdx.x, y = 1.0000001;
  float f = (float)x0;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x * y;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // F2F round trip chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { f = (float)x; x = (double)f * y; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // double division chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // double sqrt chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // FFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) f = fmaf(f, 1.0000001f, 1e-9f);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
  out[threadIdx.x] = x + f;
}

__global__ void barriers(long long* cyc, int iters) {
  __shared__ int s;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { if (threadIdx.x == i % blockDim.x) s = i; __syncthreads(); }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0);
}

// FP64 FMA issue throughput of one SM: nt threads, 8 independent chains each
__global__ void thru(double* out, long long* cyc, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + threadIdx.x + k;
  const double y = 1.0000001;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], y, 1e-9);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = t1 - t0;
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[threadIdx.x] = s;
}
// shared-memory 64-bit load/store throughput of one SM (conflict-free rows)
__global__ void smem_thru(double* out, long long* cyc, int iters) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
  __syncthreads();
  double s = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) s += buf[(threadIdx.x + 512 * k + 32 * i) & 4095];
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[8] = t1 - t0;
  out[threadIdx.x] = s;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const int it = 4096;
  chain<<<1, 32>>>(out, cyc, 1.5, it);
  cudaDeviceSynchronize();
  chain<<<1, 32>>>(out, cyc, 1.5, it);
  cudaDeviceSynchronize();
  const char* nm[] = {"DFMA", "DMUL", "F2F+DMUL roundtrip", "DDIV(1/x)", "DSQRT", "FFMA"};
  for (int i = 0; i < 6; ++i) printf("%-20s %.1f cycles/op\n", nm[i], (double)cyc[i] / it);
  for (int nt : {256, 512}) {
    barriers<<<1, nt>>>(cyc, it);
    cudaDeviceSynchronize();
    printf("__syncthreads %d threads: %.1f cycles\n", nt, (double)cyc[6] / it);
  }
  for (int nt : {32, 128, 512}) {
    thru<<<1, nt>>>(out, cyc, 2048);
    cudaDeviceSynchronize();
    printf("DFMA throughput %d threads: %.2f warp-instr/clk (%.1f lanes/clk/SM)\n", nt,
           2048.0 * 8 * (nt / 32) / cyc[7], 2048.0 * 8 * nt / cyc[7]);
  }
  for (int nt : {32, 128, 512}) {
    smem_thru<<<1, nt>>>(out, cyc, 2048);
    cudaDeviceSynchronize();
    printf("LDS.64 throughput %d threads: %.1f B/clk/SM (incl. dependent DADD)\n", nt,
           2048.0 * 8 * nt * 8 / cyc[8]);
  }
  return 0;
}
