// Probe: FP64 tensor-core (mma.sync m8n8k4 f64) throughput on sm_100a, alone
// and interleaved with DFMA chains, to see whether DMMA issues on a pipe of
// its own (developer tool; prints TFLOP/s).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int NM, int NF>
__global__ void probe(double* out, int iters, double s) {
  double c[8][2];
  double f[8];
  double a = threadIdx.x * 1e-3, b = s;
  for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = i; f[i] = i * 0.5; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NM; ++i) dmma(c[i], a, b);
#pragma unroll
    for (int j = 0; j < NF; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = fma(f[i], s, a);
  }
  double acc = 0;
  for (int i = 0; i < 8; ++i) acc += c[i][0] + c[i][1] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int NM, int NF>
void run(const char* name, double* out) {
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  probe<NM, NF><<<blocks, threads>>>(out, 16, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<NM, NF><<<blocks, threads>>>(out, iters, 1.0000001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double warps = blocks * threads / 32.0;
  const double mmaFlops = warps * iters * NM * 2.0 * 8 * 8 * 4;
  const double fmaFlops = blocks * (double)threads * iters * NF * 8 * 2.0;
  printf("%-22s %8.3f ms  dmma %6.2f TF  dfma %6.2f TF  total %6.2f TF\n", name, ms, mmaFlops / ms / 1e9,
         fmaFlops / ms / 1e9, (mmaFlops + fmaFlops) / ms / 1e9);
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
  run<8, 0>("dmma only", out);
  run<0, 4>("dfma only", out);
  run<8, 4>("dmma8 + dfma32", out);
  run<8, 2>("dmma8 + dfma16", out);
  run<4, 4>("dmma4 + dfma32", out);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
