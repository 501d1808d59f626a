// Probe: throughput of F2F.F32.F64 / F2F.F64.F32 conversions next to DFMA
// (developer tool): can part of a pair body move to the FP32 pipe?
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters, double s) {
  double d[8];
  float f[8];
  for (int i = 0; i < 8; ++i) { d[i] = threadIdx.x * 1e-3 + i; f[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) d[i] = fma(d[i], s, 1e-3);                       // DFMA only
      if (MODE == 1) f[i] = fmaf(__double2float_rn(d[i]), 1.0001f, f[i]), d[i] += 1e-9;  // F2F + FFMA + DADD
      if (MODE == 2) d[i] = fma(d[i], s, static_cast<double>(f[i])), f[i] += 1.0f;       // F2F.F64.F32 + DFMA
      if (MODE == 3) f[i] = fmaf(f[i], 1.0001f, 0.5f);                 // FFMA only
    }
  }
  double acc = 0;
  for (int i = 0; i < 8; ++i) acc += d[i] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(const char* name, double* out) {
  const int blocks = 148 * 8, threads = 256, iters = 2048;
  k<MODE><<<blocks, threads>>>(out, 16, 1.0000001);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, threads>>>(out, iters, 1.0000001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double ops = static_cast<double>(blocks) * threads * iters * 8;  // loop bodies
  printf("%-34s %8.3f ms  %8.2f G bodies/s\n", name, ms, ops / ms / 1e6);
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
  run<0>("DFMA", out);
  run<1>("F2F.F32.F64 + FFMA + DADD", out);
  run<2>("F2F.F64.F32 + DFMA + FADD", out);
  run<3>("FFMA", out);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
