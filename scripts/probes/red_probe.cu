// Probe: FP64 global atomic-add (REDG) throughput by address pattern
// (developer tool): random distinct addresses, warp-contiguous 8-byte
// addresses, and 16 lanes per 128-byte line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void red_kernel(double* z, long long n, int mode, int iters) {
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned h = static_cast<unsigned>(tid) * 2654435761u;
  for (int it = 0; it < iters; ++it) {
    long long a;
    h = h * 1664525u + 1013904223u;
    const long long warp = tid >> 5, lane = tid & 31;
    const unsigned hw = (static_cast<unsigned>(warp) * 2246822519u + it * 3266489917u);
    if (mode == 0) a = h % n;                                        // random per lane
    else if (mode == 1) a = ((hw % (n / 32)) * 32 + lane);           // warp-contiguous 256 B
    else if (mode == 2) a = ((hw % (n / 32)) * 32 + (lane & 15) + ((h >> 7) % 2) * 16);  // 2 lanes per address
    else a = ((static_cast<unsigned>(tid >> 4) * 2246822519u + it * 3266489917u) % (n / 16)) * 16 + (lane & 15);  // 16 lanes / line
    atomicAdd(z + a, 1.0);
  }
}

int main() {
  const long long n = 1ll << 25;  // 256 MB of doubles
  double* z;
  cudaMalloc(&z, n * sizeof(double));
  cudaMemset(z, 0, n * sizeof(double));
  const int blocks = 148 * 16, threads = 256, iters = 256;
  const char* names[] = {"random 8B per lane", "warp-contiguous 256B", "pairs of lanes same addr", "16 lanes per 128B line"};
  for (int mode = 0; mode < 4; ++mode) {
    red_kernel<<<blocks, threads>>>(z, n, mode, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    red_kernel<<<blocks, threads>>>(z, n, mode, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = static_cast<double>(blocks) * threads * iters;
    printf("%-28s %8.3f ms  %7.2f G atomics/s\n", names[mode], ms, ops / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
