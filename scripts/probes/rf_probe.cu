// Probe: does register-file operand bandwidth (not the FP64 pipe) bound a
// realistic DFMA stream on sm_100a? DFMA chains whose instructions read 1, 2
// or 3 "fresh" 64-bit vector-register operands (no .reuse hit possible, no
// uniform-register / immediate operand), alone and interleaved with integer
// instructions, at 2 and 16 warps per scheduler (developer tool; prints
// TFLOP/s, FMA = 2 flops).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rf_probe rf_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int C = 8;  // independent chains per thread

struct Tab {
  double v[256];
  int row[64];
};

// MODE 0: x = fma(x, s, b)      s uniform register, b immediate-like constant  (1 fresh pair)
// MODE 1: x = fma(x, y_c, 0.5)  y_c per chain                                 (2 fresh pairs)
// MODE 2: x = fma(x, y_c, w_c)  y_c, w_c per chain                            (3 fresh pairs)
// MODE 3: x = fma(x, sr, br)    sr, br per thread, same for all chains        (3 pairs, 2 reusable)
// MODE 4: t = fma(x, y_c, w_c) written to another register set (dest != src)  (3 fresh pairs, no in-place)
// NI: one 3-instruction integer update (SHF, LOP3, IMAD on private registers) on NI of every 4 DFMAs
template <int MODE, int NI>
__global__ void __launch_bounds__(256, (MODE >= 5 ? 4 : 1)) probe(double* out, const double* in, int iters, double s,
                                             const __grid_constant__ Tab tab) {
  __shared__ double sm[256];
  sm[threadIdx.x] = in[threadIdx.x];
  __syncthreads();
  double x[C], y[C], w[C];
  unsigned k[C];
  const double sr = in[threadIdx.x], br = in[threadIdx.x + 256];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    x[c] = c * 0.5;
    y[c] = in[threadIdx.x + 32 * c];
    w[c] = in[threadIdx.x + 32 * c + 512];
    k[c] = threadIdx.x * 7 + c;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (MODE == 0) x[c] = fma(x[c], s, 0.5);
        if (MODE == 1) x[c] = fma(x[c], y[c], 0.5);
        if (MODE == 2) x[c] = fma(x[c], y[c], w[c]);
        if (MODE == 3) x[c] = fma(x[c], sr, br);
        if (MODE == 4) {
          const double t = fma(x[c], y[c], w[c]);
          w[c] = y[c];
          y[c] = x[c];
          x[c] = t;
        }
        // MODE 5: multiplier from the parameter constant bank at a compile-time offset (64 registers max: not hoisted)
        if (MODE == 5) x[c] = fma(x[c], tab.v[u * C + c], 0.5);
        // MODE 6: ... at a runtime (uniform) row offset read from the same bank (LDCU + uniform address math)
        if (MODE == 6) x[c] = fma(x[c], tab.v[tab.row[u] + c], 0.5);
        // MODE 7: multiplier from shared memory at a warp-uniform address (LDS.64 broadcast per DFMA)
        if (MODE == 7) x[c] = fma(x[c], sm[(it + u * C + c) & 255], 0.5);
        // MODE 8: ... one LDS.128 per two DFMAs
        if (MODE == 8) {
          if (c % 2 == 0) {
            const double2 m = *reinterpret_cast<const double2*>(&sm[(2 * it + u * C + c) & 254]);
            x[c] = fma(x[c], m.x, 0.5);
            x[c + 1] = fma(x[c + 1], m.y, 0.5);
          }
        }
        // MODE 9: 64-bit immediates with a nonzero low word (UMOV pairs or constant bank)
        if (MODE == 9) x[c] = fma(x[c], 1.0 + 1e-9 * (u * C + c + 1), 0.5);
        if (NI > 0 && (u * C + c) % 4 < NI) k[c] = (k[c] ^ (k[(c + 1) % C] >> 3)) * 5u + 1u;
        if (NI > 4 && (u * C + c) % 4 < NI - 4) k[(c + 3) % C] = (k[(c + 3) % C] + k[(c + 5) % C]) ^ 0x5bd1e995u;
      }
    }
  }
  double acc = 0;
  unsigned ka = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    acc += x[c] + y[c] + w[c];
    ka += k[c];
  }
  if (acc == -12345.678 || ka == 0x12345u) out[0] = acc + ka;
}

template <int MODE, int NI>
void run(const char* name, int ctasPerSm, double* out, const double* in) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * ctasPerSm, iters = 4000;
  static Tab tab;
  for (int i = 0; i < 256; ++i) tab.v[i] = 1.0 + 1e-9 * i;
  for (int i = 0; i < 64; ++i) tab.row[i] = (i * 24) % 184;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<MODE, NI><<<blocks, 256>>>(out, in, iters, 1.0000001, tab);
  double best = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    probe<MODE, NI><<<blocks, 256>>>(out, in, iters, 1.0000001, tab);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * C * 8 * iters * double(blocks) * 256 / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  printf("%-44s %d warps/scheduler: %6.2f TFLOP/s  (%s)\n", name, ctasPerSm * 2, best, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *out, *in;
  cudaMalloc(&out, 8);
  cudaMalloc(&in, 2048 * 8);
  double h[2048];
  for (int i = 0; i < 2048; ++i) h[i] = 1.0 + 1e-9 * i;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int occ : {1, 2, 8}) {
#define ROW(M, NI, name)                                  \
  if (occ == 1) run<M, NI>(name, 1, out, in);             \
  else if (occ == 2) run<M, NI>(name, 2, out, in);        \
  else run<M, NI>(name, 8, out, in);
    ROW(0, 0, "1 fresh (uniform mult, imm add)")
    ROW(1, 0, "2 fresh (x, y_c; imm add)")
    ROW(2, 0, "3 fresh (x, y_c, w_c)")
    ROW(3, 0, "3 regs, 2 reusable")
    ROW(4, 0, "3 fresh, rotating dest")
    ROW(0, 1, "1 fresh + 0.75 int instr / DFMA")
    ROW(0, 2, "1 fresh + 1.5 int instr / DFMA")
    ROW(1, 1, "2 fresh + 0.75 int instr / DFMA")
    ROW(1, 2, "2 fresh + 1.5 int instr / DFMA")
    ROW(2, 1, "3 fresh + 0.75 int instr / DFMA")
    ROW(4, 1, "3 fresh rotating + 0.75 int instr / DFMA")
    ROW(1, 4, "2 fresh + 3 int instr / DFMA (issue-bound)")
    ROW(5, 0, "1 fresh, const-bank multiplier (fixed offset)")
    ROW(6, 0, "1 fresh, const-bank multiplier (runtime row)")
    ROW(7, 0, "1 fresh, LDS.64 broadcast multiplier per DFMA")
    ROW(8, 0, "1 fresh, LDS.128 broadcast per 2 DFMA")
    ROW(9, 0, "1 fresh, 64-bit immediate multiplier")
  }
  return 0;
}
