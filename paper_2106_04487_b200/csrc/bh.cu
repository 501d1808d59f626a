// Barnes-Hut monopole far field (plans built with FktOptions::barnesHut).
//
// Reference: the plan forces p = 0 and stores every node's centre of mass
// (transform.cpp:44-60); the far field of node b is
//   z_t += K(|x_t - com_b|) * sum_{src in b} y_src      for t in F_b
// (transform.cpp:131-146), evaluated as evalPositive(sqrt(dist2)); the near
// field is the same exact leaf block as the FKT (transform.cpp:163-181), so
// it reuses K3. barnesHutMultiply (transform.cpp:239-243) is multiply on
// such a plan.
//
// GPU mapping: the per-node totals are the p = 0 "moments" ([rhs][node], one
// coefficient per node), summed by CTA per (node, source tile) like K4 and
// exchanged like the FKT moments under target sharding; the far kernel is
// one thread per far-list entry (the node's centre of mass and totals are
// uniform per CTA: L1 broadcast loads).
#include "common.cuh"
#include "device_math.cuh"
#include "plan.hpp"

namespace fktb {
namespace {

constexpr int kThreads = 256;

// Centre of mass of node b: mean of its permuted points (tree.hpp pointAt).
__global__ void bh_com_kernel(int n, int d, const double* pc, const uint32_t* begin, const uint32_t* end,
                              double* com) {
  const int b = blockIdx.x;
  const uint32_t p0 = begin[b], p1 = end[b];
  __shared__ double red[kThreads / 32];
  for (int a = 0; a < d; ++a) {
    double s = 0.0;
    for (uint32_t p = p0 + threadIdx.x; p < p1; p += kThreads) s += pc[static_cast<size_t>(a) * n + p];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) t += red[w];
      com[static_cast<size_t>(b) * d + a] = t / static_cast<double>(p1 - p0);
    }
    __syncthreads();
  }
}

// totals[r][node] += sum of yp over one source tile of the node (deterministic
// mode: part[tile][r] = the tile's sum, reduced in tile order by det.cu).
__global__ void bh_sum_kernel(int n, int nodes, int nrhs, const FktbTile* tiles, const double* yp, double* totals,
                              double* part) {
  const FktbTile tile = tiles[blockIdx.x];
  __shared__ double red[kThreads / 32];
  for (int r = 0; r < nrhs; ++r) {
    double s = 0.0;
    for (int i = threadIdx.x; i < tile.count; i += kThreads) s += yp[static_cast<size_t>(r) * n + tile.start + i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) t += red[w];
      if (part)
        part[static_cast<size_t>(blockIdx.x) * nrhs + r] = t;
      else
        atomicAdd(totals + static_cast<size_t>(r) * nodes + tile.node, t);
    }
    __syncthreads();
  }
}

// z[t] += K(|x_t - com_b|) * totals[r][b] for the far-list entries of one tile.
__global__ void bh_far_kernel(int n, int d, int nodes, int nrhs, const double* pc, const double* com,
                              const FktbTile* tiles, const uint32_t* farPos, const FktbKernelDesc kd,
                              const double* totals, const ZOut out) {
  const FktbTile tile = tiles[blockIdx.x];
  for (int i = threadIdx.x; i < tile.count; i += kThreads) {
    const uint32_t pos = farPos[tile.start + i];
    double dist2 = 0.0;
    for (int a = 0; a < d; ++a) {
      const double t = pc[static_cast<size_t>(a) * n + pos] - com[static_cast<size_t>(tile.node) * d + a];
      dist2 = fma(t, t, dist2);
    }
    const double k = kernel_value_rt(kd, sqrt(dist2));
    for (int r = 0; r < nrhs; ++r) out.add(r, tile.start + i, pos, k * totals[static_cast<size_t>(r) * nodes + tile.node]);
  }
}

}  // namespace

void buildBarnesHut(DevicePlan& plan) {
  const DeviceTree& t = *plan.tree;
  plan.dCom.resize(static_cast<size_t>(t.nodes) * t.d);
  bh_com_kernel<<<t.nodes, kThreads, 0, plan.stream>>>(t.n, t.d, t.pc.get(), t.dBegin.get(), t.dEnd.get(),
                                                      plan.dCom.get());
  FKTB_CUDA(cudaGetLastError());
}

void launchBHSums(const DevicePlan& plan, const double* yp, double* totals, int nrhs, cudaStream_t st) {
  const int tiles = static_cast<int>(plan.s2mTilesHost.size());
  if (tiles == 0) return;
  double* part = plan.options.deterministic ? plan.dTilePart.get() : nullptr;
  bh_sum_kernel<<<tiles, kThreads, 0, st>>>(plan.n, plan.tree->nodes, nrhs, plan.dS2mTiles.get(), yp, totals, part);
  FKTB_CUDA(cudaGetLastError());
  if (part) launchDetTileSum(plan, part, 1, nrhs, totals, st);
}

void launchBHFar(const DevicePlan& plan, const double* totals, double* zp, int nrhs, cudaStream_t st) {
  const int tiles = static_cast<int>(plan.farTilesHost.size());
  if (tiles == 0) return;
  const DeviceTree& t = *plan.tree;
  FktbKernelDesc kd;
  fillKernelDesc(plan.kernel, kd);
  bh_far_kernel<<<tiles, kThreads, 0, st>>>(t.n, t.d, t.nodes, nrhs, t.pc.get(), plan.dCom.get(), plan.dFarTiles.get(),
                                            t.dFarPos.get(), kd, totals, zoutFor(plan, zp, nrhs, true));
  FKTB_CUDA(cudaGetLastError());
}

}  // namespace fktb
