// Plan construction and the MVM pipeline (reference proj/src/transform.cpp:39-204).
//
// Plan: GPU tree (K1) -> GPU interaction sets (K2) -> exact tables on the host
// (coefficients, harmonics, optional compression) -> kernel-parameter tables
// and work tiles. Multiply: gather y into tree order -> S2M (K4) -> near (K3)
// -> M2T (K5) -> scatter z back, all on one stream.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "device_math.cuh"
#include "fastmath.cuh"
#include "moments.hpp"
#include "plan.hpp"

namespace fktb {

int nearTileSize();
int farTileSize();
int genericGMax();
int s2mRhsChunk(int P);

namespace {

constexpr int kS2MTileSources = 4096;

bool specialised(int d, int p) {
  const int key = d * 100 + p;
  return key == 206 || key == 304 || key == 306 || key == 308 || key == 504;
}

void buildFarParams(DevicePlan& plan) {
  const int d = plan.d, p = plan.options.p;
  const HarmonicStructure& hs = *plan.harmonics;
  const CoefTable& table = coefTable(d, p);
  auto fp = std::make_unique<FktbFarParams>();
  std::memset(fp.get(), 0, sizeof(FktbFarParams));
  fp->d = d;
  fp->p = p;
  fp->compressed = plan.compressed ? 1 : 0;
  fillKernelDesc(plan.kernel, fp->kernel);
  int cOff = 0, hOff = 0, tOff = 0, pref = 0;
  for (int k = 0; k <= p; ++k) {
    fp->hOff[k] = hOff;
    fp->cOff[k] = cOff;
    fp->tOff[k] = tOff;
    const int hk = static_cast<int>(hs.degreeCount(k));
    const int su = (p - k) / 2 + 1;
    fp->slotsU[k] = su;
    fp->slots[k] = plan.compressed ? plan.factors[static_cast<size_t>(k)].rank : su;
    pref += hk * fp->slots[k];
    hOff += hk;
    cOff += hk * su;
    tOff += su;
  }
  fp->hOff[p + 1] = hOff;
  fp->cOff[p + 1] = cOff;
  fp->tOff[p + 1] = tOff;
  fp->P = cOff;
  fp->H = hOff;
  fp->Pref = pref;
  // Radial table rows: Tbar_kjm * m!
  int at = 0;
  for (int k = 0; k <= p; ++k)
    for (int s = 0; k + 2 * s <= p; ++s) {
      const int j = k + 2 * s;
      fp->tRow[fp->tOff[k] + s] = at;
      double fact = 1.0;
      for (int m = 1; m <= j; ++m) {
        fact *= m;
        if (at >= FKTB_TBAR_CAP) throw std::invalid_argument("expansion table exceeds the GPU parameter capacity");
        fp->tb[at++] = table.tbarDouble(k, j, m) * fact;
        // the compiled d = 3 kernels skip m < tbarFirstM(3, k, j) (far.cu):
        // those entries must be exact zeros of the table
        if (d == 3 && m < tbarFirstM(3, k, j) && table.tbarDouble(k, j, m) != 0.0)
          throw std::logic_error("T-bar zero pattern violated for d = 3");
      }
    }
  if (plan.compressed) {
    int f = 0, c = 0;
    for (int k = 0; k <= p; ++k) {
      fp->fOff[k] = f;
      const RadialFactor& rf = plan.factors[static_cast<size_t>(k)];
      for (int i = 0; i < rf.rank; ++i, ++f) {
        if (f >= FKTB_FACTOR_MAX) throw std::invalid_argument("compression factors exceed the GPU parameter capacity");
        const Laurent& F = rf.target[static_cast<size_t>(i)];
        const Laurent& G = rf.source[static_cast<size_t>(i)];
        fp->fLo[f] = F.minPower();
        fp->fHi[f] = F.maxPower();
        fp->fAt[f] = c;
        for (int e = F.minPower(); e <= F.maxPower(); ++e) {
          if (c >= FKTB_FACTOR_CAP) throw std::invalid_argument("compression factors exceed the GPU parameter capacity");
          fp->fc[c++] = toDouble(F.coeff(e));
        }
        fp->gLo[f] = G.minPower();
        fp->gHi[f] = G.maxPower();
        fp->gAt[f] = c;
        for (int e = G.minPower(); e <= G.maxPower(); ++e) {
          if (c >= FKTB_FACTOR_CAP) throw std::invalid_argument("compression factors exceed the GPU parameter capacity");
          fp->fc[c++] = toDouble(G.coeff(e));
        }
      }
    }
    fp->fOff[p + 1] = f;
    // dense windows (see compressed_window_lo/hi)
    fp->denseLo = compressed_window_lo(plan.kernel.id, p);
    fp->denseHi = compressed_window_hi(plan.kernel.id, p);
    const int span = fp->denseHi - fp->denseLo + 1;
    bool fits = c + f * span <= FKTB_FACTOR_CAP;
    // the specialised fused M2T reads rank <= comp_slots per degree, each
    // factor over its degree window (device_math.cuh): verify here
    for (int k = 0; k <= p && fits; ++k) {
      const int kid = plan.kernel.id;
      if (plan.factors[static_cast<size_t>(k)].rank > comp_slots(kid, p, k)) fits = false;
      if (comp_rank_exact(kid) && plan.factors[static_cast<size_t>(k)].rank != comp_slots(kid, p, k)) fits = false;
      for (const Laurent& F : plan.factors[static_cast<size_t>(k)].target)
        if (F.minPower() < comp_degree_lo(kid, p, k) || F.maxPower() > comp_degree_hi(kid, p, k)) fits = false;
    }
    fp->denseAt = -1;
    if (fits) {
      fp->denseAt = c;
      for (int k = 0; k <= p; ++k) {
        const RadialFactor& rf = plan.factors[static_cast<size_t>(k)];
        for (int i = 0; i < rf.rank; ++i) {
          const int fi = fp->fOff[k] + i;
          for (int e = fp->denseLo; e <= fp->denseHi; ++e)
            fp->fc[fp->denseAt + fi * span + e - fp->denseLo] = toDouble(rf.target[static_cast<size_t>(i)].coeff(e));
        }
      }
    }
  }
  plan.P = fp->P;
  plan.H = fp->H;

  // Per-harmonic fold Z_k * nrm_h^2 and the runtime chain table.
  std::vector<double> hscale(static_cast<size_t>(fp->H)), kappaHost(static_cast<size_t>(fp->H), 1.0);
  const int L = d > 2 ? d - 2 : 0;
  std::vector<int> cg(static_cast<size_t>(std::max(1, fp->H * L))), cc(static_cast<size_t>(fp->H)), ph(static_cast<size_t>(fp->H));
  for (int k = 0; k <= p; ++k) {
    int h = fp->hOff[k];
    for (const HarmonicChain& ch : hs.chains(k)) {
      // Z_k nrm^2 times kappa^2 for the monic-scaled Gegenbauer chains
      // evaluated on both sides (device_math.cuh gegen_kappa)
      double kappa = 1.0;
      for (int l = 1; l <= L; ++l)
        kappa *= gegen_kappa(d - 1 - l + 2 * ch.m[static_cast<size_t>(l)], ch.m[static_cast<size_t>(l - 1)] - ch.m[static_cast<size_t>(l)]);
      kappaHost[static_cast<size_t>(h)] = kappa;
      hscale[static_cast<size_t>(h)] = hs.z(k) * ch.norm * ch.norm * kappa * kappa;
      for (int l = 1; l <= L; ++l) cg[static_cast<size_t>(h * L + l - 1)] = g_index(p, l, ch.m[static_cast<size_t>(l)], ch.m[static_cast<size_t>(l - 1)] - ch.m[static_cast<size_t>(l)]);
      cc[static_cast<size_t>(h)] = d == 2 ? k : ch.m[static_cast<size_t>(d - 2)];
      ph[static_cast<size_t>(h)] = ch.phase;
      ++h;
    }
  }
  cudaStream_t st = plan.stream;
  {
    // fused M2T at d = 3 (far.cu): its Gegenbauer table holds D_n = n! C_n =
    // n! kappa_n * (monic value), n = k - m, so the staged moments carry the inverse
    std::vector<double> ms(static_cast<size_t>(std::max(1, fp->P)), 1.0);
    if (d == 3)
      for (int k = 0; k <= p; ++k) {
        const int nh = fp->hOff[k + 1] - fp->hOff[k], su = (p - k) / 2 + 1;
        for (int j = 0; j < nh; ++j) {
          const int h = fp->hOff[k] + j, n = k - cc[static_cast<size_t>(h)];
          double f = kappaHost[static_cast<size_t>(h)];
          for (int i = 2; i <= n; ++i) f *= i;
          for (int s2 = 0; s2 < su; ++s2) ms[static_cast<size_t>(fp->cOff[k] + s2 * nh + j)] = 1.0 / f;
          // compressed Laplace plans: the single target factor F_k = c_k r^-k
          // (the fused kernel multiplies by r^-(k+1) only)
          if (plan.compressed && plan.kernel.id == FKTB_KERNEL_INVERSE_R && fp->denseAt >= 0) {
            const int span = fp->denseHi - fp->denseLo + 1;
            ms[static_cast<size_t>(fp->cOff[k] + j)] *= fp->fc[fp->denseAt + fp->fOff[k] * span + (-k - fp->denseLo)];
          }
        }
      }
    plan.dM2tScale.resize(ms.size());
    FKTB_CUDA(cudaMemcpyAsync(plan.dM2tScale.get(), ms.data(), plan.dM2tScale.bytes(), cudaMemcpyHostToDevice, st));
    FKTB_CUDA(cudaStreamSynchronize(st));  // ms is a host temporary
  }
  plan.hscaleHost = hscale;
  plan.kappaHost = kappaHost;
  plan.dHScale.resize(hscale.size());
  plan.dChainG.resize(cg.size());
  plan.dChainC.resize(cc.size());
  plan.dChainPh.resize(ph.size());
  FKTB_CUDA(cudaMemcpyAsync(plan.dHScale.get(), hscale.data(), plan.dHScale.bytes(), cudaMemcpyHostToDevice, st));
  FKTB_CUDA(cudaMemcpyAsync(plan.dChainG.get(), cg.data(), plan.dChainG.bytes(), cudaMemcpyHostToDevice, st));
  FKTB_CUDA(cudaMemcpyAsync(plan.dChainC.get(), cc.data(), plan.dChainC.bytes(), cudaMemcpyHostToDevice, st));
  FKTB_CUDA(cudaMemcpyAsync(plan.dChainPh.get(), ph.data(), plan.dChainPh.bytes(), cudaMemcpyHostToDevice, st));
  plan.far = std::move(fp);
}

// Work tiles over the lists; under a shard (shard.cu) only the owned targets'
// sub-range of every list and the owned sources.
void buildTiles(DevicePlan& plan) {
  const DeviceTree& t = *plan.tree;
  const int ft = farTileSize(), nt = nearTileSize();
  plan.farTilesHost.clear();
  plan.nearTilesHost.clear();
  plan.s2mTilesHost.clear();
  const long long lo = plan.shardLo, hi = plan.shardHi;
  for (int b = 0; b < t.nodes; ++b) {
    const size_t B = static_cast<size_t>(b);
    const bool farAny = t.farOff[B + 1] > t.farOff[B];
    const long long f0 = plan.farSub.empty() ? t.farOff[B] : plan.farSub[2 * B];
    const long long f1 = plan.farSub.empty() ? t.farOff[B + 1] : plan.farSub[2 * B + 1];
    for (long long s = f0; s < f1; s += ft) plan.farTilesHost.push_back(FktbTile{b, static_cast<int>(std::min<long long>(ft, f1 - s)), s});
    const long long s0 = std::max<long long>(t.begin[B], lo), s1 = std::min<long long>(t.end[B], hi);
    if (farAny)
      for (long long s = s0; s < s1; s += kS2MTileSources)
        plan.s2mTilesHost.push_back(FktbTile{b, static_cast<int>(std::min<long long>(kS2MTileSources, s1 - s)), s});
    const long long n0 = plan.nearSub.empty() ? t.nearOff[B] : plan.nearSub[2 * B];
    const long long n1 = plan.nearSub.empty() ? t.nearOff[B + 1] : plan.nearSub[2 * B + 1];
    for (long long s = n0; s < n1; s += nt) plan.nearTilesHost.push_back(FktbTile{b, static_cast<int>(std::min<long long>(nt, n1 - s)), s});
  }
  {
    const auto t0 = std::chrono::steady_clock::now();
    buildNearRows(plan);  // streaming near field: Gram-first tile order (+ rows, once)
    plan.phaseSeconds[kPhaseNearRows] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  auto upload = [&](DeviceBuffer<FktbTile>& dst, const std::vector<FktbTile>& src) {
    dst.resize(std::max<size_t>(1, src.size()));
    if (!src.empty())
      FKTB_CUDA(cudaMemcpyAsync(dst.get(), src.data(), src.size() * sizeof(FktbTile), cudaMemcpyHostToDevice, plan.stream));
  };
  upload(plan.dFarTiles, plan.farTilesHost);
  upload(plan.dNearTiles, plan.nearTilesHost);
  upload(plan.dS2mTiles, plan.s2mTilesHost);
}

void clearGraphs(DevicePlan& plan) {
  for (auto& kv : plan.graphs) cudaGraphExecDestroy(kv.second.first);
  plan.graphs.clear();
  clearShardedGraphs(plan);
}

template <class T>
void uploadVec(DeviceBuffer<T>& dst, const std::vector<T>& src, cudaStream_t st) {
  dst.resize(std::max<size_t>(1, src.size()));
  if (!src.empty()) FKTB_CUDA(cudaMemcpyAsync(dst.get(), src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, st));
}

void buildP2MTiles(DevicePlan& plan);

// Tables, leaf tiles and the depth-ordered internal nodes of the monomial S2M.
void buildMomentPlan(DevicePlan& plan) {
  const DeviceTree& t = *plan.tree;
  const int d = plan.d, p = plan.options.p;
  // T maps monomial moments to sum_src Y_raw (unscaled solid harmonics); the
  // device chains are monic-scaled by 1/kappa, so rows carry hscale/kappa.
  std::vector<double> rowScale(plan.hscaleHost.size());
  for (size_t h = 0; h < rowScale.size(); ++h) rowScale[h] = plan.hscaleHost[h] / plan.kappaHost[h];
  MomentTables mt = buildMomentTables(d, p, *plan.harmonics, plan.factors, plan.compressed, rowScale);
  plan.monoCount = mt.count;
  cudaStream_t st = plan.stream;
  uploadVec(plan.dMomT, mt.T, st);
  {
    std::vector<double> tt(mt.T.size());
    const size_t Pn = mt.T.size() / static_cast<size_t>(mt.count);
    for (size_t c = 0; c < Pn; ++c)
      for (size_t a = 0; a < static_cast<size_t>(mt.count); ++a) tt[a * Pn + c] = mt.T[c * mt.count + a];
    uploadVec(plan.dMomTT, tt, st);
    FKTB_CUDA(cudaStreamSynchronize(st));  // tt is a host temporary
  }
  {
    // Cartesian M2T coefficients for the kernels that have the path
    // (FKTB_M2T_CART=0 keeps the harmonic M2T: A/B and test knob)
    static const bool cartOn = [] {
      const char* e = std::getenv("FKTB_M2T_CART");
      return !(e && e[0] == '0');
    }();
    FktbKernelDesc kd;
    fillKernelDesc(plan.kernel, kd);
    int pc = 0;
    std::vector<double> ct;
    if (cartOn && !plan.options.barnesHut) ct = buildCartTable(d, p, kd, pc);
    plan.cartP = ct.empty() ? 0 : pc;
    if (plan.cartP > 0) {
      std::vector<double> tt(ct.size());
      for (size_t c = 0; c < static_cast<size_t>(pc); ++c)
        for (size_t a = 0; a < static_cast<size_t>(mt.count); ++a) tt[a * pc + c] = ct[c * mt.count + a];
      uploadVec(plan.dCartTT, tt, st);
      FKTB_CUDA(cudaStreamSynchronize(st));
    }
  }
  plan.shiftEntries = static_cast<int>(mt.b.size());
  uploadVec(plan.dShiftOff, mt.off, st);
  uploadVec(plan.dShiftB, mt.b, st);
  uploadVec(plan.dShiftG, mt.g, st);
  uploadVec(plan.dShiftCoef, mt.coef, st);
  const MonomialBasis B(d, p);
  std::vector<int> exps;
  for (const auto& e : B.exps) exps.insert(exps.end(), e.begin(), e.end());
  uploadVec(plan.dMonoExps, exps, st);
  // depth of every node (pre-order, parents first)
  std::vector<int> depth(static_cast<size_t>(t.nodes), 0);
  int maxDepth = 0;
  plan.farNodesHost.clear();
  for (int b = 0; b < t.nodes; ++b) {
    if (t.left[static_cast<size_t>(b)] >= 0) {
      depth[static_cast<size_t>(t.left[static_cast<size_t>(b)])] = depth[static_cast<size_t>(b)] + 1;
      depth[static_cast<size_t>(t.right[static_cast<size_t>(b)])] = depth[static_cast<size_t>(b)] + 1;
    }
    maxDepth = std::max(maxDepth, depth[static_cast<size_t>(b)]);
    if (t.farOff[static_cast<size_t>(b) + 1] > t.farOff[static_cast<size_t>(b)]) plan.farNodesHost.push_back(b);
  }
  std::vector<int> levelNodes;
  plan.levelOff.assign(1, 0);
  for (int lv = 0; lv <= maxDepth; ++lv) {
    for (int b = 0; b < t.nodes; ++b)
      if (depth[static_cast<size_t>(b)] == lv && t.left[static_cast<size_t>(b)] >= 0) levelNodes.push_back(b);
    plan.levelOff.push_back(static_cast<int>(levelNodes.size()));
  }
  uploadVec(plan.dLevelNodes, levelNodes, st);
  uploadVec(plan.dFarNodes, plan.farNodesHost, st);
  // top levels by composite shifts from the depth-m2mTop frontier (moments.cu
  // m2m_pairs): one launch instead of one latency-bound launch per level
  // (deterministic mode: 0 -- the composite shifts add into a node from
  // several frontier nodes with atomics; the per-level M2M writes once)
  const int topDepth = plan.options.deterministic ? 0 : 8;  // B200 sweep 0/6/8/10 (cfg2 S2M 0.294/0.245/0.233/0.248 ms)
  plan.m2mTop = std::min(topDepth, maxDepth);
  std::vector<int> topPairs;
  for (int b = 0; b < t.nodes; ++b) {
    if (t.left[static_cast<size_t>(b)] < 0 || depth[static_cast<size_t>(b)] >= plan.m2mTop) continue;
    std::vector<int> stack{t.left[static_cast<size_t>(b)], t.right[static_cast<size_t>(b)]};
    while (!stack.empty()) {
      const int f = stack.back();
      stack.pop_back();
      if (depth[static_cast<size_t>(f)] >= plan.m2mTop || t.left[static_cast<size_t>(f)] < 0) {
        topPairs.push_back(b);
        topPairs.push_back(f);
      } else {
        stack.push_back(t.left[static_cast<size_t>(f)]);
        stack.push_back(t.right[static_cast<size_t>(f)]);
      }
    }
  }
  plan.topPairs = static_cast<int>(topPairs.size() / 2);
  uploadVec(plan.dTopPairs, topPairs, st);
  plan.useMoments = true;
  buildP2MTiles(plan);
}

// Leaf tiles of the monomial S2M over the owned sources (deterministic mode:
// one tile per leaf, so each leaf's moments have a single writer).
void buildP2MTiles(DevicePlan& plan) {
  const DeviceTree& t = *plan.tree;
  const long long tileLen = plan.options.deterministic ? (1ll << 30) : 4096;
  plan.p2mTilesHost.clear();
  for (int b = 0; b < t.nodes; ++b) {
    if (t.left[static_cast<size_t>(b)] >= 0) continue;
    const long long s0 = std::max<long long>(t.begin[static_cast<size_t>(b)], plan.shardLo);
    const long long s1 = std::min<long long>(t.end[static_cast<size_t>(b)], plan.shardHi);
    for (long long s = s0; s < s1; s += tileLen)
      plan.p2mTilesHost.push_back(FktbTile{b, static_cast<int>(std::min<long long>(tileLen, s1 - s)), s});
  }
  uploadVec(plan.dP2mTiles, plan.p2mTilesHost, plan.stream);
}

}  // namespace

int maxRhsPerPass(const DevicePlan& plan) {
  static const long long limit = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      v = 227 * 1024;
    return static_cast<long long>(v) - 16 * 1024;  // headroom for the kernels' static shared tables
  }();
  auto fits = [&](int r) {
    if (plan.useMoments) {
      const long long C = plan.monoCount, E = plan.shiftEntries;
      if ((E + 2 * C * (1 + r)) * 8 + (C + 1 + 2 * E) * 4 > limit) return false;  // m2m_kernel
      if ((E + C * (1 + r)) * 8 + (C + 1 + 2 * E) * 4 > limit) return false;      // m2m_pairs
    }
    return static_cast<long long>((plan.P + 1) & ~1) * r * 8 <= limit;  // M2T moments of one node
  };
  int r = 1;
  while (r < kMaxRhsPerPass && fits(r + 1)) ++r;
  if (r >= 16) return r / 16 * 16;  // keep the 16-RHS specialisations
  if (r >= 8) return r / 8 * 8;
  return r;
}

void orderAfterPrevious(DevicePlan& plan, cudaStream_t st) {
  if (plan.doneRecorded) FKTB_CUDA(cudaStreamWaitEvent(st, plan.evDone, 0));
}

void markDone(DevicePlan& plan, cudaStream_t st) {
  FKTB_CUDA(cudaEventRecord(plan.evDone, st));
  plan.doneRecorded = true;
}

void ensureWorkspace(DevicePlan& plan, int nrhs) {
  nrhs = std::min(nrhs, maxRhsPerPass(plan));
  if (nrhs <= plan.nrhsCap) return;
  // the buffers may still be in use by a previous multiply on another stream
  if (plan.doneRecorded) FKTB_CUDA(cudaEventSynchronize(plan.evDone));
  clearGraphs(plan);
  if (plan.useMoments) plan.dMono.resize(static_cast<size_t>(plan.tree->nodes) * plan.monoCount * nrhs);
  const size_t n = static_cast<size_t>(plan.n);
  plan.dYp.resize(n * nrhs);
  plan.dZp.resize(n * nrhs);
  if (plan.nearRowsBuilt) {
    // per-pass source-major weights of R <= min(nrhs, 16) columns (a power
    // of two; one column rides in the source rows)
    int r = 1;
    while (r * 2 <= std::min(nrhs, 16)) r *= 2;
    if (r > 1) plan.dNearW.resize(n * r);
    if (plan.dNearCounter.size() == 0) plan.dNearCounter.resize(2);
  }
  plan.dMoments.resize(std::max<size_t>(1, static_cast<size_t>(plan.tree->nodes) * momentStrideMax(plan) * nrhs));
  if (plan.options.deterministic) {
    // + one all-zero row: the padding slots of the per-target sums read it
    plan.dPart.resize(static_cast<size_t>(plan.slotsTotal + 1) * nrhs);
    FKTB_CUDA(cudaMemset(plan.dPart.get() + static_cast<size_t>(plan.slotsTotal) * nrhs, 0, nrhs * sizeof(double)));
    plan.dZf.resize(n * nrhs);
    if (!plan.useMoments) plan.dTilePart.resize(std::max<size_t>(1, detTilePartSize(plan, nrhs)));
  }
  plan.nrhsCap = nrhs;
}

void rebuildTiles(DevicePlan& plan) {
  FKTB_CUDA(cudaStreamSynchronize(plan.stream));  // tiles may be in use by queued work
  FKTB_CUDA(cudaStreamSynchronize(plan.side));
  clearGraphs(plan);
  buildTiles(plan);
  if (plan.useMoments) buildP2MTiles(plan);
  if (plan.options.deterministic) {
    buildDetTileRanges(plan);
    if (!plan.useMoments && plan.nrhsCap > 0) plan.dTilePart.resize(std::max<size_t>(1, detTilePartSize(plan, plan.nrhsCap)));
  }
  FKTB_CUDA(cudaStreamSynchronize(plan.stream));
}

std::unique_ptr<DevicePlan> createPlan(int n, int d, const double* hostX, const KernelSpec& kernel,
                                       const PlanOptions& options) {
  const auto t0 = std::chrono::steady_clock::now();
  auto plan = std::make_unique<DevicePlan>();
  plan->n = n;
  plan->d = d;
  plan->shardHi = static_cast<uint32_t>(n);
  plan->cuts = {0u, static_cast<uint32_t>(n)};
  plan->options = options;
  plan->kernel = kernel;
  if (options.barnesHut) plan->options.p = 0;  // transform.cpp:44
  // Validation order follows the reference constructor (transform.cpp:39-80).
  if (options.leafCapacity < 1) throw std::invalid_argument("leaf capacity must be >= 1");
  if (n < 1) throw std::invalid_argument("point cloud must be nonempty");
  if (plan->options.p < 0) throw std::invalid_argument("plan requires p >= 0");
  if (!(options.theta > 0.0 && options.theta < 1.0)) throw std::invalid_argument("theta must be in (0, 1)");
  // Barnes-Hut plans return before the expansion tables (transform.cpp:48-59):
  // no coefficient table, harmonic basis (so any d >= 1) or compression.
  const bool bh = options.barnesHut;
  if (!bh && d < 2) throw std::invalid_argument("HarmonicBasis requires d >= 2");
  const CoefTable* table = bh ? nullptr : &coefTable(d, plan->options.p);  // OrderTooLarge for p > 20
  bool compress = false;
  if (bh) {
  } else if (options.compression == 0)
    compress = kernel.recurrence.has_value();
  else if (options.compression == 1) {
    if (!kernel.recurrence) throw NotRecurrenceKernelError(kernel.name);
    compress = true;
  }
  if (!bh && !specialised(d, options.p) && (d - 2) * (options.p + 1) * (options.p + 2) / 2 > genericGMax())
    throw std::invalid_argument("unsupported on the GPU path: (d, p) too large for the runtime far-field kernels");

  FKTB_CUDA(cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking));
  FKTB_CUDA(cudaStreamCreateWithFlags(&plan->side, cudaStreamNonBlocking));
  FKTB_CUDA(cudaEventCreateWithFlags(&plan->evGather, cudaEventDisableTiming));
  FKTB_CUDA(cudaEventCreateWithFlags(&plan->evFar, cudaEventDisableTiming));
  FKTB_CUDA(cudaEventCreateWithFlags(&plan->evDone, cudaEventDisableTiming));
  // phase timings (fkt_plan_phases): each phase ends with its stream drained
  auto tPrev = std::chrono::steady_clock::now();
  auto phase = [&](int i) {
    FKTB_CUDA(cudaStreamSynchronize(plan->stream));
    const auto now = std::chrono::steady_clock::now();
    plan->phaseSeconds[i] += std::chrono::duration<double>(now - tPrev).count();
    tPrev = now;
  };
  plan->tree = std::make_unique<DeviceTree>();
  // one H2D of the coordinates (row-major, kept for the dense paths); the
  // tree is built from the device copy
  plan->dX.resize(static_cast<size_t>(n) * d);
  FKTB_CUDA(cudaMemcpyAsync(plan->dX.get(), hostX, plan->dX.bytes(), cudaMemcpyHostToDevice, plan->stream));
  buildTreeGpu(*plan->tree, hostX, n, d, options.leafCapacity, plan->stream, plan->dX.get());
  phase(kPhaseTree);
  computeSetsGpu(*plan->tree, options.theta);
  phase(kPhaseSets);

  plan->compressed = compress;
  if (bh) {
    // one coefficient per node: the source total (coefficientCount() == 1, transform.cpp:95)
    auto fp = std::make_unique<FktbFarParams>();
    std::memset(fp.get(), 0, sizeof(FktbFarParams));
    fp->d = d;
    fp->P = fp->Pref = fp->H = 1;
    plan->far = std::move(fp);
    plan->P = plan->H = 1;
  } else {
    plan->harmonics = std::make_unique<HarmonicStructure>(d, plan->options.p);
    if (compress) plan->factors = radialCompression(kernel, *table, plan->options.p);
    buildFarParams(*plan);
  }
  phase(kPhaseTables);
  buildTiles(*plan);
  phase(kPhaseTiles);
  plan->phaseSeconds[kPhaseTiles] -= plan->phaseSeconds[kPhaseNearRows];  // buildTiles timed the rows itself
  if (bh) {
    buildBarnesHut(*plan);
  } else {
    // test hook: "direct" keeps the per-node direct S2M (tests/test_gpu_moments.py
    // checks the monomial-moment path against it)
    const char* s2m = std::getenv("FKTB_S2M");
    if (momentsSupported(d, options.p) && !(s2m && std::string(s2m) == "direct")) buildMomentPlan(*plan);
  }
  phase(kPhaseMoments);
  if (options.deterministic) {
    buildDeterministic(*plan);
    buildDetTileRanges(*plan);
  }
  ensureWorkspace(*plan, 1);
  (void)expTableDevice();  // lazy device tables: initialise outside any graph capture
  (void)expTableDevice(kNearExpBits, true);
  if (const char* g = std::getenv("FKTB_GRAPHS")) plan->useGraphs = std::atoi(g) != 0;
  plan->tree->scratch = DeviceTree::Scratch{};  // lean plans: rebuildPlan re-sizes it on demand
  phase(kPhaseOther);
  plan->planSeconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return plan;
}

// Moving points (t-SNE-style iterations): the same plan on new coordinates of
// the same n points. Tree, sets, tiles, geometry rows, the moment plan and
// the shard are rebuilt on the GPU; the kernel tables (T-bar, harmonics,
// compression) and every buffer are kept, so no cudaMalloc runs once the
// first rebuild has sized the build scratch. Equals a fresh plan on x.
void rebuildPlan(DevicePlan& plan, const double* x, bool onDevice) {
  const auto t0 = std::chrono::steady_clock::now();
  FKTB_CUDA(cudaStreamSynchronize(plan.stream));
  FKTB_CUDA(cudaStreamSynchronize(plan.side));
  if (plan.doneRecorded) FKTB_CUDA(cudaEventSynchronize(plan.evDone));
  clearGraphs(plan);
  for (double& s : plan.phaseSeconds) s = 0.0;
  auto tPrev = std::chrono::steady_clock::now();
  auto phase = [&](int i) {
    FKTB_CUDA(cudaStreamSynchronize(plan.stream));
    const auto now = std::chrono::steady_clock::now();
    plan.phaseSeconds[i] += std::chrono::duration<double>(now - tPrev).count();
    tPrev = now;
  };
  DeviceTree& t = *plan.tree;
  FKTB_CUDA(cudaMemcpyAsync(plan.dX.get(), x, plan.dX.bytes(), onDevice ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            plan.stream));
  buildTreeGpu(t, nullptr, plan.n, plan.d, plan.options.leafCapacity, plan.stream, plan.dX.get());
  phase(kPhaseTree);
  computeSetsGpu(t, plan.options.theta);
  phase(kPhaseSets);
  plan.shardLo = 0;
  plan.shardHi = static_cast<uint32_t>(plan.n);
  plan.cuts = {0u, static_cast<uint32_t>(plan.n)};
  plan.farSub.clear();
  plan.nearSub.clear();
  plan.nearRowsBuilt = false;
  buildTiles(plan);
  phase(kPhaseTiles);
  plan.phaseSeconds[kPhaseTiles] -= plan.phaseSeconds[kPhaseNearRows];
  if (plan.options.barnesHut)
    buildBarnesHut(plan);
  else if (plan.useMoments)
    buildMomentPlan(plan);
  phase(kPhaseMoments);
  if (plan.options.deterministic) {
    buildDeterministic(plan);
    buildDetTileRanges(plan);
  }
  if (plan.shards > 1) setShard(plan, plan.shard, plan.shards);
  // workspaces sized by the new tree (deterministic partials, S2M tile
  // partials) at the pass width already in use
  const int cap = std::max(1, plan.nrhsCap);
  plan.nrhsCap = 0;
  ensureWorkspace(plan, cap);
  phase(kPhaseOther);
  plan.planSeconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void destroyPlan(DevicePlan* plan) {
  if (!plan) return;
  if (plan->stream) cudaStreamSynchronize(plan->stream);
  if (plan->side) cudaStreamSynchronize(plan->side);
  cudaStream_t st = plan->stream, side = plan->side;
  cudaEvent_t e0 = plan->evGather, e1 = plan->evFar, e2 = plan->evDone;
  if (plan->doneRecorded) cudaEventSynchronize(e2);
  releaseHostIo(*plan);
  clearGraphs(*plan);
  delete plan;
  if (st) cudaStreamDestroy(st);
  if (side) cudaStreamDestroy(side);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (e2) cudaEventDestroy(e2);
}

long long kernelLaunches(const DevicePlan& plan, int nrhs) {
  auto chunks = [&](int perRhsDoubles) {
    const size_t perRhs = static_cast<size_t>(128) * perRhsDoubles * sizeof(double);
    const int chunk = std::max(1, static_cast<int>((200 * 1024) / perRhs));
    return (nrhs + chunk - 1) / chunk;
  };
  long long k = 2;  // gather_y, scatter_z
  if (plan.useMoments) {
    if (!plan.p2mTilesHost.empty()) k += p2mLaunches(plan.d, plan.options.p, plan.monoCount, nrhs);
    for (size_t l = static_cast<size_t>(plan.m2mTop); l + 1 < plan.levelOff.size(); ++l)  // m2m, wide levels
      k += plan.levelOff[l + 1] > plan.levelOff[l];
    k += plan.topPairs > 0;  // m2m_pairs, the narrow top
    k += !plan.farNodesHost.empty();  // to_coef (one GEMM over all nodes)
  } else if (!plan.s2mTilesHost.empty()) {
    k += plan.options.barnesHut ? 1 : chunks(plan.P);
  }
  if (!plan.nearTilesHost.empty()) {
    // FP32 mode: one launch (near32.cu); FP64: per RHS pass, one launch per
    // pair form present (+ the weight kernel when the pass needs it, near.cu)
    k += plan.options.nearPrecision == 32 ? 1 : nearLaunches(plan, nrhs);
  }
  k += !plan.farTilesHost.empty();
  if (plan.options.deterministic) {
    k += 2;  // the far and near sums of the partials
    if (!plan.useMoments && plan.detTileNodes > 0)  // per-tile S2M partials, per RHS chunk
      k += plan.options.barnesHut ? 1 : (nrhs + s2mRhsChunk(plan.P) - 1) / s2mRhsChunk(plan.P);
  }
  return k;
}

void launchS2MAny(const DevicePlan& plan, const double* yp, double* moments, int nrhs, cudaStream_t st) {
  if (plan.options.barnesHut)
    launchBHSums(plan, yp, moments, nrhs, st);
  else if (plan.useMoments)
    launchS2MMoments(plan, yp, moments, nrhs, st);
  else
    launchS2M(plan, yp, moments, nrhs, st);
}

void launchNearAny(const DevicePlan& plan, const double* yp, double* zp, int nrhs, cudaStream_t st) {
  if (plan.options.nearPrecision == 32 && launchNear32(plan, yp, zp, nrhs, st)) return;
  launchNear(plan, yp, zp, nrhs, st);
}

namespace {
void enqueuePass(DevicePlan& plan, const double* y, double* z, int nrhs, cudaStream_t st) {
  const size_t n = static_cast<size_t>(plan.n);
  // stream st: gather -> zero z -> near ------------------------> scatter
  // side:                        \-> zero moments -> S2M -> M2T -/
  launchGatherY(plan, y, plan.dYp.get(), nrhs, st);
  FKTB_CUDA(cudaMemsetAsync(plan.dZp.get(), 0, n * nrhs * sizeof(double), st));
  FKTB_CUDA(cudaEventRecord(plan.evGather, st));
  FKTB_CUDA(cudaStreamWaitEvent(plan.side, plan.evGather, 0));
  FKTB_CUDA(cudaMemsetAsync(plan.dMoments.get(), 0,
                            static_cast<size_t>(plan.tree->nodes) * momentStride(plan, nrhs) * nrhs * sizeof(double),
                            plan.side));
  launchS2MAny(plan, plan.dYp.get(), plan.dMoments.get(), nrhs, plan.side);
  launchNearAny(plan, plan.dYp.get(), plan.dZp.get(), nrhs, st);
  launchM2T(plan, plan.dMoments.get(), plan.dZp.get(), nrhs, plan.side);
  if (plan.options.deterministic) launchDetReduce(plan, nullptr, nrhs, true, plan.side);  // z_far, behind the near field
  FKTB_CUDA(cudaEventRecord(plan.evFar, plan.side));
  FKTB_CUDA(cudaStreamWaitEvent(st, plan.evFar, 0));
  if (plan.options.deterministic) launchDetReduce(plan, plan.dZp.get(), nrhs, false, st);
  launchScatterZ(plan, plan.dZp.get(), z, nrhs, st);
}

// Right-hand sides in passes of at most maxRhsPerPass columns (the per-node
// moment rows of M2M / M2T live in shared memory).
void enqueueMultiply(DevicePlan& plan, const double* y, double* z, int nrhs, cudaStream_t st) {
  const int chunk = maxRhsPerPass(plan);
  const size_t n = static_cast<size_t>(plan.n);
  for (int r0 = 0; r0 < nrhs; r0 += chunk)
    enqueuePass(plan, y + r0 * n, z + r0 * n, std::min(chunk, nrhs - r0), st);
}
}  // namespace

void multiplyDevice(DevicePlan& plan, const double* y, double* z, int nrhs, cudaStream_t st) {
  ensureWorkspace(plan, nrhs);
  // The legacy default stream cannot be captured: run eagerly there.
  orderAfterPrevious(plan, st);  // one workspace per plan: calls on different streams run in order
  if (!plan.useGraphs || st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread) {
    enqueueMultiply(plan, y, z, nrhs, st);
    markDone(plan, st);
    return;
  }
  const auto key = std::make_tuple(static_cast<const void*>(y), static_cast<const void*>(z), nrhs, st);
  auto it = plan.graphs.find(key);
  if (it == plan.graphs.end()) {
    cudaGraph_t graph = nullptr;
    FKTB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      enqueueMultiply(plan, y, z, nrhs, st);
    } catch (...) {
      cudaStreamEndCapture(st, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    FKTB_CUDA(cudaStreamEndCapture(st, &graph));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    FKTB_CUDA(e);
    if (static_cast<int>(plan.graphs.size()) >= DevicePlan::kMaxGraphs) {
      auto victim = plan.graphs.begin();
      for (auto g = plan.graphs.begin(); g != plan.graphs.end(); ++g)
        if (g->second.second < victim->second.second) victim = g;
      // the victim may still be in flight on a stream the caller owns (or
      // has destroyed): drain the device before releasing it (rare path)
      FKTB_CUDA(cudaDeviceSynchronize());
      cudaGraphExecDestroy(victim->second.first);
      plan.graphs.erase(victim);
    }
    it = plan.graphs.emplace(key, std::make_pair(exec, 0ull)).first;
  }
  it->second.second = ++plan.graphClock;
  FKTB_CUDA(cudaGraphLaunch(it->second.first, st));
  markDone(plan, st);
}

}  // namespace fktb
