// Host-buffer multiply (fkt_plan_multiply; the drop-in FktPlan::multiply(span)
// of proj/include/fkt/transform.hpp:47 lands here with pageable std::vector
// storage): z = K y with y, z in host memory, H2D and D2H inside the call.
//
//  * Pinned buffers (cudaHostAlloc / registered) are copied by DMA directly.
//  * Large pageable buffers (>= 64 MB; below that the driver's own staging
//    is as fast) go through plan-owned pinned bounce buffers in 8 MB chunks: host threads copy chunk k while the copy engine moves chunk
//    k - 1 (upload), and the reverse on the way down, so the slower of host
//    memcpy and PCIe sets the pace instead of their sum.
//  * Many right-hand sides are split into two groups: group 1 uploads while
//    group 0 computes, and group 0 downloads while group 1 computes.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "plan.hpp"

namespace fktb {
namespace {

constexpr size_t kChunk = size_t(8) << 20;  // bytes per staged chunk

bool isPinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int hostThreads() {
  static const int t = [] {
    const unsigned h = std::thread::hardware_concurrency();
    return static_cast<int>(std::max(1u, std::min(8u, h / 2)));
  }();
  return t;
}

struct Span {
  size_t off, len;  // bytes
};

std::vector<Span> chunksOf(size_t off, size_t len) {
  std::vector<Span> c;
  for (size_t o = 0; o < len; o += kChunk) c.push_back({off + o, std::min(kChunk, len - o)});
  return c;
}

// Parallel copy of a chunk list: worker w copies its 1/T slice of every chunk
// in order (after gate(k)) and bumps the chunk's counter; wait(k) returns once
// all T slices of chunk k are done.
class ChunkCopier {
 public:
  ChunkCopier(char* dst, const char* src, std::vector<Span> chunks, int threads)
      : dst_(dst), src_(src), c_(std::move(chunks)), T_(threads), done_(c_.size()) {
    for (auto& d : done_) d.store(0);
  }
  template <class Gate>
  void start(Gate gate) {
    for (int w = 0; w < T_; ++w)
      workers_.emplace_back([this, w, gate] {
        for (size_t k = 0; k < c_.size(); ++k) {
          gate(k);
          const size_t per = (c_[k].len + T_ - 1) / T_;
          const size_t o = std::min(c_[k].len, per * w), e = std::min(c_[k].len, o + per);
          if (e > o) std::memcpy(dst_ + c_[k].off + o, src_ + c_[k].off + o, e - o);
          done_[k].fetch_add(1, std::memory_order_release);
        }
      });
  }
  void wait(size_t k) const {
    while (done_[k].load(std::memory_order_acquire) < T_) std::this_thread::yield();
  }
  void join() {
    for (auto& t : workers_) t.join();
    workers_.clear();
  }
  ~ChunkCopier() { join(); }

 private:
  char* dst_;
  const char* src_;
  std::vector<Span> c_;
  int T_;
  std::vector<std::atomic<int>> done_;
  std::vector<std::thread> workers_;
};

void ensureHostIo(DevicePlan& p, size_t doubles, bool bounce) {
  if (!p.h2d) {
    FKTB_CUDA(cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking));
    FKTB_CUDA(cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking));
    for (auto& e : p.evIo) FKTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (p.dYio.size() < doubles) {
    if (p.doneRecorded) FKTB_CUDA(cudaEventSynchronize(p.evDone));
    p.dYio.resize(doubles);
    p.dZio.resize(doubles);
  }
  if (bounce && p.bounceBytes < doubles * sizeof(double)) {
    if (p.bounceIn) cudaFreeHost(p.bounceIn);
    if (p.bounceOut) cudaFreeHost(p.bounceOut);
    p.bounceIn = p.bounceOut = nullptr;
    p.bounceBytes = 0;
    FKTB_CUDA(cudaHostAlloc(&p.bounceIn, doubles * sizeof(double), cudaHostAllocDefault));
    FKTB_CUDA(cudaHostAlloc(&p.bounceOut, doubles * sizeof(double), cudaHostAllocDefault));
    p.bounceBytes = doubles * sizeof(double);
  }
}

}  // namespace

void multiplyHost(DevicePlan& p, const double* y, double* z, int nrhs) {
  const size_t n = static_cast<size_t>(p.n), total = n * nrhs, bytes = total * sizeof(double);
  // below 64 MB the driver's own pageable staging is as fast (B200 box,
  // cfg2's 8 MB: 14.9 ms e2e driver-staged vs 17.2 ms through the bounce):
  // those take the plain cudaMemcpyAsync path like pinned buffers
  const bool big = bytes >= (size_t(64) << 20);
  const bool pinY = !big || isPinned(y), pinZ = !big || isPinned(z);
  ensureHostIo(p, total, !pinY || !pinZ);
  // two RHS groups (a multiple of 8 columns first) when the transfers are
  // large enough to be worth hiding behind the other group's compute
  int split = nrhs;
  if (nrhs >= 8 && bytes >= (size_t(64) << 20)) split = std::min(nrhs - 1, std::max(8, (nrhs / 2 + 7) / 8 * 8));
  const int r0[3] = {0, split, nrhs};
  const int groups = split < nrhs ? 2 : 1;
  char* dY = reinterpret_cast<char*>(p.dYio.get());
  char* dZ = reinterpret_cast<char*>(p.dZio.get());
  char* bIn = static_cast<char*>(p.bounceIn);
  char* bOut = static_cast<char*>(p.bounceOut);
  std::vector<Span> outChunks;
  std::vector<cudaEvent_t> outEv;
  for (int g = 0; g < groups; ++g) {
    const size_t off = static_cast<size_t>(r0[g]) * n * sizeof(double);
    const size_t gb = static_cast<size_t>(r0[g + 1] - r0[g]) * n * sizeof(double);
    // upload group g (the host copies while the GPU computes group g - 1)
    if (pinY) {
      FKTB_CUDA(cudaMemcpyAsync(dY + off, reinterpret_cast<const char*>(y) + off, gb, cudaMemcpyHostToDevice, p.h2d));
    } else {
      const auto ch = chunksOf(off, gb);
      ChunkCopier cp(bIn, reinterpret_cast<const char*>(y), ch, hostThreads());
      cp.start([](size_t) {});
      for (size_t k = 0; k < ch.size(); ++k) {
        cp.wait(k);
        FKTB_CUDA(cudaMemcpyAsync(dY + ch[k].off, bIn + ch[k].off, ch[k].len, cudaMemcpyHostToDevice, p.h2d));
      }
    }
    FKTB_CUDA(cudaEventRecord(p.evIo[g], p.h2d));
    FKTB_CUDA(cudaStreamWaitEvent(p.stream, p.evIo[g], 0));
    multiplyDevice(p, reinterpret_cast<const double*>(dY + off), reinterpret_cast<double*>(dZ + off),
                   r0[g + 1] - r0[g], p.stream);
    FKTB_CUDA(cudaEventRecord(p.evIo[2 + g], p.stream));
    // download group g as soon as it is done (overlaps group g + 1's compute)
    FKTB_CUDA(cudaStreamWaitEvent(p.d2h, p.evIo[2 + g], 0));
    if (pinZ) {
      FKTB_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(z) + off, dZ + off, gb, cudaMemcpyDeviceToHost, p.d2h));
    } else {
      for (const Span& c : chunksOf(off, gb)) {
        cudaEvent_t e;
        FKTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync));
        FKTB_CUDA(cudaMemcpyAsync(bOut + c.off, dZ + c.off, c.len, cudaMemcpyDeviceToHost, p.d2h));
        FKTB_CUDA(cudaEventRecord(e, p.d2h));
        outChunks.push_back(c);
        outEv.push_back(e);
      }
    }
  }
  if (!pinZ) {
    // host threads copy each chunk out of the bounce once its DMA landed
    ChunkCopier cp(reinterpret_cast<char*>(z), bOut, outChunks, hostThreads());
    cp.start([&outEv](size_t k) { cudaEventSynchronize(outEv[k]); });
    cp.join();
    for (auto e : outEv) cudaEventDestroy(e);
  }
  FKTB_CUDA(cudaStreamSynchronize(p.d2h));
  FKTB_CUDA(cudaStreamSynchronize(p.stream));
}

void releaseHostIo(DevicePlan& p) {
  if (p.h2d) cudaStreamSynchronize(p.h2d);
  if (p.d2h) cudaStreamSynchronize(p.d2h);
  if (p.bounceIn) cudaFreeHost(p.bounceIn);
  if (p.bounceOut) cudaFreeHost(p.bounceOut);
  p.bounceIn = p.bounceOut = nullptr;
  p.bounceBytes = 0;
  if (p.h2d) {
    cudaStreamDestroy(p.h2d);
    cudaStreamDestroy(p.d2h);
    for (auto& e : p.evIo) cudaEventDestroy(e);
  }
  p.h2d = p.d2h = nullptr;
}

}  // namespace fktb
