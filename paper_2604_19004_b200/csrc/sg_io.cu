// sg_io.cu — device -> host download of the result (C is 116 GB at R-MAT-20).
//
// The copy engine fills a ring of pinned staging buffers (allocated once per
// process) on a dedicated stream while native worker threads move finished
// buffers into the caller's pageable destination.  The workers also take the
// destination's first-touch page faults in parallel, which is what limits a
// single-threaded copy (~7 GB/s on the GPU box versus ~48 GB/s for the link).
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "sg_internal.cuh"

namespace sg {
namespace {

constexpr size_t STAGE_BYTES = (size_t)64 << 20;
constexpr int MAX_STAGES = 32;

struct StagePool {
  std::mutex mu;
  std::vector<void*> bufs;
  int device = -1;
};

StagePool& pool() {
  static StagePool p;
  return p;
}

}  // namespace
}  // namespace sg

using namespace sg;

namespace {

int download_staged(void* host_dst, const void* dev_src, size_t bytes, int threads, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int T = threads > 0 ? std::min(threads, MAX_STAGES / 2) : 8;
  const int K = std::min(MAX_STAGES, 2 * T);
  StagePool& P = pool();
  std::lock_guard<std::mutex> hold(P.mu);  // one download at a time per process
  if (P.device != dev) {
    for (void* b : P.bufs) cudaFreeHost(b);
    P.bufs.clear();
    P.device = dev;
  }
  while ((int)P.bufs.size() < K) {
    void* b = nullptr;
    if (cudaHostAlloc(&b, STAGE_BYTES, cudaHostAllocDefault) != cudaSuccess) return check_cuda("sg_download alloc", 0);
    P.bufs.push_back(b);
  }
  // the copy stream waits for the caller's stream (the producer of dev_src)
  cudaStream_t cs;
  cudaEvent_t ready;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return check_cuda("sg_download stream", 0);
  cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
  cudaEventRecord(ready, s);
  cudaStreamWaitEvent(cs, ready, 0);
  std::vector<cudaEvent_t> ev(K);
  for (int i = 0; i < K; ++i) cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming | cudaEventBlockingSync);

  const int64_t nchunks = (int64_t)((bytes + STAGE_BYTES - 1) / STAGE_BYTES);
  std::mutex mu;
  std::condition_variable cv;
  int64_t issued = 0;                      // chunks [0, issued) have copies enqueued
  std::vector<int64_t> drained(K, -1);     // last chunk drained from each buffer
  bool failed = false;
  auto worker = [&](int j) {
    for (int64_t k = j; k < nchunks; k += T) {
      const int buf = (int)(k % K);
      {
        std::unique_lock<std::mutex> l(mu);
        cv.wait(l, [&] { return issued > k || failed; });
        if (failed) return;
      }
      if (cudaEventSynchronize(ev[buf]) != cudaSuccess) {
        std::lock_guard<std::mutex> l(mu);
        failed = true;
        cv.notify_all();
        return;
      }
      const size_t off = (size_t)k * STAGE_BYTES;
      const size_t len = std::min(STAGE_BYTES, bytes - off);
      std::memcpy(static_cast<char*>(host_dst) + off, P.bufs[buf], len);
      {
        std::lock_guard<std::mutex> l(mu);
        drained[buf] = k;
      }
      cv.notify_all();
    }
  };
  std::vector<std::thread> pool_threads;
  pool_threads.reserve(T);
  for (int j = 0; j < T; ++j) pool_threads.emplace_back(worker, j);
  int rc = SG_OK;
  for (int64_t k = 0; k < nchunks; ++k) {
    const int buf = (int)(k % K);
    {
      std::unique_lock<std::mutex> l(mu);
      cv.wait(l, [&] { return k < K || drained[buf] >= k - K || failed; });
      if (failed) break;
    }
    const size_t off = (size_t)k * STAGE_BYTES;
    const size_t len = std::min(STAGE_BYTES, bytes - off);
    if (cudaMemcpyAsync(P.bufs[buf], static_cast<const char*>(dev_src) + off, len, cudaMemcpyDeviceToHost, cs) !=
            cudaSuccess ||
        cudaEventRecord(ev[buf], cs) != cudaSuccess) {
      std::lock_guard<std::mutex> l(mu);
      failed = true;
      cv.notify_all();
      break;
    }
    {
      std::lock_guard<std::mutex> l(mu);
      issued = k + 1;
    }
    cv.notify_all();
  }
  for (auto& th : pool_threads) th.join();
  if (failed) rc = check_cuda("sg_download copy", 0);
  if (rc == SG_OK && failed) {
    set_error("sg_download: copy failed");
    rc = SG_ERR_CUDA;
  }
  cudaStreamSynchronize(cs);
  for (int i = 0; i < K; ++i) cudaEventDestroy(ev[i]);
  cudaEventDestroy(ready);
  cudaStreamDestroy(cs);
  return rc;
}

// Direct path: worker threads first-touch and page-lock (cudaHostRegister)
// 256 MB page-aligned chunks of the destination, the copy engine DMAs each
// registered chunk straight from the device, then the chunks are released.
// Host memory sees the kernel's page zeroing and the DMA write only (the
// staged path adds a read and a write of every byte by the CPU).
int download_registered(void* host_dst, const void* dev_src, size_t bytes, int threads, cudaStream_t s) {
  constexpr size_t PG = 4096, CH = (size_t)256 << 20;
  char* dst = static_cast<char*>(host_dst);
  const char* src = static_cast<const char*>(dev_src);
  const uintptr_t a0 = (reinterpret_cast<uintptr_t>(dst) + PG - 1) & ~(uintptr_t)(PG - 1);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(dst) + bytes) & ~(uintptr_t)(PG - 1);
  if (a1 <= a0 + PG) return download_staged(host_dst, dev_src, bytes, threads, s);
  const size_t head = a0 - reinterpret_cast<uintptr_t>(dst), body = a1 - a0, tail = bytes - head - body;
  const int64_t nch = (int64_t)((body + CH - 1) / CH);
  const int T = threads > 0 ? std::min(threads, 32) : 8;
  cudaStream_t cs;
  cudaEvent_t ready;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return check_cuda("sg_download stream", 0);
  cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
  cudaEventRecord(ready, s);
  cudaStreamWaitEvent(cs, ready, 0);
  std::mutex mu;
  std::condition_variable cv;
  std::vector<int> state(nch, 0);  // 0 pending, 1 registered, -1 failed
  const char* ff = getenv("SG_TEST_REGISTER_FAIL");
  const int64_t fail_from = ff ? atoll(ff) : -1;
  int64_t next = 0;
  auto reg = [&]() {
    for (;;) {
      int64_t i;
      {
        std::lock_guard<std::mutex> l(mu);
        i = next++;
      }
      if (i >= nch) return;
      char* p = reinterpret_cast<char*>(a0) + (size_t)i * CH;
      const size_t len = std::min(CH, body - (size_t)i * CH);
      for (size_t o = 0; o < len; o += PG) p[o] = 0;  // first touch in parallel
      // SG_TEST_REGISTER_FAIL=k: test hook, chunks >= k fail to page-lock
      const bool ok = (fail_from < 0 || i < fail_from) && cudaHostRegister(p, len, cudaHostRegisterDefault) == cudaSuccess;
      {
        std::lock_guard<std::mutex> l(mu);
        state[i] = ok ? 1 : -1;
      }
      cv.notify_all();
    }
  };
  std::vector<std::thread> th;
  for (int j = 0; j < T; ++j) th.emplace_back(reg);
  bool failed = false;
  int64_t unreg = -1;  // first chunk whose page lock failed: staged path from there
  for (int64_t i = 0; i < nch; ++i) {
    {
      std::unique_lock<std::mutex> l(mu);
      cv.wait(l, [&] { return state[i] != 0; });
      if (state[i] < 0) unreg = i;
    }
    if (unreg >= 0) break;
    const size_t off = (size_t)i * CH, len = std::min(CH, body - off);
    if (cudaMemcpyAsync(reinterpret_cast<char*>(a0) + off, src + head + off, len, cudaMemcpyDeviceToHost, cs) !=
        cudaSuccess) {
      failed = true;
      break;
    }
  }
  for (auto& t : th) t.join();
  cudaStreamSynchronize(cs);
  int rc = failed ? SG_ERR_CUDA : check_cuda("sg_download copy", 0);
  if (failed) set_error("sg_download: host register / copy failed");
  // release the page locks in parallel
  {
    std::vector<std::thread> un;
    std::atomic<int64_t> k{0};
    for (int j = 0; j < T; ++j)
      un.emplace_back([&] {
        for (int64_t i = k++; i < nch; i = k++)
          if (state[i] == 1) cudaHostUnregister(reinterpret_cast<char*>(a0) + (size_t)i * CH);
      });
    for (auto& t : un) t.join();
  }
  cudaGetLastError();
  if (rc == SG_OK && unreg >= 0) {
    // page locking failed (memlock limit, IOMMU, memory pressure): the rest
    // of the body goes through the pinned staging ring instead of failing
    const size_t off = (size_t)unreg * CH;
    rc = download_staged(reinterpret_cast<char*>(a0) + off, src + head + off, body - off, threads, cs);
  }
  if (rc == SG_OK && head) {
    if (cudaMemcpyAsync(dst, src, head, cudaMemcpyDeviceToHost, cs) != cudaSuccess) rc = check_cuda("head", 0);
  }
  if (rc == SG_OK && tail) {
    if (cudaMemcpyAsync(dst + head + body, src + head + body, tail, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
      rc = check_cuda("tail", 0);
  }
  cudaStreamSynchronize(cs);
  cudaEventDestroy(ready);
  cudaStreamDestroy(cs);
  return rc;
}

// parallel first touch + page lock (or unlock) of [p, p + bytes) in
// PIN_CHUNK pieces measured from p (p page-aligned)
constexpr size_t PIN_CHUNK = (size_t)256 << 20;

int pin_chunks(void* p, size_t bytes, int threads, bool pin) {
  const int64_t nch = (int64_t)((bytes + PIN_CHUNK - 1) / PIN_CHUNK);
  const int T = threads > 0 ? std::min(threads, 32) : 8;
  std::atomic<int64_t> next{0};
  std::atomic<int> bad{0};
  std::vector<std::thread> th;
  for (int j = 0; j < T; ++j)
    th.emplace_back([&] {
      for (int64_t i = next++; i < nch; i = next++) {
        char* q = static_cast<char*>(p) + (size_t)i * PIN_CHUNK;
        const size_t len = std::min(PIN_CHUNK, bytes - (size_t)i * PIN_CHUNK);
        if (pin) {
          for (size_t o = 0; o < len; o += 4096) q[o] = 0;
          if (cudaHostRegister(q, len, cudaHostRegisterDefault) != cudaSuccess) bad = 1;
        } else {
          if (cudaHostUnregister(q) != cudaSuccess) bad = 1;
        }
      }
    });
  for (auto& t : th) t.join();
  if (bad) {
    cudaGetLastError();
    set_error(pin ? "sg_host_pin: cudaHostRegister failed" : "sg_host_unpin: cudaHostUnregister failed");
    return SG_ERR_CUDA;
  }
  return SG_OK;
}

// destination already pinned by sg_host_pin from host_dst: one DMA per chunk
int download_pinned(void* host_dst, const void* dev_src, size_t bytes, cudaStream_t s) {
  for (size_t off = 0; off < bytes; off += PIN_CHUNK) {
    const size_t len = std::min(PIN_CHUNK, bytes - off);
    if (cudaMemcpyAsync(static_cast<char*>(host_dst) + off, static_cast<const char*>(dev_src) + off, len,
                        cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return check_cuda("sg_download pinned", 0);
  }
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_download pinned sync", 0);
  return SG_OK;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace

extern "C" {

int sg_host_pin(void* p, size_t bytes, int threads) {
  if (!p || (reinterpret_cast<uintptr_t>(p) & 4095) || threads < 0) {
    set_error("sg_host_pin: p must be page-aligned");
    return SG_ERR_ARG;
  }
  return bytes ? pin_chunks(p, bytes, threads, true) : SG_OK;
}

int sg_host_unpin(void* p, size_t bytes, int threads) {
  if (!p || (reinterpret_cast<uintptr_t>(p) & 4095) || threads < 0) {
    set_error("sg_host_unpin: p must be page-aligned");
    return SG_ERR_ARG;
  }
  return bytes ? pin_chunks(p, bytes, threads, false) : SG_OK;
}

int sg_download(void* host_dst, const void* dev_src, size_t bytes, int threads, void* stream) {
  if ((bytes && (!host_dst || !dev_src)) || threads < 0) {
    set_error("sg_download: bad arguments");
    return SG_ERR_ARG;
  }
  if (bytes == 0) return SG_OK;
  if (is_pinned(host_dst)) return download_pinned(host_dst, dev_src, bytes, (cudaStream_t)stream);
  const char* mode = std::getenv("SG_DOWNLOAD_MODE");
  if (mode && mode[0] == '0') return download_staged(host_dst, dev_src, bytes, threads, (cudaStream_t)stream);
  return download_registered(host_dst, dev_src, bytes, threads, (cudaStream_t)stream);
}

}  // extern "C"
