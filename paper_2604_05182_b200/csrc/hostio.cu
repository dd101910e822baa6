// Host-buffer transfers of the reference API (the drop-in's NumPy in / out).
//
// The reference's functions take and return host arrays
// (lsrm/nsa_attention.py:287-327 `nsa_cross_attention(x, kv_feats, ...)`),
// so every call through the drop-in moves its inputs host -> device.  The
// bf16 engines consume bf16 rows in block-major order; this file does that
// conversion and permutation on the HOST, into pinned staging chunks that
// the copy engine ships while the next chunk is converted:
//
//   pageable f32 rows --(host threads: row gather + RNE f32->bf16)--> pinned
//   staging slot k --(cudaMemcpyAsync, stream)--> device rows, slot k reused
//   once its event has fired.
//
// Against "copy into pinned f32, DMA f32, gather + cast on the device" this
// halves the PCIe bytes, reads the pageable source once and overlaps the
// host pass with the DMA.  Round-to-nearest-even with NaN -> 0x7fff is what
// __float2bfloat16_rn (F2FP.BF16) does, so rows are bit-identical to the
// device cast.
//
// Host threads: one process-wide pool (LSRM_HOST_THREADS, default
// min(16, hardware threads)); callers serialise on it.  Staging rings are
// per device, taken from a free list per call, so concurrent callers on
// different threads never share a slot.
#include "common.cuh"

#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <unistd.h>
#include <vector>

namespace lsrm {
namespace {

class HostPool {
 public:
  static HostPool& get() {
    // never destroyed (workers outlive atexit); a forked child gets a pool of
    // its own (the parent's worker threads do not exist there)
    static std::mutex m;
    static HostPool* p = nullptr;
    static pid_t owner = 0;
    std::lock_guard<std::mutex> lk(m);
    if (p == nullptr || owner != getpid()) {
      p = new HostPool();
      owner = getpid();
    }
    return *p;
  }
  int parts() const { return (int)workers_.size() + 1; }
  // fn(part, n_parts) on every part; part n_parts-1 runs on the caller.
  void run(const std::function<void(int, int)>& fn) {
    std::lock_guard<std::mutex> serial(run_m_);
    const int n = parts();
    if (n == 1) {
      fn(0, 1);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = &fn;
      pending_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(n - 1, n);
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  HostPool() {
    int n = (int)std::thread::hardware_concurrency();
    if (const char* e = std::getenv("LSRM_HOST_THREADS")) n = std::atoi(e);
    n = std::max(1, std::min(n > 0 ? n : 1, 16));
    for (int i = 0; i + 1 < n; ++i) workers_.emplace_back([this, i] { loop(i); });
    for (auto& t : workers_) t.detach();
  }
  void loop(int i) {
    int64_t seen = 0;
    for (;;) {
      const std::function<void(int, int)>* job;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        job = job_;
      }
      (*job)(i, parts());
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_, run_m_;
  std::condition_variable cv_, done_;
  const std::function<void(int, int)>* job_ = nullptr;
  int64_t gen_ = 0;
  int pending_ = 0;
};

// Chunks of 2 MiB (measured on the B200 box, tools/h2d_sweep.py: 1, 2, 8 MiB
// slots x 8, 16 threads, and a variant where each thread streamed its own
// chunks with its own slots and copies: 2 MiB, 16 threads, all threads on one
// chunk at a time is fastest, 1.22 ms for 16815 x 1024 f32 rows = 56 GB/s
// of input, against 1.25 ms for a DMA of the same rows already in pinned
// memory).  Three slots: the copy of chunk c overlaps the conversion of
// chunk c+1 and c+2.
constexpr int kSlots = 3;
constexpr size_t kSlotBytes = 2u << 20;

struct Ring {
  int device = -1;
  void* slot[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  bool armed[kSlots] = {};
};

std::mutex g_ring_m;
std::vector<Ring*> g_free_rings;

int acquire_ring(Ring** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return set_error(LSRM_E_CUDA, "cudaGetDevice failed");
  {
    std::lock_guard<std::mutex> lk(g_ring_m);
    for (size_t i = 0; i < g_free_rings.size(); ++i)
      if (g_free_rings[i]->device == dev) {
        *out = g_free_rings[i];
        g_free_rings.erase(g_free_rings.begin() + i);
        return LSRM_OK;
      }
  }
  Ring* r = new Ring();
  r->device = dev;
  for (int k = 0; k < kSlots; ++k) {
    if (cudaHostAlloc(&r->slot[k], kSlotBytes, cudaHostAllocPortable) != cudaSuccess ||
        cudaEventCreateWithFlags(&r->ev[k], cudaEventDisableTiming) != cudaSuccess) {
      for (int j = 0; j < kSlots; ++j) {   // release what was made
        if (r->slot[j]) cudaFreeHost(r->slot[j]);
        if (r->ev[j]) cudaEventDestroy(r->ev[j]);
      }
      delete r;
      return set_error(LSRM_E_CUDA, "pinned staging allocation failed");
    }
  }
  *out = r;
  return LSRM_OK;
}

void release_ring(Ring* r) {
  std::lock_guard<std::mutex> lk(g_ring_m);
  g_free_rings.push_back(r);
}

// Round to nearest even, NaN -> 0x7fff: what __float2bfloat16_rn (F2FP.BF16)
// does.  Branch-free so the loop vectorises; an AVX2 clone is picked at load
// time when the host supports it.
__attribute__((target_clones("avx2", "default")))
void to_bf16_row(const uint32_t* __restrict__ su, uint16_t* __restrict__ du, int64_t m) {
  for (int64_t j = 0; j < m; ++j) {
    const uint32_t u = su[j];
    const uint32_t r = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
    du[j] = (uint16_t)((u & 0x7fffffffu) > 0x7f800000u ? 0x7fffu : r);
  }
}

void convert_row(const float* __restrict__ s, void* __restrict__ d, int64_t m, bool to_bf16) {
  if (to_bf16)
    to_bf16_row(reinterpret_cast<const uint32_t*>(s), static_cast<uint16_t*>(d), m);
  else
    std::memcpy(d, s, (size_t)m * 4);
}

}  // namespace
}  // namespace lsrm

using namespace lsrm;

extern "C" int lsrm_host_threads(void) { return HostPool::get().parts(); }

extern "C" int lsrm_h2d_rows(int to_bf16, const float* src, int64_t ld_src,
                             const int64_t* row_index, int64_t n_rows, int64_t row_elems,
                             void* dst, int64_t ld_dst, void* stream) {
  if (n_rows < 0 || row_elems < 0 || ld_src < row_elems || ld_dst < row_elems)
    return set_error(LSRM_E_CONFIG, "h2d_rows: bad shape (n %lld, row %lld, ld %lld/%lld)",
                     (long long)n_rows, (long long)row_elems, (long long)ld_src,
                     (long long)ld_dst);
  if (n_rows == 0 || row_elems == 0) return LSRM_OK;
  if (src == nullptr || dst == nullptr) return set_error(LSRM_E_CONFIG, "h2d_rows: null buffer");
  const int64_t eb = to_bf16 ? 2 : 4;
  const int64_t row_b = row_elems * eb;
  if ((size_t)row_b > kSlotBytes)
    return set_error(LSRM_E_CONFIG, "h2d_rows: a row exceeds the staging slot");
  const int64_t rows_per_chunk = (int64_t)kSlotBytes / row_b;
  const int64_t n_chunks = (n_rows + rows_per_chunk - 1) / rows_per_chunk;
  Ring* ring = nullptr;
  if (int st = acquire_ring(&ring)) return st;
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaSuccess;
  const char* what = "";
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int k = (int)(c % kSlots);
    const int64_t r0 = c * rows_per_chunk, nr = std::min(rows_per_chunk, n_rows - r0);
    if (ring->armed[k] && (e = cudaEventSynchronize(ring->ev[k])) != cudaSuccess) {
      what = "staging event wait";
      break;
    }
    char* stage = static_cast<char*>(ring->slot[k]);
    HostPool::get().run([&](int part, int parts) {
      const int64_t lo = nr * part / parts, hi = nr * (part + 1) / parts;
      for (int64_t t = lo; t < hi; ++t) {
        const int64_t srow = row_index ? row_index[r0 + t] : r0 + t;
        convert_row(src + srow * ld_src, stage + t * row_b, row_elems, to_bf16);
      }
    });
    if (ld_dst == row_elems)
      e = cudaMemcpyAsync(static_cast<char*>(dst) + r0 * row_b, stage, nr * row_b,
                          cudaMemcpyHostToDevice, s);
    else
      e = cudaMemcpy2DAsync(static_cast<char*>(dst) + r0 * ld_dst * eb, ld_dst * eb, stage,
                            row_b, row_b, nr, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaEventRecord(ring->ev[k], s);
    if (e != cudaSuccess) {
      what = "copy";
      break;
    }
    ring->armed[k] = true;
  }
  release_ring(ring);
  if (e != cudaSuccess)
    return set_error(LSRM_E_CUDA, "h2d_rows: %s failed: %s", what, cudaGetErrorString(e));
  return LSRM_OK;
}
