// hostcopy.h — parallel host memcpy for the host-buffer entry points (internal).
//
// The host variants of the batched entry points (tsb_score_queue) take pageable caller arrays.
// Copying those with cudaMemcpyAsync goes through the driver's small pageable bounce buffers one
// array at a time (~8 GB/s measured).  Instead, a small persistent thread team packs them into a
// pinned staging block (one H2D) and unpacks the pinned results (one D2H per output block).
#pragma once

#include <immintrin.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace tsb {

struct CopySpan {
  void* dst;
  const void* src;  // NULL: zero-fill dst
  size_t bytes;
};

class HostCopyTeam {
 public:
  static HostCopyTeam& get() {
    static HostCopyTeam team;
    return team;
  }

  // Copies every span, splitting the concatenated byte range evenly across the team.
  // Cache hygiene around DMA (measured on the B200 box, 100K-request scorer call):
  //  * PACK_NT: non-temporal stores, for a destination a DMA engine reads next.  Copied by
  //    several cores, it would otherwise sit dirty in their private L2s and every PCIe read would
  //    snoop a core (6.5 MB H2D: 0.5-1.2 ms instead of 0.13 ms).
  //  * UNPACK_FLUSH: flush the source lines after reading them, for a pinned buffer a DMA engine
  //    writes next (3.2 MB D2H into lines cached by the last unpack: 0.5 ms instead of 0.06 ms).
  enum Mode { PLAIN = 0, PACK_NT = 1, UNPACK_FLUSH = 2 };
  void run(const std::vector<CopySpan>& spans, Mode nt = PLAIN) {
    std::lock_guard<std::mutex> one_job(run_m_);
    size_t total = 0;
    for (const auto& s : spans) total += s.bytes;
    const int t = total < (size_t{1} << 18) ? 1 : n_;  // small jobs: not worth the wake-up
    if (t == 1) {
      part(spans, 0, total, nt);
      return;
    }
    {
      std::unique_lock<std::mutex> lk(m_);
      spans_ = &spans;
      nt_ = nt;
      total_ = total;
      parts_ = t;
      pending_ = t - 1;
      ++gen_;
    }
    cv_.notify_all();
    part(spans, 0, total / t, nt);  // the caller does part 0
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return pending_ == 0; });
  }

  ~HostCopyTeam() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& th : th_) th.join();
  }

 private:
  HostCopyTeam() {
    n_ = static_cast<int>(std::min(8u, std::max(1u, std::thread::hardware_concurrency())));
    for (int i = 1; i < n_; ++i) th_.emplace_back([this, i] { worker(i); });
  }

  static void copy_nt(uint8_t* d, const uint8_t* s, size_t n) {
    const size_t head = std::min(n, (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15);
    std::memcpy(d, s, head);
    d += head, s += head, n -= head;
    size_t i = 0;
    for (; i + 64 <= n; i += 64) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
      const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
      const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
    }
    std::memcpy(d + i, s + i, n - i);
  }

  __attribute__((target("clflushopt"))) static void flush_opt(const uint8_t* p, size_t n) {
    for (uintptr_t l = reinterpret_cast<uintptr_t>(p) & ~uintptr_t{63};
         l < reinterpret_cast<uintptr_t>(p + n); l += 64)
      _mm_clflushopt(reinterpret_cast<void*>(l));
    _mm_sfence();
  }
  static void flush(const uint8_t* p, size_t n) {
    static const bool opt = __builtin_cpu_supports("clflushopt");
    if (opt) return flush_opt(p, n);
    for (uintptr_t l = reinterpret_cast<uintptr_t>(p) & ~uintptr_t{63};
         l < reinterpret_cast<uintptr_t>(p + n); l += 64)
      _mm_clflush(reinterpret_cast<const void*>(l));
  }

  static void part(const std::vector<CopySpan>& spans, size_t lo, size_t hi, Mode nt) {
    size_t base = 0;
    for (const auto& s : spans) {
      const size_t a = std::max(lo, base), b = std::min(hi, base + s.bytes);
      if (a < b) {
        auto* d = static_cast<uint8_t*>(s.dst) + (a - base);
        if (!s.src)
          std::memset(d, 0, b - a);
        else if (nt == PACK_NT)
          copy_nt(d, static_cast<const uint8_t*>(s.src) + (a - base), b - a);
        else
          std::memcpy(d, static_cast<const uint8_t*>(s.src) + (a - base), b - a);
        if (s.src && nt == UNPACK_FLUSH) flush(static_cast<const uint8_t*>(s.src) + (a - base), b - a);
      }
      base += s.bytes;
      if (base >= hi) break;
    }
    if (nt == PACK_NT) _mm_sfence();  // order the streaming stores before the caller's DMA submit
  }

  void worker(int i) {
    uint64_t seen = 0;
    for (;;) {
      const std::vector<CopySpan>* spans;
      size_t lo, hi;
      Mode nt;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (i >= parts_) continue;
        spans = spans_;
        nt = nt_;
        lo = total_ * i / parts_;
        hi = total_ * (i + 1) / parts_;
      }
      part(*spans, lo, hi, nt);
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }

  int n_ = 1;
  std::vector<std::thread> th_;
  std::mutex run_m_, m_;
  std::condition_variable cv_, done_;
  const std::vector<CopySpan>* spans_ = nullptr;
  size_t total_ = 0;
  int parts_ = 1, pending_ = 0;
  Mode nt_ = PLAIN;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace tsb
