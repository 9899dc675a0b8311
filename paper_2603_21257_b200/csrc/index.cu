// index.cu — K7 device-side L2 chunk index: chained prefix-chunk hash -> L2 pool slot.
//
// SURVEY.md 8 f3.  The reference has no lookup: a request's cached prefix is the synthetic
// `cache_hit_ratio` fed to cached_token_count (types.cpp:73-79).  Here the hashes K3 computes for
// a request's full chunks are looked up in an open-addressing table (linear probing, 64-bit keys,
// atomicCAS insert) that indexes the L2 pool; the matched prefix length (leading chunks present)
// replaces the hit ratio and the matched slots are the ingest plan's sources.  Because hash c
// names the whole prefix [0, 256(c+1)), the match stops at the first absent chunk.
#include "common.cuh"
#include "kernels.h"

namespace tsb {
namespace {

constexpr uint64_t kEmpty = ~0ull;
constexpr uint64_t kTomb = ~0ull - 1;

__device__ __forceinline__ uint64_t slot_of(uint64_t h, uint64_t mask) {
  return mix64(h) & mask;  // FNV low bits are weak; remix before masking
}

// Insert phase 1: claim (or find) the key's entry, remember its position, and bid for the value
// with tag = epoch << 40 | (2^40 - 1 - i): the latest insert call wins, and inside one call the
// LOWEST batch index wins, so duplicate keys in a batch resolve deterministically.
__global__ void k_index_insert(uint64_t* __restrict__ keys, uint64_t* __restrict__ owner,
                               uint64_t mask, int64_t n, const uint64_t* __restrict__ hashes,
                               uint64_t epoch, int64_t* __restrict__ pos,
                               unsigned long long* __restrict__ stats /* [0]=new, [1]=full */) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint64_t h = hashes[i];
  const uint64_t tag = (epoch << 40) | ((1ull << 40) - 1 - static_cast<uint64_t>(i));
  uint64_t p = slot_of(h, mask);
  for (uint64_t probe = 0; probe <= mask; ++probe, p = (p + 1) & mask) {
    const uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long*>(keys + p),
                                    static_cast<unsigned long long>(kEmpty),
                                    static_cast<unsigned long long>(h));
    if (prev == kEmpty || prev == h) {
      if (prev == kEmpty) atomicAdd(stats, 1ull);
      atomicMax(reinterpret_cast<unsigned long long*>(owner + p), static_cast<unsigned long long>(tag));
      pos[i] = static_cast<int64_t>(p);
      return;
    }
  }
  pos[i] = -1;
  atomicAdd(stats + 1, 1ull);  // table full
}

// Insert phase 2: the winning bid of each entry writes its value.
__global__ void k_index_commit(const uint64_t* __restrict__ owner, int64_t* __restrict__ vals,
                               int64_t n, const int64_t* __restrict__ slots, uint64_t epoch,
                               const int64_t* __restrict__ pos) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int64_t p = pos[i];
  const uint64_t tag = (epoch << 40) | ((1ull << 40) - 1 - static_cast<uint64_t>(i));
  if (p >= 0 && owner[p] == tag) vals[p] = slots[i];
}

// Compaction: live entries of the old table re-inserted into an empty one (keys are unique, so
// one CAS per entry); tombstones are dropped.
__global__ void k_index_rehash(const uint64_t* __restrict__ okeys, const int64_t* __restrict__ ovals,
                               const uint64_t* __restrict__ oowner, uint64_t cap,
                               uint64_t* __restrict__ keys, int64_t* __restrict__ vals,
                               uint64_t* __restrict__ owner, uint64_t mask) {
  const uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (q >= cap) return;
  const uint64_t h = okeys[q];
  if (h == kEmpty || h == kTomb) return;
  uint64_t p = slot_of(h, mask);
  for (uint64_t probe = 0; probe <= mask; ++probe, p = (p + 1) & mask) {
    if (atomicCAS(reinterpret_cast<unsigned long long*>(keys + p), static_cast<unsigned long long>(kEmpty),
                  static_cast<unsigned long long>(h)) == kEmpty) {
      vals[p] = ovals[q];
      owner[p] = oowner[q];
      return;
    }
  }
}

__global__ void k_index_erase(uint64_t* __restrict__ keys, uint64_t mask, int64_t n,
                              const uint64_t* __restrict__ hashes,
                              unsigned long long* __restrict__ stats /* [2]=erased */) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint64_t h = hashes[i];
  uint64_t p = slot_of(h, mask);
  for (uint64_t probe = 0; probe <= mask; ++probe, p = (p + 1) & mask) {
    const uint64_t k = keys[p];
    if (k == kEmpty) return;
    if (k == h) {
      if (atomicCAS(reinterpret_cast<unsigned long long*>(keys + p),
                    static_cast<unsigned long long>(h), static_cast<unsigned long long>(kTomb)) == h)
        atomicAdd(stats + 2, 1ull);
      return;
    }
  }
}

// Any int64 value may be stored (a negative one names the HBM tier: slot ~v), so a miss is a
// flag, not a value.
__device__ __forceinline__ bool probe_find(const uint64_t* __restrict__ keys,
                                           const int64_t* __restrict__ vals, uint64_t mask,
                                           uint64_t h, int64_t* v) {
  uint64_t p = slot_of(h, mask);
  for (uint64_t probe = 0; probe <= mask; ++probe, p = (p + 1) & mask) {
    const uint64_t k = keys[p];
    if (k == h) {
      *v = vals[p];
      return true;
    }
    if (k == kEmpty) return false;
  }
  return false;
}

// One warp per request: 32 chunks probed in parallel per step, ballot finds the first miss.
__global__ void __launch_bounds__(256) k_index_lookup(const uint64_t* __restrict__ keys,
                                                      const int64_t* __restrict__ vals,
                                                      uint64_t mask, int64_t n_req,
                                                      const int64_t* __restrict__ chunk_offsets,
                                                      const uint64_t* __restrict__ hashes,
                                                      int64_t* __restrict__ slots_out,
                                                      int64_t* __restrict__ matched) {
  const int64_t r = blockIdx.x * 8ll + (threadIdx.x >> 5);
  if (r >= n_req) return;
  const int lane = threadIdx.x & 31;
  const int64_t b = chunk_offsets[r], e = chunk_offsets[r + 1];
  int64_t m = e - b;
  bool missed = false;
  for (int64_t c = b; c < e; c += 32) {
    const int64_t cc = c + lane;
    int64_t s = -1;
    bool found = false;
    if (!missed && cc < e) found = probe_find(keys, vals, mask, hashes[cc], &s);
    const unsigned miss = __ballot_sync(0xffffffffu, cc < e && !missed && !found);
    if (!missed && miss) {
      m = (c - b) + __ffs(miss) - 1;
      missed = true;
    }
    if (cc < e) slots_out[cc] = (missed && cc - b >= m) ? -1 : s;
  }
  if (lane == 0) matched[r] = m;
}

}  // namespace

cudaError_t launch_index_insert(uint64_t* keys, int64_t* vals, uint64_t* owner, uint64_t mask,
                                int64_t n, const uint64_t* hashes, const int64_t* slots,
                                uint64_t epoch, int64_t* pos, unsigned long long* stats,
                                cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_index_insert<<<ceil_div(n, 256), 256, 0, st>>>(keys, owner, mask, n, hashes, epoch, pos, stats);
  k_index_commit<<<ceil_div(n, 256), 256, 0, st>>>(owner, vals, n, slots, epoch, pos);
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_index_rehash(const uint64_t* okeys, const int64_t* ovals, const uint64_t* oowner,
                                uint64_t cap, uint64_t* keys, int64_t* vals, uint64_t* owner,
                                uint64_t mask, cudaStream_t st) {
  k_index_rehash<<<ceil_div(static_cast<int64_t>(cap), 256), 256, 0, st>>>(okeys, ovals, oowner, cap, keys, vals,
                                                                          owner, mask);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_index_erase(uint64_t* keys, uint64_t mask, int64_t n, const uint64_t* hashes,
                               unsigned long long* stats, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_index_erase<<<ceil_div(n, 256), 256, 0, st>>>(keys, mask, n, hashes, stats);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_index_lookup(const uint64_t* keys, const int64_t* vals, uint64_t mask,
                                int64_t n_req, const int64_t* chunk_offsets,
                                const uint64_t* hashes, int64_t* slots_out, int64_t* matched,
                                cudaStream_t st) {
  if (n_req == 0) return cudaSuccess;
  k_index_lookup<<<ceil_div(n_req, 8), 256, 0, st>>>(keys, vals, mask, n_req, chunk_offsets,
                                                     hashes, slots_out, matched);
  count_launch();
  return cudaGetLastError();
}

}  // namespace tsb
