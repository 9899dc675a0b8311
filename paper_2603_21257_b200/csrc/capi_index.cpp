// capi_index.cpp — C ABI of the device L2 chunk index (K7).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"

using tsb::fail;

struct tsb_index {
  int device = 0;
  uint64_t* keys = nullptr;
  int64_t* vals = nullptr;
  uint64_t* owner = nullptr;  // winning insert tag per entry (deterministic duplicates)
  uint64_t mask = 0;
  uint64_t epoch = 0;         // insert calls so far
  int64_t* pos = nullptr;     // per-batch entry positions (grow-only)
  int64_t pos_cap = 0;
  unsigned long long* stats = nullptr;  // [0] entries inserted, [1] full failures, [2] erased
};

namespace {

// Device scratch for the host-pointer variants.
struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
  tsb_status get(size_t need, void** out) {
    if (need > bytes) {
      cudaFree(p);
      p = nullptr;
      bytes = 0;
      TSB_CUDA_TRY(cudaMalloc(&p, need));
      bytes = need;
    }
    *out = p;
    return TSB_OK;
  }
};
thread_local Scratch g_scratch;

tsb_status check_keys(int64_t n, const uint64_t* hashes) {
  for (int64_t i = 0; i < n; ++i)
    if (hashes[i] >= ~0ull - 1)
      return fail(TSB_VALIDATION, "index: hash values 2^64-1 and 2^64-2 are reserved");
  return TSB_OK;
}

}  // namespace

extern "C" {

namespace {
void free_index_arrays(tsb_index* x) {
  cudaFree(x->keys);
  cudaFree(x->vals);
  cudaFree(x->owner);
  x->keys = nullptr;
  x->vals = nullptr;
  x->owner = nullptr;
}
cudaError_t alloc_index_arrays(tsb_index* x, int64_t cap) {
  cudaError_t e = cudaMalloc(&x->keys, sizeof(uint64_t) * cap);
  if (e == cudaSuccess) e = cudaMalloc(&x->vals, sizeof(int64_t) * cap);
  if (e == cudaSuccess) e = cudaMalloc(&x->owner, sizeof(uint64_t) * cap);
  if (e == cudaSuccess) e = cudaMemset(x->keys, 0xff, sizeof(uint64_t) * cap);
  if (e == cudaSuccess) e = cudaMemset(x->owner, 0, sizeof(uint64_t) * cap);
  return e;
}
}  // namespace

tsb_status tsb_index_create(int device, int64_t capacity, tsb_index** out) {
  if (capacity < 1 || capacity > (1ll << 40)) return fail(TSB_VALIDATION, "index: capacity out of range");
  int64_t cap = 1;
  while (cap < capacity) cap <<= 1;
  tsb::DeviceGuard dg(device);
  auto* x = new tsb_index();
  x->device = device;
  x->mask = static_cast<uint64_t>(cap - 1);
  cudaError_t e = alloc_index_arrays(x, cap);
  // insert-position scratch sized for a batch as large as the table (grown if a batch is larger)
  if (e == cudaSuccess) e = cudaMalloc(&x->pos, sizeof(int64_t) * cap);
  if (e == cudaSuccess) x->pos_cap = cap;
  if (e == cudaSuccess) e = cudaMalloc(&x->stats, 3 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(x->stats, 0, 3 * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    free_index_arrays(x);
    cudaFree(x->pos);
    cudaFree(x->stats);
    delete x;
    return tsb::cuda_fail(e, "tsb_index_create");
  }
  *out = x;
  return TSB_OK;
}

void tsb_index_destroy(tsb_index* x) {
  if (!x) return;
  tsb::DeviceGuard dg(x ? x->device : -1);
  free_index_arrays(x);
  cudaFree(x->pos);
  cudaFree(x->stats);
  delete x;
}

tsb_status tsb_index_clear(tsb_index* x, void* stream) {
  tsb::DeviceGuard dg(x ? x->device : -1);
  auto st = static_cast<cudaStream_t>(stream);
  const size_t cap = x->mask + 1;
  TSB_CUDA_TRY(cudaMemsetAsync(x->keys, 0xff, sizeof(uint64_t) * cap, st));
  TSB_CUDA_TRY(cudaMemsetAsync(x->owner, 0, sizeof(uint64_t) * cap, st));
  TSB_CUDA_TRY(cudaMemsetAsync(x->stats, 0, 3 * sizeof(unsigned long long), st));
  return TSB_OK;
}

tsb_status tsb_index_compact(tsb_index* x, void* stream, int64_t* tombstones_reclaimed) {
  tsb::DeviceGuard dg(x ? x->device : -1);
  auto st = static_cast<cudaStream_t>(stream);
  unsigned long long h[3] = {0, 0, 0};
  TSB_CUDA_TRY(cudaMemcpyAsync(h, x->stats, sizeof(h), cudaMemcpyDeviceToHost, st));
  TSB_CUDA_TRY(cudaStreamSynchronize(st));
  if (tombstones_reclaimed) *tombstones_reclaimed = static_cast<int64_t>(h[2]);
  if (h[2] == 0) return TSB_OK;
  const int64_t cap = static_cast<int64_t>(x->mask + 1);
  tsb_index old = *x;
  cudaError_t e = alloc_index_arrays(x, cap);
  if (e != cudaSuccess) {
    free_index_arrays(x);
    x->keys = old.keys;
    x->vals = old.vals;
    x->owner = old.owner;
    return tsb::cuda_fail(e, "tsb_index_compact");
  }
  TSB_CUDA_TRY(tsb::launch_index_rehash(old.keys, old.vals, old.owner, static_cast<uint64_t>(cap), x->keys,
                                        x->vals, x->owner, x->mask, st));
  const unsigned long long fresh[3] = {h[0] - h[2], 0, 0};
  TSB_CUDA_TRY(cudaMemcpyAsync(x->stats, fresh, sizeof(fresh), cudaMemcpyHostToDevice, st));
  TSB_CUDA_TRY(cudaStreamSynchronize(st));
  free_index_arrays(&old);
  return TSB_OK;
}

int64_t tsb_index_capacity(const tsb_index* x) { return static_cast<int64_t>(x->mask + 1); }

tsb_status tsb_index_insert_device(tsb_index* x, void* stream, int64_t n, const uint64_t* hashes,
                                   const int64_t* slots) {
  if (n <= 0) return TSB_OK;
  if (n >= (1ll << 40)) return fail(TSB_VALIDATION, "index: batch too large");
  tsb::DeviceGuard dg(x ? x->device : -1);
  auto st = static_cast<cudaStream_t>(stream);
  if (n > x->pos_cap) {  // grow-only scratch; the previous batch may still be using it
    TSB_CUDA_TRY(cudaStreamSynchronize(st));
    cudaFree(x->pos);
    x->pos = nullptr;
    x->pos_cap = 0;
    TSB_CUDA_TRY(cudaMalloc(&x->pos, sizeof(int64_t) * n));
    x->pos_cap = n;
  }
  ++x->epoch;
  TSB_CUDA_TRY(tsb::launch_index_insert(x->keys, x->vals, x->owner, x->mask, n, hashes, slots, x->epoch, x->pos,
                                        x->stats, st));
  return TSB_OK;
}

tsb_status tsb_index_erase_device(tsb_index* x, void* stream, int64_t n, const uint64_t* hashes) {
  TSB_CUDA_TRY(tsb::launch_index_erase(x->keys, x->mask, n, hashes, x->stats,
                                       static_cast<cudaStream_t>(stream)));
  return TSB_OK;
}

tsb_status tsb_index_lookup_device(tsb_index* x, void* stream, int64_t n_req,
                                   const int64_t* chunk_offsets, const uint64_t* hashes,
                                   int64_t* slots_out, int64_t* matched_out) {
  TSB_CUDA_TRY(tsb::launch_index_lookup(x->keys, x->vals, x->mask, n_req, chunk_offsets, hashes,
                                        slots_out, matched_out, static_cast<cudaStream_t>(stream)));
  return TSB_OK;
}

tsb_status tsb_index_stats(tsb_index* x, void* stream, int64_t* live, int64_t* full_failures) {
  unsigned long long h[3] = {0, 0, 0};
  auto st = static_cast<cudaStream_t>(stream);
  TSB_CUDA_TRY(cudaMemcpyAsync(h, x->stats, sizeof(h), cudaMemcpyDeviceToHost, st));
  TSB_CUDA_TRY(cudaStreamSynchronize(st));
  *live = static_cast<int64_t>(h[0] - h[2]);
  *full_failures = static_cast<int64_t>(h[1]);
  return TSB_OK;
}

tsb_status tsb_index_insert(tsb_index* x, void* stream, int64_t n, const uint64_t* hashes,
                            const int64_t* slots) {
  TSB_TRY(check_keys(n, hashes));
  if (n == 0) return TSB_OK;
  auto st = static_cast<cudaStream_t>(stream);
  void* d = nullptr;
  TSB_TRY(g_scratch.get(16 * static_cast<size_t>(n), &d));
  auto* dh = static_cast<uint64_t*>(d);
  auto* ds = reinterpret_cast<int64_t*>(dh + n);
  TSB_CUDA_TRY(cudaMemcpyAsync(dh, hashes, 8 * n, cudaMemcpyHostToDevice, st));
  TSB_CUDA_TRY(cudaMemcpyAsync(ds, slots, 8 * n, cudaMemcpyHostToDevice, st));
  int64_t live = 0, full0 = 0, full = 0;
  TSB_TRY(tsb_index_stats(x, stream, &live, &full0));
  TSB_TRY(tsb_index_insert_device(x, stream, n, dh, ds));
  TSB_TRY(tsb_index_stats(x, stream, &live, &full));
  if (full > full0) {
    // Tombstones left by erases may be what fills the probe paths: compact and re-insert the
    // batch once (idempotent: a later insert call wins every entry it touches).
    int64_t reclaimed = 0;
    TSB_TRY(tsb_index_compact(x, stream, &reclaimed));
    if (reclaimed > 0) {
      full0 = full;
      TSB_TRY(tsb_index_insert_device(x, stream, n, dh, ds));
      TSB_TRY(tsb_index_stats(x, stream, &live, &full));
    }
    if (full > full0)
      return fail(TSB_CAPACITY, "index: table full (" + std::to_string(full - full0) + " inserts failed)");
  }
  return TSB_OK;
}

tsb_status tsb_index_lookup(tsb_index* x, void* stream, int64_t n_req, const int64_t* chunk_offsets,
                            const uint64_t* hashes, int64_t* slots_out, int64_t* matched_out) {
  if (n_req == 0) return TSB_OK;
  if (chunk_offsets[0] != 0) return fail(TSB_VALIDATION, "index_lookup: chunk_offsets[0] must be 0");
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t total = chunk_offsets[n_req];
  const size_t bytes = 8 * (static_cast<size_t>(n_req + 1) + 2 * static_cast<size_t>(total) +
                            static_cast<size_t>(n_req));
  void* d = nullptr;
  TSB_TRY(g_scratch.get(bytes, &d));
  auto* dco = static_cast<int64_t*>(d);
  auto* dh = reinterpret_cast<uint64_t*>(dco + n_req + 1);
  auto* dslots = reinterpret_cast<int64_t*>(dh + total);
  auto* dm = dslots + total;
  TSB_CUDA_TRY(cudaMemcpyAsync(dco, chunk_offsets, 8 * (n_req + 1), cudaMemcpyHostToDevice, st));
  TSB_CUDA_TRY(cudaMemcpyAsync(dh, hashes, 8 * total, cudaMemcpyHostToDevice, st));
  TSB_TRY(tsb_index_lookup_device(x, stream, n_req, dco, dh, dslots, dm));
  TSB_CUDA_TRY(cudaMemcpyAsync(slots_out, dslots, 8 * total, cudaMemcpyDeviceToHost, st));
  TSB_CUDA_TRY(cudaMemcpyAsync(matched_out, dm, 8 * n_req, cudaMemcpyDeviceToHost, st));
  TSB_CUDA_TRY(cudaStreamSynchronize(st));
  return TSB_OK;
}

}  // extern "C"
