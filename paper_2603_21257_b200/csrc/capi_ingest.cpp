// capi_ingest.cpp — C ABI: L2 pinned chunk pool, L1 paged allocator + block_table, and the
// L2->L1 ingest launcher (K1 zero-copy / K1b bulk / CE + K2 scatter).
//
// The L1 allocator keeps TierLedger's byte semantics exactly (engine.cpp:18-49): reservations
// are granted iff nothing older waits and they fit; release grants the waiting queue strictly
// FIFO while reservations fit.  What the reference cannot express -- WHICH memory a grant
// gets -- is a FIFO free list of page ids (restated as alloc_ref in oracle/tsb_oracle.c) and a
// per-request block_table row, mirrored in pinned host memory and copied to the device by
// dirty row ranges.
//
// Block-table protocol: rows are only rewritten by grants (-1 -> page) while a request is
// live, and cleared by release, which the caller issues only after the request's device work
// has completed (the reference releases L1 at ComputeDone, engine.cpp:280-282).  Therefore an
// in-flight async copy of a row can never hand a kernel a stale page id.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <deque>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "ledger.h"

using tsb::fail;

namespace {

struct Knobs {
  int zerocopy_ctas = 64;
  int bulk_ctas = 64;
  int scatter_ctas = 148 * 32;  // HBM-source grid (K2, K1 over device pools): r01 K1 sweep
  int scatter_impl = 0;  // K2: 0 = SM load/store warps, 1 = bulk-copy (TMA engine)
  int ce_variant = 1;  // 0 = one cudaMemcpyAsync per item, 1 = one 2D copy per run of consecutive slots
  int64_t staging_bytes = 1ll << 30;  // 2 x 512 MiB: one K2 launch per layer of a 460-chunk request
};
Knobs g_knobs;

// Small pinned->device upload ring for item lists (16 slots; each slot reused only after the
// event recorded behind its consumer has completed).
struct UploadRing {
  static constexpr int kSlots = 16;
  static constexpr size_t kSlotBytes = 4u << 20;
  uint8_t* host = nullptr;
  uint8_t* dev = nullptr;
  cudaEvent_t ev[kSlots] = {};
  bool used[kSlots] = {};
  int next = 0;

  tsb_status init() {
    TSB_CUDA_TRY(cudaMallocHost(&host, kSlots * kSlotBytes));
    TSB_CUDA_TRY(cudaMalloc(&dev, kSlots * kSlotBytes));
    for (auto& e : ev) TSB_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return TSB_OK;
  }
  void destroy() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    cudaFreeHost(host);
    cudaFree(dev);
  }
  // Copies `bytes` (<= kSlotBytes) to a device slot on `st`; returns its device address.
  tsb_status stage(const void* src, size_t bytes, cudaStream_t st, void** dptr, int* slot) {
    const int s = next;
    next = (next + 1) % kSlots;
    if (used[s]) TSB_CUDA_TRY(cudaEventSynchronize(ev[s]));
    std::memcpy(host + s * kSlotBytes, src, bytes);
    TSB_CUDA_TRY(cudaMemcpyAsync(dev + s * kSlotBytes, host + s * kSlotBytes, bytes,
                                 cudaMemcpyHostToDevice, st));
    *dptr = dev + s * kSlotBytes;
    *slot = s;
    return TSB_OK;
  }
  tsb_status fence(int slot, cudaStream_t st) {
    used[slot] = true;
    TSB_CUDA_TRY(cudaEventRecord(ev[slot], st));
    return TSB_OK;
  }
};

}  // namespace

// ---------------------------------------------------------------------------------------
// L2 pool
// ---------------------------------------------------------------------------------------
struct tsb_pool {
  tsb_kv_shape shape{};
  uint8_t* host = nullptr;  // host address (NULL for device pools)
  uint8_t* dev = nullptr;   // device (UVA) address: mapped host alias, local or peer HBM
  int64_t slots = 0;
  int64_t chunk_bytes = 0;
  int location = TSB_POOL_HOST;
  int device = -1;          // owning GPU of a device pool (-1: host pool / unknown)
  bool owned = false;       // cudaFreeHost (host) or cudaFree (device) on destroy
  bool registered = false;  // cudaHostUnregister on destroy
  bool ipc = false;         // cudaIpcCloseMemHandle on destroy
  size_t mmapped = 0;       // tsb_pool_create_numa: munmap length on destroy
  int numa_node = -1;       // node the pages were bound to (-1: default policy)
};

namespace {

tsb_status new_device_pool(const tsb_kv_shape* shape, int device, int64_t n_slots,
                           tsb_pool** out) {
  int64_t cb = 0;
  TSB_TRY(tsb_kv_shape_info(shape, &cb, nullptr, nullptr));
  if (n_slots < 1) return fail(TSB_VALIDATION, "pool: n_slots must be >= 1");
  auto* p = new tsb_pool();
  p->shape = *shape;
  p->slots = n_slots;
  p->chunk_bytes = cb;
  p->location = TSB_POOL_DEVICE;
  p->device = device;
  *out = p;
  return TSB_OK;
}

}  // namespace

extern "C" {

tsb_status tsb_enable_peer_access(int device, int peer) {
  if (device == peer) return TSB_OK;
  int can = 0;
  TSB_CUDA_TRY(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can)
    return fail(TSB_UNSUPPORTED, "peer access " + std::to_string(device) + " -> " +
                                     std::to_string(peer) + " is not supported");
  int prev = 0;
  TSB_CUDA_TRY(cudaGetDevice(&prev));
  TSB_CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // not an error here; do not leave it for the next launch check
    return TSB_OK;
  }
  if (e != cudaSuccess) return tsb::cuda_fail(e, "tsb_enable_peer_access");
  return TSB_OK;
}

tsb_status tsb_pool_create_device(int device, const tsb_kv_shape* shape, int64_t n_slots,
                                  tsb_pool** out) {
  tsb_pool* p = nullptr;
  TSB_TRY(new_device_pool(shape, device, n_slots, &p));
  tsb::DeviceGuard dg(device);
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p->dev),
                                       static_cast<size_t>(p->chunk_bytes) * n_slots);
  if (e != cudaSuccess) {
    delete p;
    return tsb::cuda_fail(e, "tsb_pool_create_device (cudaMalloc)");
  }
  p->owned = true;
  *out = p;
  return TSB_OK;
}

tsb_status tsb_pool_wrap_device(int device, const tsb_kv_shape* shape, void* dev_base,
                                int64_t n_slots, tsb_pool** out) {
  cudaPointerAttributes a{};
  TSB_CUDA_TRY(cudaPointerGetAttributes(&a, dev_base));
  if (a.type != cudaMemoryTypeDevice)
    return fail(TSB_VALIDATION, "tsb_pool_wrap_device: dev_base is not device memory");
  if (a.device != device)
    return fail(TSB_VALIDATION, "tsb_pool_wrap_device: dev_base lives on device " +
                                    std::to_string(a.device));
  tsb_pool* p = nullptr;
  TSB_TRY(new_device_pool(shape, device, n_slots, &p));
  p->dev = static_cast<uint8_t*>(dev_base);
  *out = p;
  return TSB_OK;
}

tsb_status tsb_pool_ipc_handle(const tsb_pool* p, void* handle_out) {
  if (p->location != TSB_POOL_DEVICE || !p->owned)
    return fail(TSB_VALIDATION, "tsb_pool_ipc_handle: only tsb_pool_create_device pools export");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "64-byte IPC handle");
  cudaIpcMemHandle_t h;
  TSB_CUDA_TRY(cudaIpcGetMemHandle(&h, p->dev));
  std::memcpy(handle_out, &h, sizeof(h));
  return TSB_OK;
}

tsb_status tsb_pool_open_ipc(const tsb_kv_shape* shape, const void* handle, int owner_device,
                             int64_t n_slots, tsb_pool** out) {
  int cur = 0;
  TSB_CUDA_TRY(cudaGetDevice(&cur));
  if (owner_device >= 0) TSB_TRY(tsb_enable_peer_access(cur, owner_device));
  tsb_pool* p = nullptr;
  TSB_TRY(new_device_pool(shape, owner_device, n_slots, &p));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(reinterpret_cast<void**>(&p->dev), h,
                                       cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    delete p;
    return tsb::cuda_fail(e, "tsb_pool_open_ipc (cudaIpcOpenMemHandle)");
  }
  p->ipc = true;
  *out = p;
  return TSB_OK;
}

int tsb_pool_location_of(const tsb_pool* p) { return p->location; }
int tsb_pool_device(const tsb_pool* p) { return p->device; }

tsb_status tsb_pool_create(const tsb_kv_shape* shape, int64_t n_slots, tsb_pool** out) {
  int64_t cb = 0;
  TSB_TRY(tsb_kv_shape_info(shape, &cb, nullptr, nullptr));
  if (n_slots < 1) return fail(TSB_VALIDATION, "pool: n_slots must be >= 1");
  auto* p = new tsb_pool();
  p->shape = *shape;
  p->slots = n_slots;
  p->chunk_bytes = cb;
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p->host),
                                static_cast<size_t>(cb) * n_slots,
                                cudaHostAllocPortable | cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->dev), p->host, 0);
  if (e != cudaSuccess) {
    if (p->host) cudaFreeHost(p->host);
    delete p;
    return tsb::cuda_fail(e, "tsb_pool_create (cudaHostAlloc portable|mapped)");
  }
  p->owned = true;
  *out = p;
  return TSB_OK;
}

tsb_status tsb_pool_wrap(const tsb_kv_shape* shape, void* host_base, int64_t n_slots,
                         tsb_pool** out) {
  int64_t cb = 0;
  TSB_TRY(tsb_kv_shape_info(shape, &cb, nullptr, nullptr));
  auto* p = new tsb_pool();
  p->shape = *shape;
  p->slots = n_slots;
  p->chunk_bytes = cb;
  p->host = static_cast<uint8_t*>(host_base);
  cudaError_t e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->dev), host_base, 0);
  if (e != cudaSuccess) {
    delete p;
    return tsb::cuda_fail(e, "tsb_pool_wrap (memory must be page-locked and mapped)");
  }
  *out = p;
  return TSB_OK;
}

tsb_status tsb_pool_register(const tsb_kv_shape* shape, void* host_base, int64_t n_slots,
                             tsb_pool** out) {
  int64_t cb = 0;
  TSB_TRY(tsb_kv_shape_info(shape, &cb, nullptr, nullptr));
  if (n_slots < 1) return fail(TSB_VALIDATION, "pool: n_slots must be >= 1");
  TSB_CUDA_TRY(cudaHostRegister(host_base, static_cast<size_t>(cb) * n_slots,
                                cudaHostRegisterPortable | cudaHostRegisterMapped));
  tsb_status st = tsb_pool_wrap(shape, host_base, n_slots, out);
  if (st != TSB_OK) {
    cudaHostUnregister(host_base);
    return st;
  }
  (*out)->registered = true;
  return TSB_OK;
}

// ---- NUMA placement: every GPU's host link should pull from the DIMMs of
// its own socket, so an 8-GPU box does not funnel 8 links through one memory controller + UPI.
int tsb_device_numa_node(int device) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) return -1;
  for (char* c = bus; *c; ++c) *c = static_cast<char>(std::tolower(*c));
  const std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
  FILE* f = std::fopen(path.c_str(), "r");
  if (!f) return -1;
  int node = -1;
  if (std::fscanf(f, "%d", &node) != 1) node = -1;
  std::fclose(f);
  return node;
}

tsb_status tsb_pool_create_numa(const tsb_kv_shape* shape, int64_t n_slots, int numa_node,
                                tsb_pool** out) {
  int64_t cb = 0;
  TSB_TRY(tsb_kv_shape_info(shape, &cb, nullptr, nullptr));
  if (n_slots < 1) return fail(TSB_VALIDATION, "pool: n_slots must be >= 1");
  if (numa_node > 1023) return fail(TSB_VALIDATION, "pool: numa_node out of range");
  const size_t len = static_cast<size_t>(cb) * static_cast<size_t>(n_slots);
  void* base = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (base == MAP_FAILED) return fail(TSB_CAPACITY, "tsb_pool_create_numa: mmap of " + std::to_string(len) + " bytes failed");
  madvise(base, len, MADV_HUGEPAGE);  // fewer pages to pin and fewer IOMMU/GMMU entries
  int bound = -1;
  if (numa_node >= 0) {
    unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
    mask[numa_node / (8 * sizeof(unsigned long))] = 1ul << (numa_node % (8 * sizeof(unsigned long)));
    constexpr int kMpolBind = 2;
    if (syscall(SYS_mbind, base, len, kMpolBind, mask, 1024ul, 0u) != 0) {
      munmap(base, len);
      return fail(TSB_VALIDATION, "tsb_pool_create_numa: mbind to node " + std::to_string(numa_node) + " failed");
    }
    bound = numa_node;
  }
  // cudaHostRegister faults every page in -- on the bound node -- and pins it.
  tsb_status st = tsb_pool_register(shape, base, n_slots, out);
  if (st != TSB_OK) {
    munmap(base, len);
    return st;
  }
  (*out)->mmapped = len;
  (*out)->numa_node = bound;
  return TSB_OK;
}

int tsb_pool_numa_node(const tsb_pool* p) {
  if (p->location != TSB_POOL_HOST || !p->host) return -1;
  // get_mempolicy(MPOL_F_NODE | MPOL_F_ADDR): the node backing the first page.
  int node = -1;
  if (syscall(SYS_get_mempolicy, &node, nullptr, 0ul, p->host, 3ul) != 0) return p->numa_node;
  return node;
}

void tsb_pool_destroy(tsb_pool* p) {
  if (!p) return;
  tsb::DeviceGuard dg(p->location == TSB_POOL_DEVICE && p->owned ? p->device : -1);
  if (p->location == TSB_POOL_DEVICE) {
    if (p->owned) cudaFree(p->dev);
    if (p->ipc) cudaIpcCloseMemHandle(p->dev);
  } else {
    if (p->owned) cudaFreeHost(p->host);
    if (p->registered) cudaHostUnregister(p->host);
    if (p->mmapped) munmap(p->host, p->mmapped);
  }
  delete p;
}

void* tsb_pool_slot_ptr(tsb_pool* p, int64_t slot) {
  return (p->location == TSB_POOL_DEVICE ? p->dev : p->host) + slot * p->chunk_bytes;
}
int64_t tsb_pool_slots(const tsb_pool* p) { return p->slots; }
int64_t tsb_pool_chunk_bytes(const tsb_pool* p) { return p->chunk_bytes; }

tsb_status tsb_pool_fill_synthetic(tsb_pool* p, uint64_t seed, int64_t first, int64_t n,
                                   void* stream) {
  tsb::DeviceGuard dg(p->location == TSB_POOL_DEVICE ? p->device : -1);
  if (first < 0 || n < 0 || first + n > p->slots)
    return fail(TSB_VALIDATION, "pool_fill_synthetic: slot range out of bounds");
  auto st = static_cast<cudaStream_t>(stream);
  const uint64_t w0 = static_cast<uint64_t>(first) * p->chunk_bytes / 8;
  const uint64_t nw = static_cast<uint64_t>(n) * p->chunk_bytes / 8;
  auto* dst = reinterpret_cast<uint64_t*>(p->dev + first * p->chunk_bytes);
  TSB_CUDA_TRY(tsb::launch_fill_synth(dst, w0, nw, seed, st));
  TSB_CUDA_TRY(cudaStreamSynchronize(st));
  return TSB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// L1 paged allocator
// ---------------------------------------------------------------------------------------
struct tsb_l1 {
  int device = 0;
  tsb_kv_shape shape{};
  int64_t num_pages = 0;
  int64_t page_bytes = 0;  // local bytes of one page across all layers (K and V)
  int64_t ppc = 0;         // pages per chunk
  int layout = TSB_LAYOUT_FLASH_ATTN;
  tsb::Ledger ledger{2, 1};  // TierLedger(L1) byte accounting; capacity = pages * page_bytes
  // FIFO free list of page ids
  std::vector<int32_t> ring;
  int64_t head = 0, free_len = 0;
  // block table
  int64_t rows = 0, max_chunks = 0, stride = 0;
  int32_t* bt_host = nullptr;
  int32_t* bt_dev = nullptr;
  std::vector<uint8_t> row_dirty;
  std::unordered_map<int64_t, int32_t> row_of;
  std::vector<int32_t> free_rows;
  std::vector<std::vector<int32_t>> row_pages;  // pages held per row, grant order
  std::vector<int64_t> row_bytes;
  std::vector<int64_t> row_waiting;  // deferred reservations per row
  // arena
  uint8_t* arena = nullptr;
  bool arena_owned = false;
  int64_t layer_bytes = 0;
  // ingest state
  UploadRing ring_items;
  uint8_t* staging = nullptr;  // CE staging (lazy)
  int64_t staging_bytes = 0;
  int64_t group_cap = 0;       // CE staging-group cap in bytes (0: one half of the ring)
  cudaStream_t ce_stream = nullptr;
  cudaStream_t k2_stream = nullptr;  // K2 at the greatest stream priority: ahead of prefill kernels
  cudaEvent_t ev_k2_done = nullptr;
  cudaEvent_t ev_fence = nullptr;
  // two-tier ingest: the HBM-tier part runs on its own stream beside the host part; the host
  // part's first layer fence waits for it (fence_dep, consumed once)
  cudaStream_t tier_stream = nullptr;
  cudaEvent_t ev_tier_start = nullptr, ev_tier_done = nullptr;
  cudaEvent_t fence_dep = nullptr;
  cudaEvent_t ev_ce[2] = {};
  cudaEvent_t ev_k2[2] = {};
  bool k2_used[2] = {};
  int next_buf = 0;
  unsigned long long* verify_ctr = nullptr;
};

namespace {

void l1_free(tsb_l1* l) {
  if (!l) return;
  l->ring_items.destroy();
  if (l->arena_owned) cudaFree(l->arena);
  cudaFreeHost(l->bt_host);
  cudaFree(l->bt_dev);
  cudaFree(l->staging);
  cudaFree(l->verify_ctr);
  if (l->ev_fence) cudaEventDestroy(l->ev_fence);
  for (auto& e : l->ev_ce)
    if (e) cudaEventDestroy(e);
  for (auto& e : l->ev_k2)
    if (e) cudaEventDestroy(e);
  if (l->ce_stream) cudaStreamDestroy(l->ce_stream);
  if (l->k2_stream) cudaStreamDestroy(l->k2_stream);
  if (l->ev_k2_done) cudaEventDestroy(l->ev_k2_done);
  if (l->ev_tier_start) cudaEventDestroy(l->ev_tier_start);
  if (l->ev_tier_done) cudaEventDestroy(l->ev_tier_done);
  if (l->tier_stream) cudaStreamDestroy(l->tier_stream);
}

// Grants one reservation: takes pages from the free-list front into the block table row.
void grant(tsb_l1* l, int32_t block_index, int64_t bytes, int32_t row) {
  const int64_t n = bytes / l->page_bytes;
  int32_t* dst = l->bt_host + row * l->stride + static_cast<int64_t>(block_index) * l->ppc;
  const int64_t cap = static_cast<int64_t>(l->ring.size());
  for (int64_t k = 0; k < n; ++k) {
    const int32_t page = l->ring[(l->head + k) % cap];
    dst[k] = page;
    l->row_pages[row].push_back(page);
  }
  l->head = (l->head + n) % cap;
  l->free_len -= n;
  l->row_bytes[row] += bytes;
  l->row_dirty[row] = 1;
}

}  // namespace

extern "C" {

tsb_status tsb_l1_create(int device, const tsb_kv_shape* shape, int64_t num_pages,
                         int64_t max_rows, int64_t max_chunks, void* arena, tsb_l1** out) {
  int64_t cb = 0, pb = 0, lcb = 0;
  TSB_TRY(tsb_kv_shape_info(shape, &cb, &pb, &lcb));
  if (num_pages < 1 || num_pages > INT32_MAX)
    return fail(TSB_VALIDATION, "l1: num_pages must be in [1, 2^31)");
  if (max_rows < 1 || max_chunks < 1) return fail(TSB_VALIDATION, "l1: max_rows/max_chunks must be >= 1");
  tsb::DeviceGuard dg(device);
  auto* l = new tsb_l1();
  l->device = device;
  l->shape = *shape;
  l->num_pages = num_pages;
  l->page_bytes = pb;
  l->ppc = shape->chunk_tokens / shape->page_tokens;
  l->ledger = tsb::Ledger(2, num_pages * pb);
  l->ring.resize(static_cast<size_t>(num_pages));
  for (int64_t i = 0; i < num_pages; ++i) l->ring[i] = static_cast<int32_t>(i);
  l->free_len = num_pages;
  l->rows = max_rows;
  l->max_chunks = max_chunks;
  l->stride = max_chunks * l->ppc;
  l->row_dirty.assign(static_cast<size_t>(max_rows), 0);
  l->row_pages.resize(static_cast<size_t>(max_rows));
  l->row_bytes.assign(static_cast<size_t>(max_rows), 0);
  l->row_waiting.assign(static_cast<size_t>(max_rows), 0);
  for (int64_t r = max_rows - 1; r >= 0; --r) l->free_rows.push_back(static_cast<int32_t>(r));
  const int64_t Hl = shape->kv_heads / shape->tp_size;
  l->layer_bytes = 2 * num_pages * shape->page_tokens * Hl * shape->head_dim * shape->dtype_bytes;
  const size_t bt_bytes = sizeof(int32_t) * static_cast<size_t>(max_rows * l->stride);
  cudaError_t e = cudaMallocHost(&l->bt_host, bt_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&l->bt_dev, bt_bytes);
  if (e == cudaSuccess) {
    std::memset(l->bt_host, 0xff, bt_bytes);
    e = cudaMemset(l->bt_dev, 0xff, bt_bytes);
  }
  if (e == cudaSuccess && arena == nullptr) {
    e = cudaMalloc(&l->arena, static_cast<size_t>(l->layer_bytes) * shape->layers);
    l->arena_owned = e == cudaSuccess;
  } else {
    l->arena = static_cast<uint8_t*>(arena);
  }
  if (e == cudaSuccess) e = cudaMalloc(&l->verify_ctr, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    l1_free(l);
    delete l;
    return tsb::cuda_fail(e, "tsb_l1_create");
  }
  tsb_status st = l->ring_items.init();
  if (st != TSB_OK) {
    l1_free(l);
    delete l;
    return st;
  }
  *out = l;
  return TSB_OK;
}

void tsb_l1_destroy(tsb_l1* l) {
  if (!l) return;
  tsb::DeviceGuard dg(l ? l->device : -1);
  l1_free(l);
  delete l;
}

// TierLedger::request (engine.cpp:22-36) at page granularity.
tsb_status tsb_l1_request(tsb_l1* l, int64_t request_id, int32_t block_index, int64_t bytes,
                          int* granted, int32_t* bt_row) {
  std::string msg;
  if (bytes > 0 && bytes <= l->ledger.capacity()) {
    if (bytes % l->page_bytes != 0)
      return fail(TSB_VALIDATION, "l1: reservation of " + std::to_string(bytes) +
                                      " bytes is not a whole number of " +
                                      std::to_string(l->page_bytes) + "-byte pages");
    const int64_t n_pages = bytes / l->page_bytes;
    if (block_index < 0 || (static_cast<int64_t>(block_index) * l->ppc + n_pages) > l->stride)
      return fail(TSB_VALIDATION, "l1: block_index " + std::to_string(block_index) +
                                      " outside the block_table row (" +
                                      std::to_string(l->max_chunks) + " chunks)");
    if (!l->row_of.count(request_id) && l->free_rows.empty())
      return fail(TSB_CAPACITY, "l1: block_table has no free row for request " +
                                    std::to_string(request_id));
  }
  bool ok = false;
  const tsb_status st = l->ledger.request(request_id, block_index, bytes, &ok, &msg);
  if (st != TSB_OK) return fail(st, msg);
  int32_t row;
  auto it = l->row_of.find(request_id);
  if (it != l->row_of.end()) {
    row = it->second;
  } else {
    row = l->free_rows.back();
    l->free_rows.pop_back();
    l->row_of.emplace(request_id, row);
  }
  if (bt_row) *bt_row = row;
  if (ok) {
    grant(l, block_index, bytes, row);
  } else {
    l->row_waiting[row] += 1;
  }
  *granted = ok ? 1 : 0;
  return TSB_OK;
}

// ComputeDone release (engine.cpp:280-282) + TierLedger::release FIFO grants (:38-49).
tsb_status tsb_l1_release_request(tsb_l1* l, int64_t request_id, tsb_grant* out, int64_t cap,
                                  int64_t* n) {
  *n = 0;
  auto it = l->row_of.find(request_id);
  if (it == l->row_of.end())
    return fail(TSB_VALIDATION, "TierLedger: releasing more than reserved (request " +
                                    std::to_string(request_id) + " holds nothing)");
  const int32_t row = it->second;
  if (l->row_waiting[row] > 0)
    return fail(TSB_VALIDATION, "l1: request " + std::to_string(request_id) +
                                    " still has deferred reservations");
  // Return pages to the back of the free list in grant order.
  const int64_t ringcap = static_cast<int64_t>(l->ring.size());
  for (int32_t page : l->row_pages[row]) {
    l->ring[(l->head + l->free_len) % ringcap] = page;
    ++l->free_len;
  }
  const int64_t bytes = l->row_bytes[row];
  l->row_pages[row].clear();
  l->row_bytes[row] = 0;
  std::fill(l->bt_host + row * l->stride, l->bt_host + (row + 1) * l->stride, -1);
  l->row_dirty[row] = 1;
  l->row_of.erase(it);
  l->free_rows.push_back(row);
  std::string msg;
  const tsb_status st = l->ledger.release(
      bytes,
      [&](const tsb::Ledger::Pending& p) {
        const int32_t prow = l->row_of.at(p.request_id);
        l->row_waiting[prow] -= 1;
        grant(l, p.block_index, p.bytes, prow);
        if (*n < cap) out[*n] = tsb_grant{p.request_id, p.block_index, prow, p.bytes};
        ++*n;
      },
      &msg);
  if (st != TSB_OK) return fail(st, msg);
  return TSB_OK;
}

tsb_status tsb_l1_set_layout(tsb_l1* l, int layout) {
  if (layout < TSB_LAYOUT_FLASH_ATTN || layout > TSB_LAYOUT_FLASHINFER_HND)
    return fail(TSB_VALIDATION, "l1: unknown layout " + std::to_string(layout));
  if (l->ledger.reserved() != 0 || l->ledger.deferred() != 0)
    return fail(TSB_VALIDATION, "l1: the page layout can only change while nothing is reserved");
  l->layout = layout;
  return TSB_OK;
}
int tsb_l1_layout(const tsb_l1* l) { return l->layout; }

int64_t tsb_l1_reserved(const tsb_l1* l) { return l->ledger.reserved(); }
int64_t tsb_l1_capacity(const tsb_l1* l) { return l->ledger.capacity(); }
int64_t tsb_l1_deferred(const tsb_l1* l) { return l->ledger.deferred(); }
int64_t tsb_l1_free_pages(const tsb_l1* l) { return l->free_len; }
int64_t tsb_l1_num_pages(const tsb_l1* l) { return l->num_pages; }
int64_t tsb_l1_page_bytes(const tsb_l1* l) { return l->page_bytes; }
int tsb_l1_device(const tsb_l1* l) { return l->device; }
tsb_status tsb_l1_shape(const tsb_l1* l, tsb_kv_shape* out) {
  *out = l->shape;
  return TSB_OK;
}
void* tsb_l1_arena(tsb_l1* l) { return l->arena; }
void* tsb_l1_layer_ptr(tsb_l1* l, int64_t layer) { return l->arena + layer * l->layer_bytes; }
const int32_t* tsb_l1_block_table_host(const tsb_l1* l) { return l->bt_host; }
const int32_t* tsb_l1_block_table_device(const tsb_l1* l) { return l->bt_dev; }
int64_t tsb_l1_block_table_stride(const tsb_l1* l) { return l->stride; }

tsb_status tsb_l1_sync_block_table(tsb_l1* l, void* stream) {
  tsb::DeviceGuard dg(l ? l->device : -1);
  auto st = static_cast<cudaStream_t>(stream);
  int64_t r = 0;
  while (r < l->rows) {
    if (!l->row_dirty[r]) {
      ++r;
      continue;
    }
    int64_t e = r;
    while (e < l->rows && l->row_dirty[e]) l->row_dirty[e++] = 0;
    TSB_CUDA_TRY(cudaMemcpyAsync(l->bt_dev + r * l->stride, l->bt_host + r * l->stride,
                                 sizeof(int32_t) * (e - r) * l->stride, cudaMemcpyHostToDevice,
                                 st));
    r = e;
  }
  return TSB_OK;
}

tsb_status tsb_ingest_set_grid(int zerocopy_ctas, int bulk_ctas, int scatter_ctas) {
  g_knobs.zerocopy_ctas = zerocopy_ctas > 0 ? zerocopy_ctas : 64;
  g_knobs.bulk_ctas = bulk_ctas > 0 ? bulk_ctas : 64;
  g_knobs.scatter_ctas = scatter_ctas > 0 ? scatter_ctas : 148 * 32;
  return TSB_OK;
}

tsb_status tsb_ingest_set_scatter(int impl, int ctas) {
  if (impl < 0 || impl > 1) return fail(TSB_VALIDATION, "ingest_set_scatter: impl must be 0 or 1");
  g_knobs.scatter_impl = impl;
  g_knobs.scatter_ctas = ctas > 0 ? ctas : (impl == 0 ? 148 * 32 : 148);
  return TSB_OK;
}

}  // extern "C"

namespace {

// ---- tensor maps for K1b (cuTensorMapEncodeTiled through the runtime's driver entry point) ----
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// Source map whose box is one page segment.  base = slot 0 of the pool (or the staging ring),
// rows = every token row [outer][2][C] of it, pitch = bytes per token row.  NHD: 2D map over
// 8-byte columns, box (run/8, P) at column head_off/8.  HND: 3D map ordered (D, token rows, heads)
// with strides (pitch, D*E), box (D*E/8, P, H_local) -> shared memory [H_local][P][D].
tsb_status make_segment_map(const tsb::IngestGeom& g, const void* base, int64_t rows, CUtensorMap* m,
                            tsb::TmaSrc* ts, int64_t layers, int64_t C) {
  const EncodeTiledFn enc = encode_tiled();
  if (!enc) return fail(TSB_UNSUPPORTED, "ingest bulk: cuTensorMapEncodeTiled is unavailable");
  if (g.run % 16 || g.head_bytes % 16 || g.row % 16 || g.run / 8 > 256 || g.head_bytes / 8 > 256 || g.P > 256 ||
      g.run / g.head_bytes > 256 || rows >= (int64_t{1} << 31))
    return fail(TSB_UNSUPPORTED, "ingest bulk: page segment exceeds one TMA box (rows <= 2 KiB, < 2^31 rows)");
  ts->layers = layers;
  ts->C = C;
  ts->x0 = static_cast<int32_t>(g.head_off / 8);
  ts->head0 = static_cast<int32_t>(g.head_off / g.head_bytes);
  CUresult r;
  if (g.hnd) {
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.head_bytes / 8), static_cast<cuuint64_t>(rows),
                                static_cast<cuuint64_t>(g.row / g.head_bytes)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.row), static_cast<cuuint64_t>(g.head_bytes)};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(g.head_bytes / 8), static_cast<cuuint32_t>(g.P),
                               static_cast<cuuint32_t>(g.run / g.head_bytes)};
    const cuuint32_t es[3] = {1, 1, 1};
    r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.row / 8), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.row)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(g.run / 8), static_cast<cuuint32_t>(g.P)};
    const cuuint32_t es[2] = {1, 1};
    r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS)
    return fail(TSB_UNSUPPORTED, "ingest bulk: cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return TSB_OK;
}

// K2: HBM staging -> pages, with the SM load/store kernel or the tensor-map TMA kernel (K1b).
tsb_status launch_scatter(const tsb::IngestGeom& g, const uint8_t* src, uint8_t* arena,
                          const tsb_ingest_item* items, const int32_t* bt, int64_t n, cudaStream_t st,
                          int device) {
  if (g_knobs.scatter_impl == 1) {
    CUtensorMap m;
    tsb::TmaSrc ts{};
    TSB_TRY(make_segment_map(g, src, n * g.n_layers * 2 * (g.kv_src / g.row), &m, &ts, g.n_layers,
                             g.kv_src / g.row));
    int sms = 148;
    TSB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    TSB_CUDA_TRY(tsb::launch_ingest_tma(m, g, ts, arena, items, bt, n, sms * tsb::tma_ctas_per_sm(g.seg_bytes), st));
    return TSB_OK;
  }
  TSB_CUDA_TRY(tsb::launch_ingest_ldg(g, src, arena, items, bt, n, g_knobs.scatter_ctas, st, true));
  return TSB_OK;
}

}  // namespace

namespace {

tsb::IngestGeom make_geom(const tsb_l1* l, int64_t layer_lo, int64_t layer_hi) {
  const tsb_kv_shape& s = l->shape;
  tsb::IngestGeom g{};
  const int64_t Hl = s.kv_heads / s.tp_size;
  g.row = s.kv_heads * s.head_dim * s.dtype_bytes;
  g.run = Hl * s.head_dim * s.dtype_bytes;
  g.head_off = s.tp_rank * g.run;
  g.chunk_bytes = s.layers * 2 * s.chunk_tokens * g.row;
  g.kv_src = s.chunk_tokens * g.row;
  g.layer_src = 2 * g.kv_src;
  g.P = s.page_tokens;
  g.ppc = l->ppc;
  g.seg_bytes = g.P * g.run;
  g.num_pages = l->num_pages;
  g.layer_dst = 2 * l->num_pages * g.seg_bytes;
  if (l->layout == TSB_LAYOUT_FLASH_ATTN) {  // [2][pages][P][H][D]
    g.kv_dst = l->num_pages * g.seg_bytes;
    g.page_dst = g.seg_bytes;
  } else {                                   // [pages][2][P][H][D] or [pages][2][H][P][D]
    g.kv_dst = g.seg_bytes;
    g.page_dst = 2 * g.seg_bytes;
  }
  g.head_bytes = s.head_dim * s.dtype_bytes;
  // With one local head, HND pages [2][1][P][D] are byte-identical to NHD [2][P][1][D]: take the
  // NHD addressing (contiguous page planes; K1 / K1b / K2 skip the per-row head transpose).
  g.hnd = l->layout == TSB_LAYOUT_FLASHINFER_HND && Hl > 1 ? 1 : 0;
  g.bt_stride = l->stride;
  g.layer_lo = static_cast<int32_t>(layer_lo);
  g.n_layers = static_cast<int32_t>(layer_hi - layer_lo);
  g.staged = 0;
  g.item_stride = 0;
  return g;
}

// Copy-engine cost model for head-sharded slices, measured on B200
// (repo:profiles/r01_ce_strided_probe.jsonl): a strided cudaMemcpy3DAsync moves a rank's slice
// at the contiguous H2D rate (55.3-55.6 GB/s for 256 B - 1 KiB runs) but costs ~4.6 us per
// call, while SM zero-copy loads cap at ~51.4 GB/s with no per-call cost.  The copy engines
// win once a call carries more than 4.6 us / (1/51.4 - 1/55.6 GB/s) ~ 3.1 MB.
constexpr double kCeBytesPerCallBreakEven = 3.1e6;

// Consecutive-slot runs in an item list: the number of 3D copies one layer needs.
int64_t slot_runs(const tsb_ingest_item* it, int64_t n) {
  int64_t runs = n > 0 ? 1 : 0;
  for (int64_t k = 1; k < n; ++k) runs += it[k].src_slot != it[k - 1].src_slot + 1;
  return runs;
}

// Geometry of one layer of items staged packed in HBM: each item's slice of this rank's heads,
// [K|V][C][run] contiguous, item k at k * layer_src.  K2 reads it as contiguous segments.
tsb::IngestGeom make_staged_geom(const tsb_l1* l, int64_t layer, int64_t n_layers = 1) {
  tsb::IngestGeom g = make_geom(l, layer, layer + n_layers);
  g.row = g.run;
  g.head_off = 0;
  g.kv_src = l->shape.chunk_tokens * g.run;
  g.layer_src = 2 * g.kv_src;
  g.staged = 1;
  g.item_stride = n_layers * g.layer_src;  // item k's layers at k * n_layers * layer slice
  return g;
}

int resolve_mode(const tsb_l1* l, const tsb_pool* pool, int mode, const tsb_ingest_item* items_host,
                 int64_t n_items) {
  if (mode != TSB_INGEST_AUTO) return mode;
  // A device pool (local or peer HBM) is read by SM loads: no host link to saturate.
  if (pool->location == TSB_POOL_DEVICE) return TSB_INGEST_ZEROCOPY;
  // Device-side item lists cannot drive host-issued copies.
  if (!items_host) return TSB_INGEST_ZEROCOPY;
  // Measured on B200 (profiles/r01_*): SM-initiated host reads plateau at ~92.6% of the copy
  // engines' H2D rate, so full-head chunks go through CE + K2.
  if (l->shape.tp_size == 1) return TSB_INGEST_CE;
  // Head-sharded chunks: the copy engines pull only this rank's heads with one strided 3D copy
  // per run of consecutive slots; worth it when the runs are long enough.
  const tsb_kv_shape& s = l->shape;
  const double slice = 2.0 * s.chunk_tokens * (s.kv_heads / s.tp_size) * s.head_dim * s.dtype_bytes;
  const double per_call = slice * n_items / static_cast<double>(slot_runs(items_host, n_items));
  return per_call >= kCeBytesPerCallBreakEven ? TSB_INGEST_CE : TSB_INGEST_ZEROCOPY;
}

tsb_status ensure_staging(tsb_l1* l) {
  if (l->staging) return TSB_OK;
  l->staging_bytes = g_knobs.staging_bytes;
  TSB_CUDA_TRY(cudaMalloc(&l->staging, l->staging_bytes));
  TSB_CUDA_TRY(cudaStreamCreateWithFlags(&l->ce_stream, cudaStreamNonBlocking));
  // K2 runs at the greatest priority so that, while a prefill occupies the SMs, the scatter
  // that drains the staging ring gets the next free SM slots and the copy engines never stall.
  int lo_prio = 0, hi_prio = 0;
  TSB_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  TSB_CUDA_TRY(cudaStreamCreateWithPriority(&l->k2_stream, cudaStreamNonBlocking, hi_prio));
  TSB_CUDA_TRY(cudaEventCreateWithFlags(&l->ev_k2_done, cudaEventDisableTiming));
  TSB_CUDA_TRY(cudaEventCreateWithFlags(&l->ev_fence, cudaEventDisableTiming));
  for (int b = 0; b < 2; ++b) {
    TSB_CUDA_TRY(cudaEventCreateWithFlags(&l->ev_ce[b], cudaEventDisableTiming));
    TSB_CUDA_TRY(cudaEventCreateWithFlags(&l->ev_k2[b], cudaEventDisableTiming));
  }
  return TSB_OK;
}

// Copies layers [layer, layer + nl) of items [0, n) into stage, packed: item k's layers at
// k * nl * (packed layer slice), each layer [K|V][C][this rank's run] -- on the copy-engine
// stream.  A chunk's layers are adjacent in the pool slot, so nl layers are one contiguous
// span (full heads) or one strided run of nl * 2 * C rows (head shards).
tsb_status ce_copy_layers(tsb_l1* l, tsb_pool* pool, const tsb_ingest_item* it, int64_t n,
                          int64_t layer, int64_t nl, uint8_t* stage) {
  const tsb::IngestGeom src = make_geom(l, layer, layer + 1);  // pool (slot) geometry
  const int64_t lb = make_staged_geom(l, layer).layer_src;      // packed slice of one item-layer
  const int64_t span = nl * lb;                                 // one item's bytes in the stage
  const uint8_t* base = pool->host + layer * src.layer_src + src.head_off;
  if (src.run != src.row) {
    // Head-sharded: one 3D copy per run of consecutive slots.  x = this rank's run of each token
    // row, y = the nl*2*C rows of the layers (pitch = the full row), z = slots (slice pitch = one
    // chunk = L*2*C rows).  The destination is packed.
    const size_t rows_per_chunk = static_cast<size_t>(src.chunk_bytes / src.row);
    const size_t rows = static_cast<size_t>(nl * 2 * l->shape.chunk_tokens);
    int64_t k = 0;
    while (k < n) {
      int64_t e = k + 1;
      while (e < n && it[e].src_slot == it[e - 1].src_slot + 1) ++e;
      cudaMemcpy3DParms p{};
      p.srcPtr = make_cudaPitchedPtr(const_cast<uint8_t*>(base + it[k].src_slot * src.chunk_bytes),
                                     static_cast<size_t>(src.row), static_cast<size_t>(src.run),
                                     rows_per_chunk);
      p.dstPtr = make_cudaPitchedPtr(stage + k * span, static_cast<size_t>(src.run),
                                     static_cast<size_t>(src.run), rows);
      p.extent = make_cudaExtent(static_cast<size_t>(src.run), rows, static_cast<size_t>(e - k));
      p.kind = cudaMemcpyHostToDevice;
      TSB_CUDA_TRY(cudaMemcpy3DAsync(&p, l->ce_stream));
      k = e;
    }
    return TSB_OK;
  }
  switch (g_knobs.ce_variant) {
    case 0:
      for (int64_t k = 0; k < n; ++k)
        TSB_CUDA_TRY(cudaMemcpyAsync(stage + k * span, base + it[k].src_slot * src.chunk_bytes, span,
                                     cudaMemcpyHostToDevice, l->ce_stream));
      return TSB_OK;
    default: {  // one 2D copy per run of consecutive pool slots (pitch = chunk bytes)
      int64_t k = 0;
      while (k < n) {
        int64_t e = k + 1;
        while (e < n && it[e].src_slot == it[e - 1].src_slot + 1) ++e;
        TSB_CUDA_TRY(cudaMemcpy2DAsync(stage + k * span, span, base + it[k].src_slot * src.chunk_bytes,
                                       src.chunk_bytes, span, e - k, cudaMemcpyHostToDevice,
                                       l->ce_stream));
        k = e;
      }
      return TSB_OK;
    }
  }
}

// Records a requested layer fence; the first one of a call waits for l->fence_dep (the HBM-tier
// part of a two-tier ingest) so that every fence covers both tiers.
tsb_status record_fence(tsb_l1* l, void* ev, cudaStream_t st) {
  if (l->fence_dep) {
    TSB_CUDA_TRY(cudaStreamWaitEvent(st, l->fence_dep, 0));
    l->fence_dep = nullptr;
  }
  TSB_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(ev), st));
  return TSB_OK;
}

// CE + K2: per staging group, the copy engines land the group's slices in one half of the HBM
// staging ring while K2 scatters the other half into pages.  A group is a set of items and a span
// of layers: when one layer of every item fits a half, consecutive layers up to the next requested
// fence share a group (fewer, larger copies and K2 launches); else one layer, items split.
tsb_status ingest_ce(tsb_l1* l, tsb_pool* pool, const tsb_ingest_item* items_dev,
                     const tsb_ingest_item* items_host, int64_t n_items, int64_t lo, int64_t hi,
                     cudaStream_t st, void* const* layer_events) {
  if (pool->location != TSB_POOL_HOST)
    return fail(TSB_UNSUPPORTED, "ingest CE mode reads host pools; use zerocopy/bulk for device pools");
  if (!items_host)
    return fail(TSB_UNSUPPORTED, "ingest CE mode needs host-visible items (use tsb_ingest)");
  TSB_TRY(ensure_staging(l));
  const int64_t lb = make_staged_geom(l, lo).layer_src;
  const int64_t half = l->staging_bytes / 2;
  if (lb > half) return fail(TSB_UNSUPPORTED, "ingest CE: one chunk layer exceeds the staging ring");
  // A group fills at most `cap` bytes of its half (at least one item-layer).
  const int64_t cap = l->group_cap > 0 ? std::max(lb, std::min(half, l->group_cap)) : half;
  const int64_t items_per_half = cap / lb;
  // Host reads are ordered after the work already queued on `st` (stream semantics).
  TSB_CUDA_TRY(cudaEventRecord(l->ev_fence, st));
  TSB_CUDA_TRY(cudaStreamWaitEvent(l->ce_stream, l->ev_fence, 0));
  TSB_CUDA_TRY(cudaStreamWaitEvent(l->k2_stream, l->ev_fence, 0));
  cudaStream_t ks = l->k2_stream;
  int64_t layer = lo;
  while (layer < hi) {
    int64_t span_end = hi;  // exclusive end of the layers before (and including) the next fence
    if (layer_events) {
      span_end = layer + 1;
      while (span_end < hi && !layer_events[span_end - 1 - lo]) ++span_end;
    }
    const int64_t nl = n_items <= items_per_half
                           ? std::max<int64_t>(1, std::min(span_end - layer, cap / (n_items * lb)))
                           : 1;
    const int64_t per_group = n_items <= items_per_half ? n_items : items_per_half;
    const tsb::IngestGeom g = make_staged_geom(l, layer, nl);
    for (int64_t i0 = 0; i0 < n_items; i0 += per_group) {
      const int64_t n = std::min(per_group, n_items - i0);
      const int b = l->next_buf;
      l->next_buf ^= 1;
      uint8_t* stage = l->staging + b * half;
      if (l->k2_used[b]) TSB_CUDA_TRY(cudaStreamWaitEvent(l->ce_stream, l->ev_k2[b], 0));
      TSB_TRY(ce_copy_layers(l, pool, items_host + i0, n, layer, nl, stage));
      TSB_CUDA_TRY(cudaEventRecord(l->ev_ce[b], l->ce_stream));
      TSB_CUDA_TRY(cudaStreamWaitEvent(ks, l->ev_ce[b], 0));
      TSB_TRY(launch_scatter(g, stage, l->arena, items_dev + i0, l->bt_dev, n, ks, l->device));
      TSB_CUDA_TRY(cudaEventRecord(l->ev_k2[b], ks));
      l->k2_used[b] = true;
    }
    layer += nl;
    if (layer_events && layer_events[layer - 1 - lo]) TSB_TRY(record_fence(l, layer_events[layer - 1 - lo], ks));
  }
  // The caller's stream resumes after the last scatter (stream semantics for what follows).
  TSB_CUDA_TRY(cudaEventRecord(l->ev_k2_done, ks));
  TSB_CUDA_TRY(cudaStreamWaitEvent(st, l->ev_k2_done, 0));
  return TSB_OK;
}

// CE-direct: the copy engines write the pages themselves (no SM work).  For full-head chunks a
// (layer, K|V, page j) segment is P contiguous token rows in the chunk and one contiguous page
// plane; consecutive pages of a chunk that landed on consecutive page ids (flash-attn planes)
// merge into one run, and runs that advance by constant strides on both sides (a document's
// chunks in consecutive slots on consecutive pages) merge into one 2D copy per (layer, K|V).
// A lone run moves K and V (y, pitch = the K|V stride) of every layer up to the next requested
// fence (z, slice = the layer stride) in one 3D copy.  The batched-memcpy entry points are closed
// on this GPU pool (they raised GPU faults), so every copy is a plain per-call 2D / 3D / 1D copy.
bool ce_direct_ok(const tsb_l1* l, const tsb_pool* pool) {
  return pool->location == TSB_POOL_HOST && l->shape.tp_size == 1 && l->layout != TSB_LAYOUT_FLASHINFER_HND;
}

tsb_status ingest_ce_direct(tsb_l1* l, tsb_pool* pool, const tsb_ingest_item* items_host, int64_t n_items,
                            int64_t lo, int64_t hi, cudaStream_t st, void* const* layer_events) {
  if (!ce_direct_ok(l, pool))
    return fail(TSB_UNSUPPORTED, "ingest CE direct: full-head chunks from a host pool into flash-attn / NHD pages only");
  if (!items_host) return fail(TSB_UNSUPPORTED, "ingest CE direct needs host-visible items (use tsb_ingest)");
  TSB_TRY(ensure_staging(l));  // the copy stream and its events (no staging memory is touched)
  TSB_CUDA_TRY(cudaEventRecord(l->ev_fence, st));
  TSB_CUDA_TRY(cudaStreamWaitEvent(l->ce_stream, l->ev_fence, 0));
  const tsb::IngestGeom g = make_geom(l, 0, 1);
  const int64_t ppc = l->ppc, seg = g.seg_bytes;
  const bool planes = l->layout == TSB_LAYOUT_FLASH_ATTN;  // consecutive pages are contiguous
  int max_pitch = 0;
  TSB_CUDA_TRY(cudaDeviceGetAttribute(&max_pitch, cudaDevAttrMaxPitch, l->device));
  // Runs of one layer's K plane (V and the other layers sit at fixed offsets): (item, pages j..e)
  // with consecutive page ids.  Runs of equal width whose source and destination both advance by
  // a constant stride form a strip -- e.g. the chunks of a document in consecutive slots landing
  // on consecutive pages -- and a strip is one 2D copy per (layer, K|V).
  struct Run {
    int64_t src, dst, width;  // byte offsets: pool slot area, arena (layer 0, K)
  };
  std::vector<Run> runs;
  runs.reserve(static_cast<size_t>(n_items));
  for (int64_t i = 0; i < n_items; ++i) {
    const tsb_ingest_item& it = items_host[i];
    const int32_t* pages = l->bt_host + it.bt_row * l->stride + static_cast<int64_t>(it.chunk_index) * ppc;
    int64_t j = 0;
    while (j < ppc) {
      int64_t e = j + 1;
      while (planes && e < ppc && pages[e] == pages[e - 1] + 1) ++e;
      runs.push_back(Run{it.src_slot * g.chunk_bytes + j * g.P * g.row, static_cast<int64_t>(pages[j]) * g.page_dst,
                         (e - j) * seg});
      j = e;
    }
  }
  struct Strip {
    size_t first, count;
    int64_t spitch, dpitch;
  };
  std::vector<Strip> strips;
  for (size_t k = 0; k < runs.size();) {
    Strip sp{k, 1, 0, 0};
    if (k + 1 < runs.size() && runs[k + 1].width == runs[k].width) {
      sp.spitch = runs[k + 1].src - runs[k].src;
      sp.dpitch = runs[k + 1].dst - runs[k].dst;
      if (sp.spitch >= runs[k].width && sp.dpitch >= runs[k].width && sp.spitch <= max_pitch && sp.dpitch <= max_pitch) {
        sp.count = 2;
        while (k + sp.count < runs.size() && runs[k + sp.count].width == runs[k].width &&
               runs[k + sp.count].src - runs[k + sp.count - 1].src == sp.spitch &&
               runs[k + sp.count].dst - runs[k + sp.count - 1].dst == sp.dpitch)
          ++sp.count;
      }
    }
    strips.push_back(sp);
    k += sp.count;
  }
  // A single run moves K|V x the span's layers in one 3D copy when both K|V strides are within
  // the copy engines' pitch limit.
  const bool use_3d = g.kv_dst <= max_pitch && g.kv_src <= max_pitch;
  int64_t layer = lo;
  while (layer < hi) {
    int64_t span_end = layer + 1;  // exclusive: the layers up to and including the next fence
    while (span_end < hi && !(layer_events && layer_events[span_end - 1 - lo])) ++span_end;
    const int64_t nl = span_end - layer;
    for (const Strip& sp : strips) {
      const Run& r = runs[sp.first];
      const uint8_t* src = pool->host + layer * g.layer_src + r.src;
      uint8_t* dst = l->arena + layer * g.layer_dst + r.dst;
      const auto width = static_cast<size_t>(r.width);
      if (sp.count > 1) {
        for (int64_t ly = 0; ly < nl; ++ly)
          for (int64_t kv = 0; kv < 2; ++kv)
            TSB_CUDA_TRY(cudaMemcpy2DAsync(dst + ly * g.layer_dst + kv * g.kv_dst, static_cast<size_t>(sp.dpitch),
                                           src + ly * g.layer_src + kv * g.kv_src, static_cast<size_t>(sp.spitch),
                                           width, sp.count, cudaMemcpyHostToDevice, l->ce_stream));
      } else if (use_3d) {
        cudaMemcpy3DParms p{};
        p.srcPtr = make_cudaPitchedPtr(const_cast<uint8_t*>(src), static_cast<size_t>(g.kv_src), width,
                                       static_cast<size_t>(g.layer_src / g.kv_src));
        p.dstPtr = make_cudaPitchedPtr(dst, static_cast<size_t>(g.kv_dst), width,
                                       static_cast<size_t>(g.layer_dst / g.kv_dst));
        p.extent = make_cudaExtent(width, 2, static_cast<size_t>(nl));
        p.kind = cudaMemcpyHostToDevice;
        TSB_CUDA_TRY(cudaMemcpy3DAsync(&p, l->ce_stream));
      } else {
        for (int64_t ly = 0; ly < nl; ++ly)
          for (int64_t kv = 0; kv < 2; ++kv)
            TSB_CUDA_TRY(cudaMemcpyAsync(dst + ly * g.layer_dst + kv * g.kv_dst, src + ly * g.layer_src + kv * g.kv_src,
                                         width, cudaMemcpyHostToDevice, l->ce_stream));
      }
    }
    layer = span_end;
    if (layer_events && layer_events[layer - 1 - lo]) TSB_TRY(record_fence(l, layer_events[layer - 1 - lo], l->ce_stream));
  }
  TSB_CUDA_TRY(cudaEventRecord(l->ev_k2_done, l->ce_stream));
  TSB_CUDA_TRY(cudaStreamWaitEvent(st, l->ev_k2_done, 0));
  return TSB_OK;
}

tsb_status ingest_sm(tsb_l1* l, tsb_pool* pool, const tsb_ingest_item* items_dev, int64_t n_items,
                     int64_t lo, int64_t hi, int mode, cudaStream_t st, void* const* layer_events) {
  // One launch per span of layers ending at a requested fence (or at hi): per-layer fences give
  // per-layer launches, a fence only on the first and last layer gives two launches.
  // Host pools are link-bound and saturate with a small grid; HBM / NVLink sources need the
  // HBM grid (4736 CTAs, 4 loads in flight per lane) to keep enough loads in flight.
  const bool on_device = pool->location == TSB_POOL_DEVICE;
  int64_t l0 = lo;
  while (l0 < hi) {
    int64_t l1 = l0 + 1;  // exclusive end of this launch
    if (layer_events)
      while (l1 < hi && !layer_events[l1 - 1 - lo]) ++l1;
    else
      l1 = hi;
    const tsb::IngestGeom g = make_geom(l, l0, l1);
    if (mode == TSB_INGEST_ZEROCOPY) {
      TSB_CUDA_TRY(tsb::launch_ingest_ldg(g, pool->dev, l->arena, items_dev, l->bt_dev, n_items,
                                          on_device ? g_knobs.scatter_ctas : g_knobs.zerocopy_ctas,
                                          st, on_device));
    } else {
      if (g.seg_bytes * 2 > tsb::kBulkSmem)
        return fail(TSB_UNSUPPORTED, "ingest bulk: page segment too large for the smem ring");
      // K1b: one tensor-map TMA load per page segment, NHD or HND (the map does the transpose).
      // From a host pool the link saturates with a small grid; from HBM / NVLink, every SM runs
      // as many rings as its shared memory holds.
      CUtensorMap m;
      tsb::TmaSrc ts{};
      const int64_t C = l->shape.chunk_tokens;
      TSB_TRY(make_segment_map(g, pool->dev, pool->slots * l->shape.layers * 2 * C, &m, &ts, l->shape.layers, C));
      int sms = 148;
      if (on_device) TSB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, l->device));
      TSB_CUDA_TRY(tsb::launch_ingest_tma(m, g, ts, l->arena, items_dev, l->bt_dev, n_items,
                                          on_device ? sms * tsb::tma_ctas_per_sm(g.seg_bytes) : g_knobs.bulk_ctas, st));
    }
    if (layer_events && layer_events[l1 - 1 - lo]) TSB_TRY(record_fence(l, layer_events[l1 - 1 - lo], st));
    l0 = l1;
  }
  return TSB_OK;
}

tsb_status ingest_impl(tsb_l1* l, tsb_pool* pool, const tsb_ingest_item* items_dev,
                       const tsb_ingest_item* items_host, int64_t n_items, int64_t lo, int64_t hi,
                       int mode, cudaStream_t st, void* const* layer_events) {
  if (lo < 0 || hi > l->shape.layers || lo >= hi)
    return fail(TSB_VALIDATION, "ingest: layer range must satisfy 0 <= lo < hi <= layers");
  if (pool->chunk_bytes != make_geom(l, 0, 1).chunk_bytes)
    return fail(TSB_VALIDATION, "ingest: pool chunk geometry differs from the L1 shape");
  mode = resolve_mode(l, pool, mode, items_host, n_items);
  if (n_items == 0) {
    for (int64_t k = 0; layer_events && k < hi - lo; ++k)
      if (layer_events[k]) TSB_TRY(record_fence(l, layer_events[k], st));
    return TSB_OK;
  }
  switch (mode) {
    case TSB_INGEST_ZEROCOPY:
    case TSB_INGEST_BULK:
      return ingest_sm(l, pool, items_dev, n_items, lo, hi, mode, st, layer_events);
    case TSB_INGEST_CE:
      return ingest_ce(l, pool, items_dev, items_host, n_items, lo, hi, st, layer_events);
    case TSB_INGEST_CE_DIRECT:
      return ingest_ce_direct(l, pool, items_host, n_items, lo, hi, st, layer_events);
    default:
      return fail(TSB_VALIDATION, "ingest: unknown mode " + std::to_string(mode));
  }
}

}  // namespace

extern "C" {

tsb_status tsb_l1_copy_chunks(tsb_l1* l, const tsb_page_copy* items, int64_t n_items, int64_t layer_lo,
                              int64_t layer_hi, void* stream) {
  tsb::DeviceGuard dg(l ? l->device : -1);
  if (layer_lo < 0 || layer_hi > l->shape.layers || layer_lo >= layer_hi)
    return fail(TSB_VALIDATION, "copy_chunks: layer range must satisfy 0 <= lo < hi <= layers");
  const int64_t per = static_cast<int64_t>(UploadRing::kSlotBytes / sizeof(tsb_page_copy));
  if (n_items > per) return fail(TSB_VALIDATION, "copy_chunks: at most " + std::to_string(per) + " items per call");
  for (int64_t k = 0; k < n_items; ++k) {
    const tsb_page_copy& it = items[k];
    if (it.src_row < 0 || it.src_row >= l->rows || it.dst_row < 0 || it.dst_row >= l->rows || it.src_chunk < 0 ||
        it.src_chunk >= l->max_chunks || it.dst_chunk < 0 || it.dst_chunk >= l->max_chunks)
      return fail(TSB_VALIDATION, "copy_chunks: item " + std::to_string(k) + " is outside the block table");
  }
  if (n_items == 0) return TSB_OK;
  auto st = static_cast<cudaStream_t>(stream);
  void* dptr = nullptr;
  int slot = 0;
  TSB_TRY(l->ring_items.stage(items, sizeof(tsb_page_copy) * n_items, st, &dptr, &slot));
  const tsb::IngestGeom g = make_geom(l, layer_lo, layer_hi);
  TSB_CUDA_TRY(tsb::launch_page_copy(g, l->arena, static_cast<const tsb_page_copy*>(dptr), l->bt_dev, n_items,
                                     g_knobs.scatter_ctas, st));
  TSB_TRY(l->ring_items.fence(slot, st));
  return TSB_OK;
}

int tsb_ingest_ce_direct_supported(const tsb_l1* l1, const tsb_pool* pool) {
  return l1 && pool && ce_direct_ok(l1, pool) ? 1 : 0;
}

tsb_status tsb_ingest(tsb_l1* l, tsb_pool* pool, const tsb_ingest_item* items, int64_t n_items,
                      int64_t layer_lo, int64_t layer_hi, int mode, void* stream,
                      void* const* layer_events) {
  tsb::DeviceGuard dg(l ? l->device : -1);
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t per = static_cast<int64_t>(UploadRing::kSlotBytes / sizeof(tsb_ingest_item));
  if (n_items > per)
    return fail(TSB_VALIDATION, "ingest: at most " + std::to_string(per) + " items per call");
  // Host items are checked before any device work: an out-of-range slot or row would make the
  // kernels read outside the pool (a sticky fault for the context) instead of failing the call.
  for (int64_t k = 0; k < n_items; ++k) {
    const tsb_ingest_item& it = items[k];
    if (it.src_slot < 0 || it.src_slot >= pool->slots || it.bt_row < 0 || it.bt_row >= l->rows ||
        it.chunk_index < 0 || it.chunk_index >= l->max_chunks)
      return fail(TSB_VALIDATION, "ingest: item " + std::to_string(k) + " (slot " +
                                      std::to_string(it.src_slot) + ", row " + std::to_string(it.bt_row) +
                                      ", chunk " + std::to_string(it.chunk_index) +
                                      ") is outside the pool / block table");
  }
  // The copy engines take one call per run of consecutive pool slots (~4.5 us of copy-engine time
  // per call, repo:profiles/r02_ce_percall_probe.jsonl), and the order of the items inside one
  // call is free (each names its own pages; fences cover the whole call), so host-pool calls that
  // may go through the copy engines are issued in slot order.
  std::vector<tsb_ingest_item> by_slot;
  if (pool->location == TSB_POOL_HOST && n_items > 1 &&
      (mode == TSB_INGEST_AUTO || mode == TSB_INGEST_CE || mode == TSB_INGEST_CE_DIRECT)) {
    bool ordered = true;
    for (int64_t k = 1; k < n_items && ordered; ++k) ordered = items[k].src_slot >= items[k - 1].src_slot;
    if (!ordered) {
      by_slot.assign(items, items + n_items);
      std::stable_sort(by_slot.begin(), by_slot.end(),
                       [](const tsb_ingest_item& x, const tsb_ingest_item& y) { return x.src_slot < y.src_slot; });
      items = by_slot.data();
    }
  }
  void* dptr = nullptr;
  int slot = 0;
  if (n_items > 0)
    TSB_TRY(l->ring_items.stage(items, sizeof(tsb_ingest_item) * n_items, st, &dptr, &slot));
  TSB_TRY(ingest_impl(l, pool, static_cast<const tsb_ingest_item*>(dptr), items, n_items,
                      layer_lo, layer_hi, mode, st, layer_events));
  if (n_items > 0) TSB_TRY(l->ring_items.fence(slot, st));
  return TSB_OK;
}

tsb_status tsb_ingest_tiered(tsb_l1* l, tsb_pool* pool, tsb_pool* hbm_pool,
                             const tsb_ingest_item* items, int64_t n_items, int64_t layer_lo,
                             int64_t layer_hi, int mode, void* stream, void* const* layer_events) {
  tsb::DeviceGuard dg(l ? l->device : -1);
  std::vector<tsb_ingest_item> host, tier;
  for (int64_t k = 0; k < n_items; ++k) {
    if (items[k].src_slot >= 0) {
      host.push_back(items[k]);
    } else {
      if (!hbm_pool)
        return fail(TSB_VALIDATION, "ingest: item " + std::to_string(k) +
                                        " names the HBM tier (negative slot) but none is set");
      tier.push_back(tsb_ingest_item{~items[k].src_slot, items[k].bt_row, items[k].chunk_index});
    }
  }
  if (!pool && !host.empty()) return fail(TSB_VALIDATION, "ingest: host-tier items but no L2 pool");
  if (tier.empty() && host.empty()) {  // nothing to move: the fences are recorded as is
    for (int64_t k = 0; layer_events && k < layer_hi - layer_lo; ++k)
      if (layer_events[k])
        TSB_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(layer_events[k]), static_cast<cudaStream_t>(stream)));
    return TSB_OK;
  }
  if (tier.empty())
    return tsb_ingest(l, pool, host.data(), static_cast<int64_t>(host.size()), layer_lo, layer_hi,
                      mode, stream, layer_events);
  // The HBM tier runs on an internal stream beside the host part (the link never waits for it);
  // the host part's first fence, and everything queued on `stream` after the call, wait for it.
  auto st = static_cast<cudaStream_t>(stream);
  if (!l->tier_stream) {
    TSB_CUDA_TRY(cudaStreamCreateWithFlags(&l->tier_stream, cudaStreamNonBlocking));
    TSB_CUDA_TRY(cudaEventCreateWithFlags(&l->ev_tier_start, cudaEventDisableTiming));
    TSB_CUDA_TRY(cudaEventCreateWithFlags(&l->ev_tier_done, cudaEventDisableTiming));
  }
  TSB_CUDA_TRY(cudaEventRecord(l->ev_tier_start, st));
  TSB_CUDA_TRY(cudaStreamWaitEvent(l->tier_stream, l->ev_tier_start, 0));
  TSB_TRY(tsb_ingest(l, hbm_pool, tier.data(), static_cast<int64_t>(tier.size()), layer_lo, layer_hi,
                     TSB_INGEST_AUTO, l->tier_stream, nullptr));
  TSB_CUDA_TRY(cudaEventRecord(l->ev_tier_done, l->tier_stream));
  if (host.empty()) {  // every chunk came from the tier: the fences only wait for it
    TSB_CUDA_TRY(cudaStreamWaitEvent(st, l->ev_tier_done, 0));
    for (int64_t k = 0; layer_events && k < layer_hi - layer_lo; ++k)
      if (layer_events[k]) TSB_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(layer_events[k]), st));
    return TSB_OK;
  }
  l->fence_dep = l->ev_tier_done;
  const tsb_status hs = tsb_ingest(l, pool, host.data(), static_cast<int64_t>(host.size()), layer_lo,
                                   layer_hi, mode, stream, layer_events);
  l->fence_dep = nullptr;
  TSB_TRY(hs);
  TSB_CUDA_TRY(cudaStreamWaitEvent(st, l->ev_tier_done, 0));
  return TSB_OK;
}

tsb_status tsb_ingest_device(tsb_l1* l, tsb_pool* pool, const tsb_ingest_item* items_dev,
                             int64_t n_items, int64_t layer_lo, int64_t layer_hi, int mode,
                             void* stream, void* const* layer_events) {
  tsb::DeviceGuard dg(l ? l->device : -1);
  return ingest_impl(l, pool, items_dev, nullptr, n_items, layer_lo, layer_hi, mode,
                     static_cast<cudaStream_t>(stream), layer_events);
}

tsb_status tsb_ingest_resolve_mode(const tsb_l1* l, const tsb_pool* pool,
                                   const tsb_ingest_item* items, int64_t n_items, int mode,
                                   int* resolved) {
  if (mode < TSB_INGEST_AUTO || mode > TSB_INGEST_CE_DIRECT)
    return fail(TSB_VALIDATION, "ingest: unknown mode " + std::to_string(mode));
  *resolved = resolve_mode(l, pool, mode, items, n_items);
  return TSB_OK;
}

tsb_status tsb_l1_set_ce_group_bytes(tsb_l1* l, int64_t bytes) {
  if (!l) return fail(TSB_VALIDATION, "l1_set_ce_group_bytes: null L1");
  if (bytes < 0) return fail(TSB_VALIDATION, "l1_set_ce_group_bytes: bytes must be >= 0");
  l->group_cap = bytes;
  return TSB_OK;
}

int64_t tsb_l1_ce_group_bytes(const tsb_l1* l) { return l ? l->group_cap : 0; }

tsb_status tsb_ingest_set_ce(int variant, int64_t staging_bytes) {
  if (variant < 0 || variant > 1) return fail(TSB_VALIDATION, "ingest_set_ce: variant must be 0 or 1");
  g_knobs.ce_variant = variant;
  g_knobs.staging_bytes = staging_bytes > 0 ? staging_bytes : (1ll << 30);
  return TSB_OK;
}

tsb_status tsb_scatter_device(tsb_l1* l, const void* staging, const tsb_ingest_item* items_dev,
                              int64_t n_items, int64_t layer_lo, int64_t layer_hi,
                              void* stream) {
  tsb::DeviceGuard dg(l ? l->device : -1);
  if (layer_lo < 0 || layer_hi > l->shape.layers || layer_lo >= layer_hi)
    return fail(TSB_VALIDATION, "scatter: layer range must satisfy 0 <= lo < hi <= layers");
  tsb::IngestGeom g = make_geom(l, layer_lo, layer_hi);
  g.staged = 1;  // item i's layers [lo, hi) at staging + i * (hi - lo) * layer bytes
  g.item_stride = (layer_hi - layer_lo) * g.layer_src;
  TSB_TRY(launch_scatter(g, static_cast<const uint8_t*>(staging), l->arena, items_dev, l->bt_dev, n_items,
                         static_cast<cudaStream_t>(stream), l->device));
  return TSB_OK;
}

tsb_status tsb_scatter_device_packed(tsb_l1* l, const void* staging,
                                     const tsb_ingest_item* items_dev, int64_t n_items,
                                     int64_t layer_lo, int64_t layer_hi, void* stream) {
  tsb::DeviceGuard dg(l ? l->device : -1);
  if (layer_lo < 0 || layer_hi > l->shape.layers || layer_lo >= layer_hi)
    return fail(TSB_VALIDATION, "scatter: layer range must satisfy 0 <= lo < hi <= layers");
  const tsb::IngestGeom g = make_staged_geom(l, layer_lo, layer_hi - layer_lo);
  TSB_TRY(launch_scatter(g, static_cast<const uint8_t*>(staging), l->arena, items_dev, l->bt_dev, n_items,
                         static_cast<cudaStream_t>(stream), l->device));
  return TSB_OK;
}

tsb_status tsb_l1_verify_synthetic(tsb_l1* l, const tsb_ingest_item* items, int64_t n_items,
                                   int64_t layer_lo, int64_t layer_hi, uint64_t seed,
                                   int64_t pool_chunk_bytes, void* stream,
                                   uint64_t* mismatches) {
  tsb::DeviceGuard dg(l ? l->device : -1);
  // Independent of the ingest address math (verify.cu): invert the host block table into
  // page -> (slot, first token), then check every word of those pages from the layout definition.
  auto st = static_cast<cudaStream_t>(stream);
  const tsb_kv_shape& sh = l->shape;
  const int64_t L = sh.layers;
  if (layer_lo < 0 || layer_hi > L || layer_lo > layer_hi)
    return fail(TSB_VALIDATION, "verify: layer range out of bounds");
  if (pool_chunk_bytes != L * 2 * sh.chunk_tokens * sh.kv_heads * sh.head_dim * sh.dtype_bytes)
    return fail(TSB_VALIDATION, "verify: pool chunk bytes differ from the L1 shape");
  tsb::PageCheck c{};
  c.H = sh.kv_heads;
  c.Hl = sh.kv_heads / sh.tp_size;
  c.D = sh.head_dim;
  c.E = sh.dtype_bytes;
  c.C = sh.chunk_tokens;
  c.P = sh.page_tokens;
  c.tp_rank = sh.tp_rank;
  c.num_pages = l->num_pages;
  c.pool_chunk_bytes = pool_chunk_bytes;
  c.layout = l->layout;
  c.layer_lo = static_cast<int32_t>(layer_lo);
  c.layer_hi = static_cast<int32_t>(layer_hi);
  std::vector<tsb::PageSource> pages;
  pages.reserve(static_cast<size_t>(n_items * l->ppc));
  std::vector<uint8_t> seen(static_cast<size_t>(l->num_pages), 0);
  uint64_t host_bad = 0;
  const int64_t words_per_page = (layer_hi - layer_lo) * 2 * c.P * c.Hl * c.D * c.E / 8;
  for (int64_t i = 0; i < n_items; ++i) {
    const tsb_ingest_item& it = items[i];
    if (it.bt_row < 0 || it.bt_row >= l->rows || it.chunk_index < 0 || it.chunk_index >= l->max_chunks) {
      host_bad += static_cast<uint64_t>(l->ppc * words_per_page);
      continue;
    }
    for (int64_t j = 0; j < l->ppc; ++j) {
      const int32_t page = l->bt_host[it.bt_row * l->stride + it.chunk_index * l->ppc + j];
      if (page < 0 || page >= l->num_pages || seen[static_cast<size_t>(page)]) {
        host_bad += static_cast<uint64_t>(words_per_page);  // unmapped or shared page: all wrong
        continue;
      }
      seen[static_cast<size_t>(page)] = 1;
      pages.push_back(tsb::PageSource{it.src_slot, page, static_cast<int32_t>(j * c.P)});
    }
  }
  TSB_CUDA_TRY(cudaMemsetAsync(l->verify_ctr, 0, sizeof(unsigned long long), st));
  const int64_t per = static_cast<int64_t>(UploadRing::kSlotBytes / sizeof(tsb::PageSource));
  for (int64_t p0 = 0; p0 < static_cast<int64_t>(pages.size()); p0 += per) {
    const int64_t n = std::min<int64_t>(per, static_cast<int64_t>(pages.size()) - p0);
    void* dptr = nullptr;
    int slot = 0;
    TSB_TRY(l->ring_items.stage(pages.data() + p0, sizeof(tsb::PageSource) * n, st, &dptr, &slot));
    TSB_CUDA_TRY(tsb::launch_verify_pages(c, l->arena, static_cast<const tsb::PageSource*>(dptr), n, seed,
                                          l->verify_ctr, st));
    TSB_TRY(l->ring_items.fence(slot, st));
  }
  unsigned long long h = 0;
  TSB_CUDA_TRY(cudaMemcpyAsync(&h, l->verify_ctr, sizeof(h), cudaMemcpyDeviceToHost, st));
  TSB_CUDA_TRY(cudaStreamSynchronize(st));
  *mismatches = h + host_bad;
  return TSB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// Standalone TierLedger (engine.hpp:22-53) over the same tsb::Ledger the L1 allocator uses.
// ---------------------------------------------------------------------------------------
struct tsb_ledger {
  tsb::Ledger l;
};

extern "C" {

tsb_status tsb_ledger_create(int tier, int64_t capacity, tsb_ledger** out) {
  if (capacity <= 0) return fail(TSB_VALIDATION, "TierLedger: capacity must be > 0");
  *out = new tsb_ledger{tsb::Ledger(tier, capacity)};
  return TSB_OK;
}

void tsb_ledger_destroy(tsb_ledger* l) { delete l; }

tsb_status tsb_ledger_request(tsb_ledger* l, int64_t request_id, int32_t block_index,
                              int64_t bytes, int* granted) {
  std::string msg;
  bool ok = false;
  const tsb_status st = l->l.request(request_id, block_index, bytes, &ok, &msg);
  if (st != TSB_OK) return fail(st, msg);
  *granted = ok ? 1 : 0;
  return TSB_OK;
}

tsb_status tsb_ledger_release(tsb_ledger* l, int64_t bytes, tsb_grant* out, int64_t cap,
                              int64_t* n) {
  std::string msg;
  *n = 0;
  const tsb_status st = l->l.release(
      bytes,
      [&](const tsb::Ledger::Pending& p) {
        if (*n < cap) out[*n] = tsb_grant{p.request_id, p.block_index, -1, p.bytes};
        ++*n;
      },
      &msg);
  if (st != TSB_OK) return fail(st, msg);
  return TSB_OK;
}

int64_t tsb_ledger_reserved(const tsb_ledger* l) { return l->l.reserved(); }
int64_t tsb_ledger_capacity(const tsb_ledger* l) { return l->l.capacity(); }
int64_t tsb_ledger_deferred(const tsb_ledger* l) { return l->l.deferred(); }

}  // extern "C"
