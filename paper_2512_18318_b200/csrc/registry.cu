// registry.cu -- zero-copy stage hand-off.
//
// The reference moves every payload through its wire codecs by value
// (stage.cpp:176-301: WireWriter::samples copies each int16, decode copies
// them back) and has no pixels to move at all (AlignedPairMsg,
// stage.hpp:81-93, carries counts).  On the GPU the payloads -- segment PCM
// in the segmenter's stream buffers, mel rows, face crops, rendered frames --
// already live in HBM; stages hand them on as references into this registry
// and only the 48-byte reference crosses the message bus.
//
// Device side: one arena per registry (cudaMalloc once, at create).
// Host side: a (uuid, kind) index, a first-fit free list with coalescing, and
// stream-ordered reuse -- a released block is parked with an event recorded
// on the context stream and only returns to the free list once that event has
// completed, so kernels still reading the old contents are never overwritten.
#include <cstring>
#include <map>
#include <unordered_map>
#include <vector>

#include "lsg_common.cuh"

namespace {

using lsg::Ctx;
using lsg::DevBuf;

constexpr int64_t kGranule = 256;  // allocation alignment (TMA / vector loads)

struct Key {
  uint8_t uuid[16];
  int32_t kind;
  bool operator==(const Key& o) const { return kind == o.kind && std::memcmp(uuid, o.uuid, 16) == 0; }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    uint64_t a, b;
    std::memcpy(&a, k.uuid, 8);
    std::memcpy(&b, k.uuid + 8, 8);
    uint64_t h = a * 0x9E3779B97F4A7C15ull ^ (b + 0x632BE59BD9B4E019ull + (uint64_t)k.kind);
    h ^= h >> 31;
    return (size_t)(h * 0xBF58476D1CE4E5B9ull);
  }
};

struct Entry {
  int64_t off = -1;  // arena offset, -1 = adopted view
  int64_t bytes = 0;
  int64_t span = 0;  // arena bytes held (granule multiple)
  const void* view = nullptr;
  int32_t refs = 1;
  uint64_t gen = 0;
};

struct Parked {
  int64_t off, span;
  cudaEvent_t done;
};

}  // namespace

struct lsg_reg_s {
  Ctx* ctx = nullptr;
  DevBuf<uint8_t> arena;
  int64_t cap = 0;
  std::map<int64_t, int64_t> free_;  // offset -> span, coalesced, ready for reuse
  std::vector<Parked> parked;        // released, waiting for their stream event
  std::vector<cudaEvent_t> spare_events;
  std::unordered_map<Key, Entry, KeyHash> index;
  uint64_t next_gen = 1;
  int64_t used = 0, peak = 0;

  void give_back(int64_t off, int64_t span) {
    auto it = free_.emplace(off, span).first;
    if (it != free_.begin()) {  // merge with the block before
      auto prev = std::prev(it);
      if (prev->first + prev->second == off) {
        prev->second += span;
        free_.erase(it);
        it = prev;
      }
    }
    auto next = std::next(it);
    if (next != free_.end() && it->first + it->second == next->first) {
      it->second += next->second;
      free_.erase(next);
    }
  }

  // Parked blocks whose stream work has completed go back to the free list;
  // with `wait`, the oldest parked block is waited for if none has.
  bool reclaim(bool wait) {
    bool any = false;
    for (size_t i = 0; i < parked.size();) {
      const cudaError_t q = cudaEventQuery(parked[i].done);
      if (q == cudaSuccess) {
        give_back(parked[i].off, parked[i].span);
        spare_events.push_back(parked[i].done);
        parked.erase(parked.begin() + (std::ptrdiff_t)i);
        any = true;
      } else if (q == cudaErrorNotReady) {
        ++i;
      } else {
        LSG_CUDA(q);
      }
    }
    if (!any && wait && !parked.empty()) {
      LSG_CUDA(cudaEventSynchronize(parked.front().done));
      return reclaim(false);
    }
    return any;
  }

  int64_t first_fit(int64_t span) {
    for (auto it = free_.begin(); it != free_.end(); ++it) {
      if (it->second < span) continue;
      const int64_t off = it->first, rest = it->second - span;
      free_.erase(it);
      if (rest) free_.emplace(off + span, rest);
      return off;
    }
    return -1;
  }

  int64_t allocate(int64_t bytes) {
    const int64_t span = std::max<int64_t>(kGranule, (bytes + kGranule - 1) / kGranule * kGranule);
    int64_t off = first_fit(span);
    while (off < 0 && !parked.empty()) {
      reclaim(true);
      off = first_fit(span);
    }
    if (off < 0)
      lsg::fail(LSG_ERUNTIME, "registry: arena exhausted (" + std::to_string(bytes) + " bytes requested, " +
                                  std::to_string(cap - used) + " of " + std::to_string(cap) + " free)");
    used += span;
    peak = std::max(peak, used);
    return off;
  }

  void park(int64_t off, int64_t span) {
    cudaEvent_t ev;
    if (!spare_events.empty()) {
      ev = spare_events.back();
      spare_events.pop_back();
    } else {
      LSG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    LSG_CUDA(cudaEventRecord(ev, ctx->stream));
    parked.push_back({off, span, ev});
    used -= span;
  }

  Entry& lookup(const lsg_devref* ref) {
    Key k;
    std::memcpy(k.uuid, ref->uuid, 16);
    k.kind = ref->kind;
    auto it = index.find(k);
    if (it == index.end() || it->second.gen != ref->generation)
      lsg::logic("registry: unknown or stale reference (kind " + std::to_string(ref->kind) + ", generation " +
                 std::to_string(ref->generation) + ")");
    return it->second;
  }

  void* pointer(const Entry& e) const {
    return e.off >= 0 ? (void*)(arena.p + e.off) : const_cast<void*>(e.view);
  }

  // Validates a new key before any arena space is taken.
  void check_new(const uint8_t* uuid16, int32_t kind) const {
    if (kind < LSG_BUF_AUDIO || kind > LSG_BUF_RENDER) lsg::invalid("registry: bad buffer kind");
    Key k;
    std::memcpy(k.uuid, uuid16, 16);
    k.kind = kind;
    if (index.count(k)) lsg::logic("registry: (uuid, kind) already registered");
  }

  lsg_devref insert(const uint8_t* uuid16, int32_t kind, Entry e) {
    Key k;
    std::memcpy(k.uuid, uuid16, 16);
    k.kind = kind;
    e.gen = next_gen++;
    index.emplace(k, e);
    lsg_devref r{};
    std::memcpy(r.uuid, uuid16, 16);
    r.kind = kind;
    r.device = ctx->device;
    r.generation = e.gen;
    r.offset = e.off;
    r.bytes = e.bytes;
    return r;
  }

  ~lsg_reg_s() {
    for (auto& p : parked) cudaEventDestroy(p.done);
    for (auto ev : spare_events) cudaEventDestroy(ev);
  }
};

namespace {

void need(const void* p, const char* what) {
  if (!p) lsg::invalid(std::string("registry: null ") + what);
}

}  // namespace

extern "C" {

lsg_status lsg_reg_create(lsg_ctx ctx, int64_t arena_bytes, lsg_reg* out) {
  return lsg::guard(__func__, [&] {
    need(ctx, "context");
    need(out, "output handle");
    if (arena_bytes < kGranule) lsg::invalid("registry: arena must hold at least 256 bytes");
    lsg::DeviceGuard g(ctx);
    auto r = new lsg_reg_s();
    try {
      r->ctx = ctx;
      r->cap = (arena_bytes + kGranule - 1) / kGranule * kGranule;
      r->arena.alloc((size_t)r->cap);
      r->free_.emplace(0, r->cap);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

lsg_status lsg_reg_destroy(lsg_reg r) {
  return lsg::guard(__func__, [&] {
    if (!r) return;
    lsg::DeviceGuard g(r->ctx);
    r->ctx->sync();  // queued readers of the arena finish first
    delete r;
  });
}

lsg_status lsg_reg_put(lsg_reg r, const uint8_t* uuid16, int32_t kind, const void* src, int64_t bytes,
                       lsg_devref* ref) {
  return lsg::guard(__func__, [&] {
    need(r, "registry");
    need(uuid16, "uuid");
    need(ref, "reference");
    if (bytes < 0 || (bytes > 0 && !src)) lsg::invalid("registry: bad source range");
    lsg::DeviceGuard g(r->ctx);
    r->check_new(uuid16, kind);
    Entry e;
    e.bytes = bytes;
    e.off = r->allocate(bytes);
    e.span = std::max<int64_t>(kGranule, (bytes + kGranule - 1) / kGranule * kGranule);
    *ref = r->insert(uuid16, kind, e);
    if (bytes) LSG_CUDA(cudaMemcpyAsync(r->arena.p + e.off, src, (size_t)bytes, cudaMemcpyDefault, r->ctx->stream));
  });
}

lsg_status lsg_reg_put_view(lsg_reg r, const uint8_t* uuid16, int32_t kind, const void* dev_ptr, int64_t bytes,
                            lsg_devref* ref) {
  return lsg::guard(__func__, [&] {
    need(r, "registry");
    need(uuid16, "uuid");
    need(ref, "reference");
    if (bytes < 0 || (bytes > 0 && !dev_ptr)) lsg::invalid("registry: bad view range");
    lsg::DeviceGuard g(r->ctx);
    if (bytes > 0 && !lsg::is_device_ptr(dev_ptr)) lsg::invalid("registry: put_view needs device memory");
    r->check_new(uuid16, kind);
    Entry e;
    e.bytes = bytes;
    e.view = dev_ptr;
    *ref = r->insert(uuid16, kind, e);
  });
}

lsg_status lsg_reg_alloc(lsg_reg r, const uint8_t* uuid16, int32_t kind, int64_t bytes, void** dev_ptr,
                         lsg_devref* ref) {
  return lsg::guard(__func__, [&] {
    need(r, "registry");
    need(uuid16, "uuid");
    need(ref, "reference");
    need(dev_ptr, "pointer output");
    if (bytes < 0) lsg::invalid("registry: negative size");
    lsg::DeviceGuard g(r->ctx);
    r->check_new(uuid16, kind);
    Entry e;
    e.bytes = bytes;
    e.off = r->allocate(bytes);
    e.span = std::max<int64_t>(kGranule, (bytes + kGranule - 1) / kGranule * kGranule);
    *ref = r->insert(uuid16, kind, e);
    *dev_ptr = r->arena.p + e.off;
  });
}

lsg_status lsg_reg_resolve(lsg_reg r, const lsg_devref* ref, void** dev_ptr, int64_t* bytes) {
  return lsg::guard(__func__, [&] {
    need(r, "registry");
    need(ref, "reference");
    if (ref->device != r->ctx->device) lsg::logic("registry: reference belongs to another device");
    const Entry& e = r->lookup(ref);
    if (dev_ptr) *dev_ptr = r->pointer(e);
    if (bytes) *bytes = e.bytes;
  });
}

lsg_status lsg_reg_find(lsg_reg r, const uint8_t* uuid16, int32_t kind, lsg_devref* ref) {
  return lsg::guard(__func__, [&] {
    need(r, "registry");
    need(uuid16, "uuid");
    need(ref, "reference");
    Key k;
    std::memcpy(k.uuid, uuid16, 16);
    k.kind = kind;
    auto it = r->index.find(k);
    if (it == r->index.end()) lsg::logic("registry: no buffer for (uuid, kind)");
    const Entry& e = it->second;
    std::memset(ref, 0, sizeof(*ref));
    std::memcpy(ref->uuid, uuid16, 16);
    ref->kind = kind;
    ref->device = r->ctx->device;
    ref->generation = e.gen;
    ref->offset = e.off;
    ref->bytes = e.bytes;
  });
}

lsg_status lsg_reg_retain(lsg_reg r, const lsg_devref* ref) {
  return lsg::guard(__func__, [&] {
    need(r, "registry");
    need(ref, "reference");
    r->lookup(ref).refs++;
  });
}

lsg_status lsg_reg_release(lsg_reg r, const lsg_devref* ref) {
  return lsg::guard(__func__, [&] {
    need(r, "registry");
    need(ref, "reference");
    lsg::DeviceGuard g(r->ctx);
    Entry& e = r->lookup(ref);
    if (--e.refs > 0) return;
    if (e.off >= 0) r->park(e.off, e.span);
    Key k;
    std::memcpy(k.uuid, ref->uuid, 16);
    k.kind = ref->kind;
    r->index.erase(k);
    r->reclaim(false);
  });
}

lsg_status lsg_reg_stats(lsg_reg r, int64_t* used, int64_t* entries, int64_t* peak) {
  return lsg::guard(__func__, [&] {
    need(r, "registry");
    if (used) *used = r->used;
    if (entries) *entries = (int64_t)r->index.size();
    if (peak) *peak = r->peak;
  });
}

// Little-endian, field order of the struct (WireWriter::u32/i64 conventions,
// stage.cpp:38-49): uuid[16] kind u32 device u32 generation u64 offset i64 bytes i64.
lsg_status lsg_devref_encode(const lsg_devref* ref, uint8_t* out) {
  return lsg::guard(__func__, [&] {
    need(ref, "reference");
    need(out, "output");
    auto put = [&](int at, uint64_t v, int n) {
      for (int i = 0; i < n; ++i) out[at + i] = (uint8_t)(v >> (8 * i));
    };
    std::memcpy(out, ref->uuid, 16);
    put(16, (uint32_t)ref->kind, 4);
    put(20, (uint32_t)ref->device, 4);
    put(24, ref->generation, 8);
    put(32, (uint64_t)ref->offset, 8);
    put(40, (uint64_t)ref->bytes, 8);
  });
}

lsg_status lsg_devref_decode(const uint8_t* in, lsg_devref* ref) {
  return lsg::guard(__func__, [&] {
    need(in, "input");
    need(ref, "reference");
    auto get = [&](int at, int n) {
      uint64_t v = 0;
      for (int i = 0; i < n; ++i) v |= (uint64_t)in[at + i] << (8 * i);
      return v;
    };
    std::memcpy(ref->uuid, in, 16);
    ref->kind = (int32_t)get(16, 4);
    ref->device = (int32_t)get(20, 4);
    ref->generation = get(24, 8);
    ref->offset = (int64_t)get(32, 8);
    ref->bytes = (int64_t)get(40, 8);
  });
}

}  // extern "C"
