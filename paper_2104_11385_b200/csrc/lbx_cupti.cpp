// CUPTI activity-record timer: the fourth cost strategy.
//
// The paper's "Timers" strategy reads per-box kernel durations from CUPTI
// activity records (modeled by the reference as
// the `instrumented` provider with overhead_factor 2.0, cost.py:208-213).
// LBX_COST_TIMERS reproduces it with CUDA events around each per-box launch;
// LBX_COST_CUPTI uses the real mechanism: the same per-box launches, with
// CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL records supplying the GPU start/end
// timestamps (ns) of every `timers_push_kernel` on the run's stream.
//
// libcupti is opened with dlopen on first use, so libLBX loads (and every
// other strategy runs) on hosts without it.  CUPTI's activity callbacks are
// process-global: the records are filtered by kernel name and stream id and
// handed out in GPU start order -- one stream executes its launches in
// issue order, so the k-th record of a step is the k-th non-empty box.
#include <cupti.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "lbx_internal.h"

namespace lbx {
namespace {

using FnRegister = CUptiResult (*)(CUpti_BuffersCallbackRequestFunc, CUpti_BuffersCallbackCompleteFunc);
using FnKind = CUptiResult (*)(CUpti_ActivityKind);
using FnFlush = CUptiResult (*)(uint32_t);
using FnNext = CUptiResult (*)(uint8_t*, size_t, CUpti_Activity**);
using FnStream = CUptiResult (*)(CUcontext, CUstream, uint8_t, uint32_t*);
using FnDropped = CUptiResult (*)(CUcontext, uint32_t, size_t*);

struct Span {
  uint32_t stream;
  uint64_t start, end;
};

struct Cupti {
  std::mutex mu;
  void* dl = nullptr;
  bool loaded = false, registered = false;
  int users = 0;
  FnRegister reg = nullptr;
  FnKind enable = nullptr, disable = nullptr;
  FnFlush flush = nullptr;
  FnNext next = nullptr;
  FnStream stream_id = nullptr;
  FnDropped dropped = nullptr;
  std::vector<Span> spans;  // completed timers_push_kernel records, not yet collected
};

Cupti& g() {
  static Cupti c;
  return c;
}

constexpr size_t kBufBytes = 1 << 20;
constexpr uint32_t kAnyStream = 0xffffffffu;

void CUPTIAPI buffer_requested(uint8_t** buf, size_t* size, size_t* max_records) {
  *buf = static_cast<uint8_t*>(std::aligned_alloc(8, kBufBytes));
  *size = *buf ? kBufBytes : 0;
  *max_records = 0;
}

void CUPTIAPI buffer_completed(CUcontext, uint32_t, uint8_t* buf, size_t, size_t valid) {
  Cupti& c = g();
  std::vector<Span> got;
  CUpti_Activity* rec = nullptr;
  while (c.next(buf, valid, &rec) == CUPTI_SUCCESS) {
    if (rec->kind != CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL && rec->kind != CUPTI_ACTIVITY_KIND_KERNEL)
      continue;
    const auto* k = reinterpret_cast<const CUpti_ActivityKernel9*>(rec);
    if (k->name && std::strstr(k->name, "timers_push_kernel"))
      got.push_back(Span{k->streamId, k->start, k->end});
  }
  std::free(buf);
  std::lock_guard<std::mutex> lock(c.mu);
  c.spans.insert(c.spans.end(), got.begin(), got.end());
}

template <class F>
bool sym(void* dl, const char* name, F* out) {
  *out = reinterpret_cast<F>(dlsym(dl, name));
  return *out != nullptr;
}

}  // namespace

int cupti_acquire() {
  Cupti& c = g();
  std::lock_guard<std::mutex> lock(c.mu);
  if (!c.loaded) {
    for (const char* lib : {"libcupti.so.12", "libcupti.so", "/usr/local/cuda/lib64/libcupti.so.12"}) {
      c.dl = dlopen(lib, RTLD_NOW | RTLD_LOCAL);
      if (c.dl) break;
    }
    if (!c.dl) return set_error(LBX_EINVAL, "CUPTI strategy: libcupti not found (%s)", dlerror());
    if (!sym(c.dl, "cuptiActivityRegisterCallbacks", &c.reg) ||
        !sym(c.dl, "cuptiActivityEnable", &c.enable) ||
        !sym(c.dl, "cuptiActivityDisable", &c.disable) ||
        !sym(c.dl, "cuptiActivityFlushAll", &c.flush) ||
        !sym(c.dl, "cuptiActivityGetNextRecord", &c.next) ||
        !sym(c.dl, "cuptiGetStreamIdEx", &c.stream_id))
      return set_error(LBX_EINVAL, "CUPTI strategy: libcupti lacks the activity API");
    sym(c.dl, "cuptiActivityGetNumDroppedRecords", &c.dropped);
    c.loaded = true;
  }
  if (!c.registered) {
    if (c.reg(buffer_requested, buffer_completed) != CUPTI_SUCCESS)
      return set_error(LBX_EINVAL, "CUPTI strategy: cuptiActivityRegisterCallbacks failed "
                                   "(another CUPTI client in this process?)");
    c.registered = true;
  }
  if (c.users == 0 && c.enable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL) != CUPTI_SUCCESS)
    return set_error(LBX_EINVAL, "CUPTI strategy: cannot enable kernel activity records");
  ++c.users;
  return LBX_OK;
}

void cupti_release() {
  Cupti& c = g();
  bool last = false;
  {
    std::lock_guard<std::mutex> lock(c.mu);
    if (c.users == 0) return;
    last = --c.users == 0;
  }
  if (last) {
    c.flush(CUPTI_ACTIVITY_FLAG_FLUSH_FORCED);
    c.disable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL);
    std::lock_guard<std::mutex> lock(c.mu);
    c.spans.clear();
  }
}

// CUPTI's id of `stream`, or kAnyStream when CUPTI cannot name it (the
// legacy default stream): then every timers_push_kernel record counts.
int cupti_stream(void* stream, uint32_t* id) {
  Cupti& c = g();
  if (!c.loaded) return set_error(LBX_EINVAL, "CUPTI strategy not initialised");
  if (!stream || c.stream_id(nullptr, static_cast<CUstream>(stream), 0, id) != CUPTI_SUCCESS)
    *id = kAnyStream;
  return LBX_OK;
}

// Durations (ns) of the next `n` timers_push_kernel launches on `stream_id`,
// in GPU start order.  The caller has synchronised the stream, so every
// record of the step exists; the forced flush delivers them.
int cupti_collect(uint32_t stream_id, int n, double* dur_ns) {
  Cupti& c = g();
  if (c.flush(CUPTI_ACTIVITY_FLAG_FLUSH_FORCED) != CUPTI_SUCCESS)
    return set_error(LBX_EINVAL, "CUPTI strategy: cuptiActivityFlushAll failed");
  std::lock_guard<std::mutex> lock(c.mu);
  std::vector<Span> mine, rest;
  for (const Span& s : c.spans)
    (stream_id == kAnyStream || s.stream == stream_id ? mine : rest).push_back(s);
  if ((int)mine.size() < n) {
    size_t lost = 0;
    if (c.dropped) c.dropped(nullptr, 0, &lost);
    return set_error(LBX_EINVAL, "CUPTI strategy: %d of %d per-box kernel records (%zu dropped)",
                     (int)mine.size(), n, lost);
  }
  std::stable_sort(mine.begin(), mine.end(),
                   [](const Span& a, const Span& b) { return a.start < b.start; });
  for (int i = 0; i < n; ++i) dur_ns[i] = (double)(mine[i].end - mine[i].start);
  rest.insert(rest.end(), mine.begin() + n, mine.end());
  c.spans.swap(rest);
  return LBX_OK;
}

}  // namespace lbx
