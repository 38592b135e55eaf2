// pstereo/gpu_runtime.hpp -- the device side of the drop-in headers: which
// CUDA device a call runs on, and the per-thread cache of library contexts
// (include/pstereo_gpu.h: one context per device and host thread, not
// re-entrant). Not a reference header; the reference's headers that this
// tree replaces include it.
//
//   pstereo::gpu::set_device(d)   pin the calling thread's calls to device d
//                                 (default: the thread's current CUDA device)
//   pstereo::gpu::clear_contexts() free the calling thread's contexts
#pragma once

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <map>
#include <memory>
#include <string>
#include <utility>

#include "config.hpp"
#include "errors.hpp"
#include "../pstereo_gpu.h"

namespace pstereo {
namespace gpu {

// failures the reference has no type for (CUDA errors, no sm_100 device)
struct GpuError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {

[[noreturn]] inline void raise(int code, const std::string& msg) {
  if (code == PSTEREO_ECONFIG) throw ConfigError(msg);
  if (code == PSTEREO_EDEGENERATE) throw DegenerateInputError(msg);
  if (code == PSTEREO_EIO) {
    const int k = pstereo_last_io_kind();
    throw IoError(k >= 0 && k <= 3 ? IoErrorKind(k) : IoErrorKind::decode_failure, msg);
  }
  throw GpuError(msg);
}

inline int& device_pin() {
  thread_local int d = -1;
  return d;
}

struct CtxDeleter {
  void operator()(pstereo_ctx* c) const { pstereo_gpu_destroy(c); }
};

struct CtxSlot {
  std::unique_ptr<pstereo_ctx, CtxDeleter> ctx;
  int w = 0, h = 0, n = 0;  // capacity
};

inline std::map<std::pair<int, std::string>, CtxSlot>& ctx_cache() {
  thread_local std::map<std::pair<int, std::string>, CtxSlot> cache;
  return cache;
}

}  // namespace detail

inline void set_device(int device) { detail::device_pin() = device; }

inline int device() {
  if (detail::device_pin() >= 0) return detail::device_pin();
  int d = 0;
  if (pstereo_gpu_current_device(&d) != PSTEREO_OK) throw GpuError("no CUDA device");
  return d;
}

inline void clear_contexts() { detail::ctx_cache().clear(); }

namespace detail {

// The calling thread's context for these params on the current device, with
// room for n pairs of w x h. One context per (device, params); it grows (is
// re-created larger) when a call needs more, so varying batch or image sizes
// reuse one context instead of accumulating them.
inline pstereo_ctx* context_for(const pstereo_params& p, int w, int h, int n) {
  const int dev = device();
  CtxSlot& slot = ctx_cache()[{dev, std::string(reinterpret_cast<const char*>(&p), sizeof p)}];
  if (!slot.ctx || w > slot.w || h > slot.h || n > slot.n) {
    const int cw = std::max(w, slot.w), ch = std::max(h, slot.h), cn = std::max(n, slot.n);
    slot.ctx.reset();
    pstereo_ctx* c = nullptr;
    const int rc = pstereo_gpu_create(dev, &p, cw, ch, cn, &c);
    if (rc != PSTEREO_OK) {
      char msg[256] = {0};
      if (rc == PSTEREO_ECONFIG) pstereo_validate(&p, msg, sizeof msg);
      raise(rc, rc == PSTEREO_ECONFIG ? msg : "pstereo_gpu_create failed on device " +
                                                  std::to_string(dev));
    }
    slot.ctx.reset(c);
    slot.w = cw;
    slot.h = ch;
    slot.n = cn;
  }
  return slot.ctx.get();
}

}  // namespace detail
}  // namespace gpu
}  // namespace pstereo
