// bdis_multi.cpp -- pair sharding over several devices, host
// C++ over the C ABI: one context and one persistent host thread per device
// entry, contiguous pair blocks, no collective. This is the B200 counterpart
// of the reference's only parallelism, parallel_patches
// (src/coarse_to_fine.cpp:184-205), moved from patches to whole pairs: pairs
// are independent, so each device uploads, matches and downloads its own
// block and nothing crosses between devices.
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pstereo_gpu.h"

namespace {

struct Job {
  int n = 0, w = 0, h = 0, c = 0;
  const uint8_t* left = nullptr;
  const uint8_t* right = nullptr;
  double focal = 1.0, baseline = 1.0;
  pstereo_outputs out{};
};

struct Worker {
  int device = 0;
  pstereo_ctx* ctx = nullptr;
  std::thread thread;
  // mailbox, guarded by the owner's mutex
  bool has_job = false;
  Job job;
  int rc = PSTEREO_OK;
  double ms = 0.0;
  std::string err;
};

}  // namespace

struct pstereo_multi {
  std::vector<std::unique_ptr<Worker>> workers;
  std::mutex mu;
  std::condition_variable cv_job, cv_done;
  int pending = 0;
  bool quit = false;
  pstereo_params params{};
  std::string err;

  void loop(Worker* wk) {
    for (;;) {
      Job job;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_job.wait(lk, [&] { return quit || wk->has_job; });
        if (quit) return;
        job = wk->job;
      }
      const auto t0 = std::chrono::steady_clock::now();
      int rc = PSTEREO_OK;
      std::string msg;
      if (job.n > 0) {
        rc = pstereo_gpu_match_u8(wk->ctx, job.n, job.w, job.h, job.c, job.left, job.right, 0,
                                  job.focal, job.baseline, &job.out, nullptr);
        if (rc) msg = pstereo_gpu_last_error(wk->ctx);
      }
      const double ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      {
        std::lock_guard<std::mutex> lk(mu);
        wk->has_job = false;
        wk->rc = rc;
        wk->ms = ms;
        wk->err = msg;
        if (--pending == 0) cv_done.notify_all();
      }
    }
  }
};

namespace {

char* offset(void* p, size_t bytes) { return p ? static_cast<char*>(p) + bytes : nullptr; }

}  // namespace

extern "C" {

int pstereo_multi_create(const int* devices, int n_devices, const pstereo_params* p,
                         int max_width, int max_height, int max_pairs, pstereo_multi** out) {
  if (!out) return PSTEREO_EINTERNAL;
  *out = nullptr;
  if (!devices || n_devices < 1 || !p) return PSTEREO_EINTERNAL;
  char msg[256] = {0};
  if (pstereo_validate(p, msg, sizeof msg) != PSTEREO_OK) return PSTEREO_ECONFIG;
  auto m = std::make_unique<pstereo_multi>();
  m->params = *p;
  int caller_dev = 0;
  const bool restore = pstereo_gpu_current_device(&caller_dev) == PSTEREO_OK;
  // each context holds at most its block: ceil(max_pairs / n_devices)
  const int per = (max_pairs + n_devices - 1) / n_devices;
  for (int d = 0; d < n_devices; ++d) {
    auto wk = std::make_unique<Worker>();
    wk->device = devices[d];
    const int rc = pstereo_gpu_create(devices[d], p, max_width, max_height, per > 0 ? per : 1,
                                      &wk->ctx);
    if (rc != PSTEREO_OK) {
      for (auto& w : m->workers) pstereo_gpu_destroy(w->ctx);
      return rc;
    }
    m->workers.push_back(std::move(wk));
  }
  if (restore) pstereo_gpu_set_current_device(caller_dev);
  for (auto& wk : m->workers) {
    Worker* raw = wk.get();
    pstereo_multi* mm = m.get();
    wk->thread = std::thread([mm, raw] { mm->loop(raw); });
  }
  *out = m.release();
  return PSTEREO_OK;
}

void pstereo_multi_destroy(pstereo_multi* m) {
  if (!m) return;
  {
    std::lock_guard<std::mutex> lk(m->mu);
    m->quit = true;
  }
  m->cv_job.notify_all();
  for (auto& wk : m->workers)
    if (wk->thread.joinable()) wk->thread.join();
  for (auto& wk : m->workers) pstereo_gpu_destroy(wk->ctx);
  delete m;
}

const char* pstereo_multi_last_error(const pstereo_multi* m) { return m ? m->err.c_str() : ""; }

int pstereo_multi_n_devices(const pstereo_multi* m) { return m ? int(m->workers.size()) : 0; }

int pstereo_multi_match_u8(pstereo_multi* m, int n_pairs, int width, int height, int channels,
                           const uint8_t* left, const uint8_t* right, double focal_px,
                           double baseline, const pstereo_outputs* out, double* ms_per_device) {
  if (!m || !out || n_pairs < 0) return PSTEREO_EINTERNAL;
  if (out->on_device) {
    m->err = "pstereo_multi_match_u8: host output buffers only";
    return PSTEREO_EINTERNAL;
  }
  const int nd = int(m->workers.size());
  const size_t px = size_t(width) * height;
  const size_t vsz = out->dtype == PSTEREO_F64 ? 8 : 4;
  // MatchStats rows per pair = the level count, fixed by the params
  int n_levels = 0;
  if (out->stats) {
    int ws[PSTEREO_MAX_LEVELS], hs[PSTEREO_MAX_LEVELS], es[PSTEREO_MAX_LEVELS];
    if (pstereo_level_dims(&m->params, width, height, &n_levels, ws, hs, es) != PSTEREO_OK) {
      m->err = "pstereo_multi_match_u8: image smaller than a patch at the coarsest level";
      return PSTEREO_EDEGENERATE;
    }
  }
  {
    std::unique_lock<std::mutex> lk(m->mu);
    m->pending = nd;
    for (int d = 0; d < nd; ++d) {
      const int b0 = int((long long)n_pairs * d / nd);
      const int b1 = int((long long)n_pairs * (d + 1) / nd);
      Job j;
      j.n = b1 - b0;
      j.w = width;
      j.h = height;
      j.c = channels;
      j.left = left + size_t(b0) * px * channels;
      j.right = right + size_t(b0) * px * channels;
      j.focal = focal_px;
      j.baseline = baseline;
      j.out = *out;
      j.out.async_host = 0;
      const size_t vo = size_t(b0) * px * vsz, bo = size_t(b0) * px;
      j.out.disparity = offset(out->disparity, vo);
      j.out.disparity_valid = (uint8_t*)offset(out->disparity_valid, bo);
      j.out.probability = offset(out->probability, vo);
      j.out.depth = offset(out->depth, vo);
      j.out.depth_valid = (uint8_t*)offset(out->depth_valid, bo);
      j.out.depth_sigma = offset(out->depth_sigma, vo);
      j.out.sigma_valid = (uint8_t*)offset(out->sigma_valid, bo);
      j.out.match_disparity = offset(out->match_disparity, vo);
      j.out.match_valid = (uint8_t*)offset(out->match_valid, bo);
      j.out.var_disp = offset(out->var_disp, vo);
      j.out.finest = out->finest ? out->finest + size_t(b0) * out->finest_cap : nullptr;
      j.out.finest_count = out->finest_count ? out->finest_count + b0 : nullptr;
      j.out.stats = out->stats ? out->stats + size_t(b0) * n_levels : nullptr;
      m->workers[d]->job = j;
      m->workers[d]->has_job = true;
    }
  }
  m->cv_job.notify_all();
  {
    std::unique_lock<std::mutex> lk(m->mu);
    m->cv_done.wait(lk, [&] { return m->pending == 0; });
  }
  int rc = PSTEREO_OK;
  m->err.clear();
  for (int d = 0; d < nd; ++d) {
    if (ms_per_device) ms_per_device[d] = m->workers[d]->ms;
    if (m->workers[d]->rc != PSTEREO_OK && rc == PSTEREO_OK) {
      rc = m->workers[d]->rc;
      m->err = "device " + std::to_string(m->workers[d]->device) + ": " + m->workers[d]->err;
    }
  }
  return rc;
}

}  // extern "C"
