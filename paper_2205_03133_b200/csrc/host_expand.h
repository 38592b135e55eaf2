// host_expand.h -- the nearest-neighbour replication of upsample_to_full
// (src/coarse_to_fine.cpp:166-180) done on the HOST side of the device->host
// link: a host-output call downloads each requested plane at the finest
// level's resolution (a quarter of the bytes at finest_exp 1) into pinned
// staging, and a pool of host threads writes every value to its 2^e x 2^e
// full-resolution block in the caller's buffer with streaming stores.
// The values are untouched, so the planes stay bit-identical to the device-side
// replication (k_output_x4); only the PCIe traffic changes.
#pragma once

#include <condition_variable>
#include <cstddef>
#include <mutex>

namespace bdis {

// completion counter of one staging set
struct ExpandCounter {
  std::mutex m;
  std::condition_variable cv;
  long pending = 0;
  void add(long n);
  void done(long n);
  void wait();
};

// out(x, y) = src(min(x >> e, fw - 1), min(y >> e, fh - 1)) for one plane of
// `n_pairs` frames; rows bottom to top when flip (the PFM payload order)
struct ExpandJob {
  const void* src;  // [n_pairs][fh][fw], pinned staging
  void* dst;        // [n_pairs][H][W], the caller's buffer
  int esz;          // bytes per element: 1, 4 or 8
  int fw, fh, W, H, e;
  int n_pairs;
  int flip;
};

// one plane of one frame, on the calling thread
void expand_frame(const ExpandJob& j, int pair);

// queue the frames of `jobs[0..n)` on the process-wide pool; `c` is credited as
// frames finish (the caller has already add()ed n_pairs per job)
void expand_submit(const ExpandJob* jobs, int n, ExpandCounter* c);

// worker threads of the pool (PSTEREO_HOST_THREADS, default: 3/8 of the
// host's cores, at most 6); started on first use
int expand_threads();

// totals since the pool started: worker time inside expand_frame, frames done
void expand_stats(double* busy_ms, long long* frames);

}  // namespace bdis
