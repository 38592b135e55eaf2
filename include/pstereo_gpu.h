/*
 * pstereo_gpu.h -- C ABI of the B200-native BDIS matching core.
 *
 * Drop-in boundary for the reference's matching core:
 *   PipelineOutput run_pipeline(const GrayImage&, const GrayImage&,
 *                               const PipelineConfig&, const CameraParams&)
 *       (proj/include/pstereo/pipeline.hpp:20-22, src/pipeline.cpp:9-37)
 *   MatchResult match_stereo(const GrayImage&, const GrayImage&,
 *                            const PipelineConfig&)
 *       (proj/include/pstereo/coarse_to_fine.hpp:102-103)
 * The reference has no FFI; its callers are C++ (src/bench.cpp:24,
 * src/runner.cpp:140). This header is what such a caller -- or a ctypes /
 * cgo / JNI binding -- links against instead: plain pointers and sizes, no
 * C++ or torch types. include/pstereo_gpu.hpp re-exposes the reference's own
 * C++ signatures on top of it.
 *
 * Semantics follow the reference exactly (bit-identical disparity,
 * probability, validity and depth), batched over
 * independent pairs. There is no CPU fallback: every entry point that
 * computes requires a CUDA device with compute capability 10.0 (sm_100a).
 *
 * Error convention (inc/runner.hpp:16-19, src/runner.cpp:107-124):
 *   PSTEREO_ECONFIG     <- ConfigError (validate, src/coarse_to_fine.cpp:18-49)
 *   PSTEREO_EDEGENERATE <- DegenerateInputError (build_pyramid,
 *                          src/pyramid.cpp:46-58,84-89; make_patch_grid :56-61)
 *   PSTEREO_EINTERNAL   <- anything else (CUDA errors, bad arguments)
 * pstereo_gpu_last_error() returns the message of the last failure.
 */
#ifndef PSTEREO_GPU_H
#define PSTEREO_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSTEREO_OK 0
#define PSTEREO_EINTERNAL 1
#define PSTEREO_ECONFIG 2
#define PSTEREO_EIO 3 /* IoError (kExitIoError, inc/runner.hpp:18) */
#define PSTEREO_EDEGENERATE 4

#define PSTEREO_MAX_OFFSETS 16
#define PSTEREO_MAX_PATCH 32
#define PSTEREO_MAX_LEVELS 17

#define PSTEREO_F32 0
#define PSTEREO_F64 1

/* PipelineConfig (inc/config.hpp:12-33), window offsets inline. */
typedef struct pstereo_params {
  int coarsest_exp;          /* default 5 */
  int finest_exp;            /* default 1 */
  int patch_size;            /* default 10 (GPU path: 2..PSTEREO_MAX_PATCH) */
  double overlap;            /* default 0.55 */
  int min_iterations;        /* default 12 */
  int max_iterations;        /* default 12 */
  double early_stop_good;    /* default 0.05 */
  double early_stop_bad;     /* default 0.95 */
  double early_stop_improve; /* default 0.10 */
  int n_window_offsets;      /* default 2 */
  double window_offsets[PSTEREO_MAX_OFFSETS]; /* default {0.5, 1.0} */
  double sigma_s;            /* default 4.0 */
  double pixel_threshold;    /* default 0.15 */
  double gamma;              /* default 0.75 */
  double valid_patch_ratio;  /* default 0.75 */
  int estimate_variance;     /* default 0 */
  int threads;               /* default 1; validated, scheduling only */
} pstereo_params;

/* MatchStats::Level (inc/coarse_to_fine.hpp:80-89). */
typedef struct pstereo_level_stats {
  int exp;
  int grid_patches;
  int extracted;
  int converged;
  int accepted;
} pstereo_level_stats;

/* PatchEstimate (inc/coarse_to_fine.hpp:39-47) of the finest level. */
typedef struct pstereo_patch_estimate {
  double cx, cy, u, prob, posterior, sigma_k;
} pstereo_patch_estimate;

/*
 * Output planes, all [n_pairs][height][width] row-major top-to-bottom.
 * Value planes are float (PSTEREO_F32) or double (PSTEREO_F64); values at
 * invalid pixels equal the reference's (the unfiltered match value, or 0).
 * Any pointer may be NULL to skip that plane. When on_device is 0 the
 * pointers are host memory and the call blocks until they are written.
 *   disparity / disparity_valid   <- PipelineOutput::disparity (filtered)
 *   probability                   <- PipelineOutput::probability (its valid
 *                                    mask equals disparity_valid)
 *   depth / depth_valid           <- DepthResult::depth
 *   depth_sigma / sigma_valid     <- DepthResult::sigma (estimate_variance)
 *   match_disparity/match_valid   <- MatchResult::disparity (pre-filter)
 *   var_disp                      <- MatchResult::var_disp (estimate_variance;
 *                                    valid mask equals match_valid)
 *   stats       (host) [n_pairs][n_levels], coarsest level first
 *   finest      (host) [n_pairs][finest_cap] accepted finest-level patches
 *               in patch-index order, count per pair in finest_count[n_pairs]
 */
typedef struct pstereo_outputs {
  int dtype;
  int on_device;
  void* disparity;
  uint8_t* disparity_valid;
  void* probability;
  void* depth;
  uint8_t* depth_valid;
  void* depth_sigma;
  uint8_t* sigma_valid;
  void* match_disparity;
  uint8_t* match_valid;
  void* var_disp;
  pstereo_level_stats* stats;
  pstereo_patch_estimate* finest;
  int* finest_count;
  int finest_cap;
  /* When fill_invalid != 0, the disparity / depth / depth_sigma planes hold
   * invalid_value wherever their validity is 0 (the reference persists maps
   * that way: write_pfm stores -1 at invalid pixels, src/io.cpp:297-310), so a
   * caller can skip the u8 validity planes (4 instead of 5 bytes per pixel
   * for disparity alone). */
  int fill_invalid;
  double invalid_value;
  /* Host output buffers only: when async_host != 0 the call returns once its
   * work is queued; the host planes are complete after pstereo_gpu_wait (or
   * a device synchronize). Consecutive calls then overlap (the next batch's
   * uploads and kernels run under this batch's downloads). Ignored when
   * stats or finest records are requested (those are finished on the host). */
  int async_host;
  /* When flip_rows != 0 every output plane is written bottom row first --
   * the row order of the PFM payload (write_pfm, src/io.cpp:297-310) -- so
   * a disparity plane with fill_invalid / invalid_value -1 is the PFM body
   * verbatim (pstereo_write_pfm with rows_bottom_up = 1). */
  int flip_rows;
} pstereo_outputs;

typedef struct pstereo_ctx pstereo_ctx;

/* Published defaults, inc/config.hpp:12-33. */
void pstereo_default_params(pstereo_params* p);

/* validate(), src/coarse_to_fine.cpp:18-49 (plus the GPU path's patch-size
 * cap). Returns PSTEREO_OK or PSTEREO_ECONFIG with the message in msg. */
int pstereo_validate(const pstereo_params* p, char* msg, size_t msg_cap);

/* Number of pyramid levels and their dimensions for a width x height pair. */
int pstereo_level_dims(const pstereo_params* p, int width, int height,
                       int* n_levels, int* widths, int* heights, int* exps);

/*
 * Creates a context on `device` sized for up to max_pairs pairs of at most
 * max_width x max_height (any channel count). Validates params
 * (PSTEREO_ECONFIG) and checks the device is sm_100 (PSTEREO_EINTERNAL).
 * One context per device and host thread; a context is not re-entrant.
 */
int pstereo_gpu_create(int device, const pstereo_params* p, int max_width,
                       int max_height, int max_pairs, pstereo_ctx** out);
void pstereo_gpu_destroy(pstereo_ctx* ctx);
const char* pstereo_gpu_last_error(const pstereo_ctx* ctx);

/*
 * Batched run_pipeline on uint8 rasters (Raster, inc/image.hpp:12-17;
 * channels 1 = gray, 3 = RGB, 4 = RGBA with alpha==0 invalid), converted
 * with the reference's to_grayscale (src/image.cpp:16-43) on the device.
 * left/right: [n_pairs][height][width][channels] contiguous, host or device
 * memory per inputs_on_device. focal_px * baseline is the CameraParams
 * product (inc/depth_variance.hpp:20-23). `stream` is a cudaStream_t (NULL =
 * the context's own stream). With device inputs and device outputs and no
 * host stats/finest requested, the call only enqueues work on `stream`.
 */
int pstereo_gpu_match_u8(pstereo_ctx* ctx, int n_pairs, int width, int height,
                         int channels, const uint8_t* left,
                         const uint8_t* right, int inputs_on_device,
                         double focal_px, double baseline,
                         const pstereo_outputs* out, void* stream);

/*
 * Batched run_pipeline on GrayImage planes (inc/image.hpp:21-26): fp32
 * [n_pairs][height][width] plus optional u8 validity (NULL = all valid).
 */
int pstereo_gpu_match_f32(pstereo_ctx* ctx, int n_pairs, int width, int height,
                          const float* left, const uint8_t* left_valid,
                          const float* right, const uint8_t* right_valid,
                          int inputs_on_device, double focal_px,
                          double baseline, const pstereo_outputs* out,
                          void* stream);

/* Kernel launches issued by the last match call (telemetry for bench.py). */
/* compute_metrics (src/metrics.cpp:10-52; FrameMetrics,
 * inc/metrics.hpp:14-25) for n_frames ScalarFields of width x height:
 * errors |estimate - reference| over pixels valid on both sides; mean error
 * (the reference's sequential sum, bit-identical), median error (middle order
 * statistic, mean of the two middle ones for an even count), coverage_rate =
 * share of compared pixels with a valid sigma and |error| <= 1.96 sigma (NaN
 * when sigma is NULL). valid_px counts the estimate's valid pixels. Planes are
 * [frame][height][width] doubles / bytes, on the device when
 * inputs_on_device, else host memory; out is host memory. */
typedef struct pstereo_frame_metrics {
  long long valid_px;
  long long compared;
  int has_errors;      /* 0 when no pixel was comparable (mean/median NaN) */
  double mean_err;
  double median_err;
  double coverage_rate;
} pstereo_frame_metrics;
int pstereo_gpu_metrics(pstereo_ctx* ctx, int n_frames, int width, int height,
                        const double* estimate, const uint8_t* estimate_valid,
                        const double* reference, const uint8_t* reference_valid,
                        const double* sigma, const uint8_t* sigma_valid,
                        int inputs_on_device, pstereo_frame_metrics* out, void* stream);

/* Waits for every stream of the context and for `stream` (may be NULL). */
int pstereo_gpu_wait(pstereo_ctx* ctx, void* stream);

int pstereo_gpu_last_launch_count(const pstereo_ctx* ctx);

/* Stage timing with CUDA events recorded on the launch stream (no extra
 * synchronisation inside match calls). set_profiling(ctx, 1) resets the
 * accumulators; stage_times() waits for the recorded calls and returns the
 * number of stages, writing the total device ms per stage summed over
 * *n_calls calls. Stages: h2d, pyramid, patches_e<exp> per level (coarsest
 * first), finalize, d2h; names via pstereo_gpu_stage_name. */
int pstereo_gpu_set_profiling(pstereo_ctx* ctx, int enable);
/* Device-buffer calls of n pairs run as `chunks` sub-batches alternating over
 * two compute streams (their coarse levels and finalize overlap the other
 * sub-batch's finest level); 0 or 1 = one launch sequence. Results are
 * identical either way. Default: PSTEREO_DEVICE_CHUNKS or 2. */
int pstereo_gpu_set_device_chunks(pstereo_ctx* ctx, int chunks);
/* Host output buffers with finest_exp >= 1: every full-resolution plane is the
 * 2^e x 2^e block replication of a finest-level plane (upsample_to_full,
 * src/coarse_to_fine.cpp:166-180). With enable != 0 (the default;
 * PSTEREO_HOST_EXPAND=0 turns it off) the planes cross the link at the finest
 * level's resolution -- a quarter of the D2H bytes at finest_exp 1 -- and a
 * pool of host threads (PSTEREO_HOST_THREADS, default min(3 cores / 8, 6); count
 * via pstereo_gpu_host_threads) writes the blocks into the caller's buffers
 * while later chunks download. With 0 the device writes full-resolution
 * planes and the call copies them as they are. The bytes in the caller's
 * buffers are identical either way. */
int pstereo_gpu_set_host_expand(pstereo_ctx* ctx, int enable);
int pstereo_gpu_host_threads(void);
/* Totals since the pool started: worker milliseconds spent replicating and
 * frames (one plane of one pair) finished. */
int pstereo_host_expand_stats(double* busy_ms, long long* frames);
/* The host-side replication on its own (no device): dst[f][y][x] =
 * src[f][min(y >> e, fh - 1)][min(x >> e, fw - 1)] for n_frames frames of
 * elem_size (1, 4 or 8) bytes per element, rows bottom to top when flip_rows;
 * fw x fh must be W x H halved e times (rounding up). Runs on the pool. */
int pstereo_host_expand(const void* src, void* dst, int elem_size, int fw, int fh, int W, int H,
                        int e, int n_frames, int flip_rows);
/* Small launches: each pyramid level's patch grid is cut into enough row
 * bands that the launch has at least `ctas` CTAs (default 148, one per SM:
 * the lowest latency for a single call). A caller that keeps several calls
 * in flight on several contexts fills the GPU with those instead and sets 0
 * (measured: four 32-pair calls in flight 3% faster). Results are identical
 * for every value. */
int pstereo_gpu_set_fill_target(pstereo_ctx* ctx, int ctas);
/* Graph mode (default off). With it on, a call with device inputs and device
 * outputs and no host stats / finest records is captured into a CUDA graph
 * the second time its exact signature (sizes, pointers, stream, output
 * request) is seen, and replayed from then on: the same kernels with the
 * same arguments -- identical results -- without the per-call host work and
 * most inter-launch gaps (single-pair latency -8%). Up to 8 signatures per
 * context are kept; a graph is dropped when the context reallocated any
 * buffer since its capture. Turning it off frees them. */
int pstereo_gpu_set_graphs(pstereo_ctx* ctx, int enable);
int pstereo_gpu_stage_times(pstereo_ctx* ctx, double* ms_total, int cap, int* n_calls);
const char* pstereo_gpu_stage_name(const pstereo_ctx* ctx, int stage);

/* ---- test hook ----
 * eval_patch_residual (src/lk_solver.cpp:38-81) of size x size lattice
 * patches with footprint origin (x0[q], y0[q]) at disparity u[q], on one
 * width x height level, through the same device function k_patches uses.
 * Host buffers; returns PSTEREO_OK or PSTEREO_EINTERNAL. Used by the parity
 * tests to probe the evaluation at adversarial disparities. */
int pstereo_debug_eval_residual(int device, int width, int height,
                                const float* left, const uint8_t* left_valid,
                                const float* right, const uint8_t* right_valid,
                                int patch_size, int n_queries, const int* x0,
                                const int* y0, const double* u, double* msq,
                                double* jr, int* n);

/* ---- deterministic synthetic pairs (BASELINE.json configs) ---- */
typedef struct pstereo_synth_spec {
  int width, height, channels;
  uint64_t seed;
  int octaves;
  double base_wavelength;
  double d_min, d_range, blur_sigma;
  double noise_sigma;
  int stress;
} pstereo_synth_spec;

/* Defaults for BASELINE.json configs[config] (0..3). */
void pstereo_synth_default(pstereo_synth_spec* s, int config);
int pstereo_synth_pair(const pstereo_synth_spec* s, uint64_t seed,
                       uint8_t* left, uint8_t* right, float* disparity);
int pstereo_synth_batch(const pstereo_synth_spec* s, int n_pairs,
                        uint64_t seed0, uint8_t* left, uint8_t* right,
                        int threads);

/* The same generator on the device: pairs seed0 ..
 * seed0+n_pairs-1 written to DEVICE buffers left/right
 * [n_pairs][height][width][channels] and, when non-NULL, the ground-truth
 * disparity [n_pairs][height][width] -- byte-for-byte what
 * pstereo_synth_pair produces on the host for the same (spec, seed): both
 * evaluate csrc/synth_core.h with IEEE-exact operations only. Enqueued on
 * `stream` (a cudaStream_t, NULL = legacy default) after the blur taps are
 * uploaded (which waits for the stream's earlier work); scratch comes from
 * the stream-ordered allocator. Returns PSTEREO_OK, PSTEREO_ECONFIG (bad spec)
 * or PSTEREO_EINTERNAL; the message is in pstereo_synth_last_error(). */
int pstereo_gpu_synth(int device, const pstereo_synth_spec* s, int n_pairs,
                      uint64_t seed0, uint8_t* left, uint8_t* right,
                      float* disparity, void* stream);
const char* pstereo_synth_last_error(void);

/* ---- analytic test scenes ----
 * SceneSpec (inc/pstereo/synth.hpp:20-50) as a POD, enums as ints. */
#define PSTEREO_SURFACE_PLANE 0
#define PSTEREO_SURFACE_SLANTED 1
#define PSTEREO_SURFACE_SPHERE 2
#define PSTEREO_TEXTURE_PERLIN 0
#define PSTEREO_TEXTURE_CHECKER 1
#define PSTEREO_TEXTURE_CONSTANT 2
#define PSTEREO_SHADING_DIFFUSE 0
#define PSTEREO_SHADING_NONLAMBERTIAN 1
typedef struct pstereo_scene_spec {
  char name[64];
  int surface;
  double disparity, disparity0, disparity_gradient;
  double sphere_depth, sphere_radius, background_depth;
  int texture;
  double texture_scale;
  int texture_octaves;
  int shading;
  double ambient, highlight_strength, highlight_falloff;
  double noise_std;
  uint64_t seed;
  int seed_explicit;
  double focal_px, baseline;
  int width, height;
} pstereo_scene_spec;

/* SceneSpec's member defaults (inc/pstereo/synth.hpp:20-50). */
void pstereo_scene_default(pstereo_scene_spec* s);
/* The value checks of load_scene_spec (src/synth.cpp:365-390). */
int pstereo_scene_validate(const pstereo_scene_spec* s, char* msg, size_t msg_cap);
/* load_scene_spec (src/synth.cpp:301-393): "key = value" file, '#'
 * comments, unknown / duplicate keys and bad values are PSTEREO_ECONFIG, an
 * unreadable file PSTEREO_EIO. */
int pstereo_load_scene_spec(const char* path, pstereo_scene_spec* out, char* msg,
                            size_t msg_cap);
/* render_scene (src/synth.cpp:209-284) for n_scenes scenes of one size on
 * the device: DEVICE buffers left/right fp32 [n][h][w] (GrayImage, all
 * valid) and, when non-NULL, the reference disparity / depth fields as
 * doubles [n][h][w] (all valid). Enqueued on `stream` after the specs are
 * uploaded (which waits for the stream's earlier work). */
int pstereo_gpu_render(int device, const pstereo_scene_spec* specs, int n_scenes,
                       float* left, float* right, double* ref_disparity,
                       double* ref_depth, void* stream);
/* The same with HOST buffers (blocking; device scratch inside). */
int pstereo_render_host(int device, const pstereo_scene_spec* specs, int n_scenes,
                        float* left, float* right, double* ref_disparity,
                        double* ref_depth);
const char* pstereo_render_last_error(void);

/* ---- caller-side formats (src/io.cpp) ----
 * Host functions; return PSTEREO_OK, PSTEREO_ECONFIG or PSTEREO_EIO with the
 * message in msg. */
/* load_calibration (src/io.cpp:266-281) */
int pstereo_load_calibration(const char* path, double* focal_px, double* baseline_mm,
                             int* width, int* height, char* msg, size_t msg_cap);
/* load_image (src/io.cpp:253-263) for binary PGM/PPM (decode_pnm :151-198)
 * and 8-bit PNG (gray, gray+alpha -> RGBA, RGB, RGBA, palette -> RGB,
 * tRNS -> alpha; 16-bit samples stripped to their high byte, as
 * decode_png :200-249 configures libpng). Two calls: pixels == NULL returns
 * the dimensions; then pixels (capacity cap bytes) receives
 * [height][width][channels]. */
int pstereo_load_image(const char* path, int* width, int* height, int* channels,
                       uint8_t* pixels, size_t cap, char* msg, size_t msg_cap);
/* write_pfm (src/io.cpp:297-310): "Pf\n<w> <h>\n-1.0\n" then little-endian
 * float rows bottom to top. `values` holds [height][width] floats in the
 * order rows_bottom_up says (1 = already bottom to top, as a match call with
 * pstereo_outputs.flip_rows writes them); `valid` (NULL = all valid) turns
 * invalid pixels into the -1 sentinel. */
int pstereo_write_pfm(const char* path, int width, int height, const float* values,
                      const uint8_t* valid, int rows_bottom_up, char* msg, size_t msg_cap);
/* read_pfm (src/io.cpp:312-341): values [height][width] top to bottom;
 * values == NULL returns the dimensions only. */
int pstereo_read_pfm(const char* path, int* width, int* height, float* values, size_t cap,
                     char* msg, size_t msg_cap);
/* metrics CSV (src/io.cpp:346-439): header, rows formatted with the
 * shortest round-trip representation (std::to_chars), nan for unavailable. */
typedef struct pstereo_metrics_row {
  char frame[128];
  double mean_err;
  double median_err;
  long long valid_px;
  double runtime_ms;
  double coverage_rate;
  int has_errors;
} pstereo_metrics_row;
const char* pstereo_metrics_csv_header(void);
/* writes the row's CSV text (no newline) into buf; returns its length or -1 */
int pstereo_format_metrics_row(const pstereo_metrics_row* row, char* buf, size_t cap);
int pstereo_write_metrics_csv(const char* path, const pstereo_metrics_row* rows, int n_rows,
                              char* msg, size_t msg_cap);
/* rows == NULL: *n_rows receives the row count */
int pstereo_read_metrics_csv(const char* path, pstereo_metrics_row* rows, int cap,
                             int* n_rows, char* msg, size_t msg_cap);

/* IoErrorKind (inc/errors.hpp:14-19) of the last PSTEREO_EIO returned on the
 * calling thread by one of the functions above, -1 if none. */
#define PSTEREO_IO_MISSING_FILE 0
#define PSTEREO_IO_DECODE_FAILURE 1
#define PSTEREO_IO_DIMENSION_MISMATCH 2
#define PSTEREO_IO_WRITE_FAILURE 3
int pstereo_last_io_kind(void);

/* ---- helpers of the C++ drop-in headers (include/pstereo/ headers) ---- */
/* The calling host thread's current CUDA device (cudaGetDevice). */
int pstereo_gpu_current_device(int* device);
/* cudaSetDevice for the calling host thread. */
int pstereo_gpu_set_current_device(int device);
/* to_grayscale (src/image.cpp:16-43) of one HOST raster [height][width]
 * [channels] on `device` (the k_gray_u8 kernel of the match path): fp32 gray
 * and u8 validity (alpha == 0 invalid) into host buffers. Channels other
 * than 1, 3, 4 return PSTEREO_ECONFIG (the reference throws
 * std::invalid_argument). Blocking. */
int pstereo_gpu_to_grayscale(int device, int width, int height, int channels,
                             const uint8_t* pixels, float* gray, uint8_t* valid);

/* ---- pair sharding over several devices ----
 * The reference's only parallelism is parallel_patches
 * (src/coarse_to_fine.cpp:184-205): worker threads over the patches of one
 * pair. Here whole pairs are the unit: a pstereo_multi owns one context and
 * one persistent host thread per entry of `devices` (entries may repeat: two
 * contexts on one GPU). A match call splits n_pairs into contiguous blocks,
 * block d = pairs [d*n/N, (d+1)*n/N), and every worker runs its block through
 * its own context from HOST buffers (its own uploads, kernels and downloads;
 * no collective, no peer traffic), writing the block's slice of every output
 * plane, stats and finest records. The call returns when every block is
 * done; results are identical to one context running all pairs. max_pairs is
 * the largest n_pairs a call may pass. Like a context, a pstereo_multi is not
 * re-entrant: one call at a time. */
typedef struct pstereo_multi pstereo_multi;
int pstereo_multi_create(const int* devices, int n_devices, const pstereo_params* p,
                         int max_width, int max_height, int max_pairs,
                         pstereo_multi** out);
void pstereo_multi_destroy(pstereo_multi* m);
const char* pstereo_multi_last_error(const pstereo_multi* m);
int pstereo_multi_n_devices(const pstereo_multi* m);
/* pstereo_gpu_match_u8 semantics with host inputs and host outputs
 * (out->on_device must be 0; async_host is ignored). When `ms_per_device` is
 * non-NULL it receives each worker's wall time of its block (ms). */
int pstereo_multi_match_u8(pstereo_multi* m, int n_pairs, int width, int height,
                           int channels, const uint8_t* left, const uint8_t* right,
                           double focal_px, double baseline,
                           const pstereo_outputs* out, double* ms_per_device);

#ifdef __cplusplus
}
#endif

#endif /* PSTEREO_GPU_H */
