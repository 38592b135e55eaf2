/*
 * bdis_oracle.h -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * One C interface, two implementations:
 *   - oracle/bdis_oracle.c      : plain-C restatement of the reference's
 *                                 per-frame BDIS path (each function cites
 *                                 the reference file:line it follows);
 *   - oracle/ref_glue.cpp       : thin wrapper that calls the UNMODIFIED
 *                                 reference sources compiled from
 *                                 /root/reference/proj/src into
 *                                 oracle/_ref/libbdis_ref.so (see Makefile).
 * Tests pin the restatement against the reference build and the committed
 * golden fixtures; the GPU product is then checked against the restatement.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these libraries.
 *
 * Reference paths are abbreviated src/ = proj/src/, inc/ = proj/include/pstereo/.
 */
#ifndef BDIS_ORACLE_H
#define BDIS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BO_MAX_OFFSETS 16
#define BO_OK 0
#define BO_EINTERNAL 1
#define BO_ECONFIG 2
#define BO_EDEGENERATE 4

/* Mirrors PipelineConfig (inc/config.hpp:12-33). */
typedef struct bo_config {
  int coarsest_exp;
  int finest_exp;
  int patch_size;
  double overlap;
  int min_iterations;
  int max_iterations;
  double early_stop_good;
  double early_stop_bad;
  double early_stop_improve;
  int n_window_offsets;
  double window_offsets[BO_MAX_OFFSETS];
  double sigma_s;
  double pixel_threshold;
  double gamma;
  double valid_patch_ratio;
  int estimate_variance;
  int threads;
} bo_config;

/* GrayImage (inc/image.hpp:21-36): fp32 row-major + u8 validity. */
typedef struct bo_image {
  int width;
  int height;
  const float* data;
  const uint8_t* valid;
} bo_image;

/* LkParams (inc/lk_solver.hpp:34-46). */
typedef struct bo_lk_params {
  int min_iterations;
  int max_iterations;
  double update_epsilon;
  double stop_good;
  double stop_bad;
  double stop_improve;
} bo_lk_params;

/* Patch + PatchSystem scalars (inc/patch.hpp:14-25, inc/lk_solver.hpp:20-27). */
typedef struct bo_patch_info {
  double mean;
  double valid_fraction;
  int valid_count;
  double hessian;
  double template_msq;
  int degenerate;
} bo_patch_info;

/* run_pipeline outputs (inc/pipeline.hpp:10-16). Every pointer is caller
 * allocated width*height (stats: n_levels*5 ints: exp, grid, extracted,
 * converged, accepted). depth_sigma/sigma_valid may be NULL. */
typedef struct bo_outputs {
  double* disparity;
  uint8_t* disparity_valid;
  double* probability;
  uint8_t* probability_valid;
  double* depth;
  uint8_t* depth_valid;
  double* depth_sigma;
  uint8_t* sigma_valid;
  int has_sigma;
  int* stats;
  int n_levels;
  double runtime_ms;
} bo_outputs;

/* match_stereo outputs (inc/coarse_to_fine.hpp:92-99). var_disp may be NULL.
 * finest: up to finest_cap rows of 7 doubles
 * {cx, cy, u, prob, posterior, sigma_k, has_sigma}. */
typedef struct bo_match_outputs {
  double* disparity;
  uint8_t* disparity_valid;
  double* probability;
  uint8_t* probability_valid;
  double* var_disp;
  uint8_t* var_valid;
  int has_variance;
  int* stats;
  int n_levels;
  int finest_cap;
  int finest_count;
  double* finest;
} bo_match_outputs;

/* ---- config ---- */
void bo_default_config(bo_config* cfg);
int bo_validate(const bo_config* cfg, char* msg, int msg_cap);

/* ---- numerics / image stages ---- */
double bo_fast_exp(double x);
void bo_spatial_mask(int size, double sigma_s, double* out);
void bo_to_grayscale(int w, int h, int channels, const uint8_t* px, float* out,
                     uint8_t* valid);
int bo_sample_bilinear(const bo_image* img, double x, double y, double* value);
void bo_downsample_half(int w, int h, const float* data, const uint8_t* valid,
                        float* out, uint8_t* out_valid);
void bo_gradient_x(int w, int h, const float* data, float* out);

/* ---- patch level ---- */
int bo_extract_patch(const bo_image* img, double cx, double cy, int size,
                     double* values, uint8_t* valid, bo_patch_info* info);
int bo_patch_system(const bo_image* left, const float* grad, double cx,
                    double cy, int size, double* jacobian, bo_patch_info* info);
int bo_eval_residual(const bo_image* left, const float* grad,
                     const bo_image* right, double cx, double cy, int size,
                     double u, double* msq, double* jr, int* n);
int bo_solve_patch(const bo_image* left, const float* grad,
                   const bo_image* right, double cx, double cy, int size,
                   double u_init, const bo_lk_params* p, double* u,
                   int* converged, int* iterations, double* final_residual);
int bo_sample_window(const bo_image* left, const float* grad,
                     const bo_image* right, double cx, double cy, int size,
                     double u_k, int n_mags, const double* mags,
                     double* offsets, double* residuals, uint8_t* valid,
                     int* center_index);
double bo_dynamic_sigma(int n, const double* residuals, const uint8_t* valid,
                        double sigma_floor);
void bo_window_priors(int n, const double* residuals, const uint8_t* valid,
                      double sigma_r, int patch_size, int use_fast_exp,
                      double* priors);
int bo_patch_posterior(int n, const double* residuals, const uint8_t* valid,
                       int center_index, double sigma_r, int patch_size,
                       int use_fast_exp, double* probability, int* is_min);
void bo_estimate_variance(int n, const double* offsets, const uint8_t* valid,
                          int center_index, const double* priors,
                          double sigma_fallback, double* sigma_k, double* c_k,
                          int* accepted, int* reason, double* fit_residual);

/* ---- level / grid ---- */
int bo_make_patch_grid(int w, int h, int patch_size, double overlap,
                       int* stride, int* nx, int* ny, double* xs, double* ys,
                       int cap);
double bo_level_weight(int n, int n_levels, const int* levels);
double bo_propagate_probability(double posterior, double inherited, int n,
                                int n_levels, const int* levels);
void bo_fuse_level(int n_patches, const double* cx, const double* cy,
                   const double* u, const double* prob, const double* sigma_k,
                   int size, double sigma_s, int w, int h, int with_variance,
                   double* disp, uint8_t* disp_valid, double* prob_out,
                   uint8_t* prob_valid, double* var, uint8_t* var_valid);
void bo_init_next_level(int cw, int ch, const double* values,
                        const uint8_t* valid, int fw, int fh, double* out);
void bo_upsample_to_full(int w, int h, const double* values,
                         const uint8_t* valid, int fw, int fh, int exp,
                         double scale_per_level, double* out,
                         uint8_t* out_valid);

/* ---- filter / depth ---- */
void bo_remove_small_components(const uint8_t* valid, int w, int h,
                                long long min_px, uint8_t* out);
void bo_filter_validity(int w, int h, const uint8_t* disp_valid,
                        const double* prob, const uint8_t* prob_valid,
                        double gamma, double pixel_threshold, int patch_size,
                        uint8_t* out_valid);
void bo_disparity_to_depth(int w, int h, const double* disp,
                           const uint8_t* disp_valid, const double* var,
                           const uint8_t* var_valid, double focal_px,
                           double baseline, double min_disparity,
                           double* depth, uint8_t* depth_valid, double* sigma,
                           uint8_t* sigma_valid);

/* ---- metrics (src/metrics.cpp:10-52) ---- */
typedef struct bo_frame_metrics {
  long long valid_px;   /* estimate.valid_count() */
  long long compared;   /* pixels valid in estimate and reference */
  int has_errors;
  double mean_err, median_err, coverage_rate; /* NaN when unavailable */
} bo_frame_metrics;
/* sigma / sigma_valid may be NULL (coverage_rate stays NaN) */
void bo_compute_metrics(int w, int h, const double* est, const uint8_t* est_valid,
                        const double* ref, const uint8_t* ref_valid, const double* sigma,
                        const uint8_t* sigma_valid, bo_frame_metrics* out);

/* ---- analytic scene renderer (src/synth.cpp) ----
 * SceneSpec (inc/pstereo/synth.hpp:20-50) as a POD; enums as ints
 * (surface 0 plane / 1 slanted_plane / 2 sphere, texture 0 perlin /
 * 1 checker / 2 constant, shading 0 diffuse / 1 nonlambertian). Same layout
 * as the product's pstereo_scene_spec. */
typedef struct bo_scene {
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
} bo_scene;
double bo_scene_disparity_at(const bo_scene* s, double x, double y);
double bo_scene_intensity_at(const bo_scene* s, double x, double y);
double bo_value_noise(double x, double y, uint64_t seed, int octaves, double base_scale);
double bo_gaussian_noise(uint64_t seed, uint64_t stream, uint64_t index);
/* render_scene (src/synth.cpp:209-284): left/right fp32 [h][w] (GrayImage,
 * all valid), reference disparity / depth doubles [h][w] (all valid). */
int bo_render_scene(const bo_scene* s, float* left, float* right, double* ref_disparity,
                    double* ref_depth);

/* ---- whole path ---- */
int bo_match_stereo(const bo_image* left, const bo_image* right,
                    const bo_config* cfg, bo_match_outputs* out, char* msg,
                    int msg_cap);
int bo_run_pipeline(const bo_image* left, const bo_image* right,
                    const bo_config* cfg, double focal_px, double baseline,
                    bo_outputs* out, char* msg, int msg_cap);

#ifdef __cplusplus
}
#endif

#endif /* BDIS_ORACLE_H */
