// Drop-in check of the caller side in the reference's own language (SURVEY.md
// 8f row 4): the same scene specs go through the reference's render_scene +
// run_benchmark (src/synth.cpp, src/bench.cpp, compiled unmodified into
// oracle/_ref) and through this repo's shim (pstereo::gpu::render_scene /
// run_benchmark over the C ABI); the rendered views and fields must be
// identical and so must every metrics row except the timing column.
// Test infrastructure: built by tests/cpp/build.sh, run by
// tests/test_gpu_dropin.py.
//
// Usage: dropin_bench [width height]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pstereo/bench.hpp"  // the reference (inc/)
#include "pstereo/synth.hpp"
#include "pstereo_gpu.hpp"    // the drop-in (include/)

namespace {

int g_fail = 0;

void check(bool ok, const char* what, long long i) {
  if (!ok && g_fail++ < 10) std::fprintf(stderr, "MISMATCH %s at %lld\n", what, i);
}

bool same_double(double a, double b) {
  return (std::isnan(a) && std::isnan(b)) || std::memcmp(&a, &b, sizeof a) == 0;
}

pstereo::SceneSpec to_ref(const pstereo::gpu::SceneSpec& g) {
  pstereo::SceneSpec s;
  s.name = g.name;
  s.surface = g.surface == 1 ? pstereo::SurfaceKind::slanted_plane
              : g.surface == 2 ? pstereo::SurfaceKind::sphere : pstereo::SurfaceKind::plane;
  s.disparity = g.disparity;
  s.disparity0 = g.disparity0;
  s.disparity_gradient = g.disparity_gradient;
  s.sphere_depth = g.sphere_depth;
  s.sphere_radius = g.sphere_radius;
  s.background_depth = g.background_depth;
  s.texture = g.texture == 1 ? pstereo::TextureKind::checker
              : g.texture == 2 ? pstereo::TextureKind::constant : pstereo::TextureKind::perlin;
  s.texture_scale = g.texture_scale;
  s.texture_octaves = g.texture_octaves;
  s.shading = g.shading == 1 ? pstereo::ShadingKind::nonlambertian
                             : pstereo::ShadingKind::diffuse;
  s.ambient = g.ambient;
  s.highlight_strength = g.highlight_strength;
  s.highlight_falloff = g.highlight_falloff;
  s.noise_std = g.noise_std;
  s.seed = g.seed;
  s.focal_px = g.focal_px;
  s.baseline = g.baseline;
  s.width = g.width;
  s.height = g.height;
  return s;
}

}  // namespace

int main(int argc, char** argv) {
  const int w = argc > 2 ? std::atoi(argv[1]) : 320, h = argc > 2 ? std::atoi(argv[2]) : 240;
  std::vector<pstereo::gpu::SceneSpec> gs;
  auto add = [&](int surface, int texture, int shading, double noise, double grad) {
    pstereo::gpu::SceneSpec s = pstereo::gpu::default_scene();
    std::snprintf(s.name, sizeof s.name, "scene%zu", gs.size());
    s.surface = surface;
    s.texture = texture;
    s.shading = shading;
    s.noise_std = noise;
    s.disparity0 = 6.0;
    s.disparity_gradient = grad;
    s.seed = 3 + gs.size();
    s.width = w;
    s.height = h;
    gs.push_back(s);
  };
  add(0, 0, 0, 0.0, 0.0);
  add(0, 0, 0, 0.01, 0.0);
  add(1, 0, 0, 0.0, 0.01);
  add(2, 0, 0, 0.0, 0.0);
  add(2, 0, 1, 0.0, 0.0);
  add(0, 1, 0, 0.0, 0.0);
  std::vector<pstereo::SceneSpec> rs;
  for (const auto& s : gs) rs.push_back(to_ref(s));

  for (std::size_t k = 0; k < gs.size(); ++k) {
    const pstereo::RenderedScene a = pstereo::render_scene(rs[k]);
    const pstereo::gpu::RenderedScene b = pstereo::gpu::render_scene(gs[k]);
    for (std::size_t i = 0; i < a.left.data.size(); ++i) {
      check(std::memcmp(&a.left.data[i], &b.left.data[i], 4) == 0, "left", (long long)i);
      check(std::memcmp(&a.right.data[i], &b.right.data[i], 4) == 0, "right", (long long)i);
      check(same_double(a.ref_depth.values[i], b.ref_depth.values[i]), "ref_depth", (long long)i);
      check(same_double(a.ref_disparity.values[i], b.ref_disparity.values[i]), "ref_disparity",
            (long long)i);
    }
  }
  pstereo::PipelineConfig rc;
  rc.coarsest_exp = 4;
  rc.patch_size = 8;
  rc.overlap = 0.5;
  pstereo::gpu::PipelineConfig gc;
  gc.coarsest_exp = 4;
  gc.patch_size = 8;
  gc.overlap = 0.5;
  for (int var = 0; var < 2; ++var) {
    rc.estimate_variance = var != 0;
    gc.estimate_variance = var != 0;
    const pstereo::BenchResult a = pstereo::run_benchmark(rs, rc, 1);
    const pstereo::gpu::BenchResult b = pstereo::gpu::run_benchmark(gs, gc, 1);
    std::vector<pstereo::FrameMetrics> ra = a.frames;
    ra.push_back(a.aggregate);
    std::vector<pstereo::gpu::FrameMetrics> rb = b.frames;
    rb.push_back(b.aggregate);
    for (std::size_t k = 0; k < ra.size(); ++k) {
      check(ra[k].frame == rb[k].frame, "frame", (long long)k);
      check((long long)ra[k].valid_px == rb[k].valid_px, "valid_px", (long long)k);
      check(ra[k].has_errors == rb[k].has_errors, "has_errors", (long long)k);
      check(same_double(ra[k].mean_err, rb[k].mean_err), "mean_err", (long long)k);
      check(same_double(ra[k].median_err, rb[k].median_err), "median_err", (long long)k);
      // coverage depends on sigma, which goes through libm exp (1e-3 rel)
      const double ca = ra[k].coverage_rate, cb = rb[k].coverage_rate;
      check((std::isnan(ca) && std::isnan(cb)) || std::fabs(ca - cb) <= 1e-3, "coverage",
            (long long)k);
      std::printf("%-8s valid %ld mean %.17g median %.17g coverage %g\n", ra[k].frame.c_str(),
                  (long)ra[k].valid_px, ra[k].mean_err, ra[k].median_err, ra[k].coverage_rate);
    }
  }
  if (g_fail) {
    std::printf("%d mismatches\n", g_fail);
    return 1;
  }
  std::printf("identical: %zu scenes rendered, benchmark rows x2\n", gs.size());
  return 0;
}
