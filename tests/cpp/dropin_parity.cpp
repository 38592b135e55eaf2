// Drop-in check in the reference's own language. The same caller code runs
// pstereo::run_pipeline / pstereo::match_stereo -- the reference (its
// unmodified sources, compiled into oracle/_ref) -- and
// pstereo::gpu::run_pipeline / pstereo::gpu::match_stereo -- this repo's C++
// shim over the C ABI (include/pstereo_gpu.hpp) -- on identical GrayImages,
// and requires identical results. Test infrastructure: built by
// tests/cpp/build.sh where /root/reference exists, run by
// tests/test_gpu_dropin.py on a GPU box.
//
// Usage: dropin_parity [config 0..4] [seed] [width height]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pstereo/coarse_to_fine.hpp"  // the reference (inc/)
#include "pstereo/config.hpp"
#include "pstereo/image.hpp"
#include "pstereo/pipeline.hpp"
#include "pstereo_gpu.hpp"             // the drop-in (include/)

namespace {

int g_fail = 0;

void check(bool ok, const char* what, long long i) {
  if (!ok && g_fail++ < 10) std::fprintf(stderr, "MISMATCH %s at %lld\n", what, i);
}

template <class A, class B>
void same_field(const A& a, const B& b, const char* name, double rtol) {
  check(a.width == b.width && a.height == b.height, name, -1);
  for (std::size_t i = 0; i < a.values.size(); ++i) {
    check(a.valid[i] == b.valid[i], name, (long long)i);
    if (!a.valid[i]) continue;
    const double x = a.values[i], y = b.values[i];
    const bool ok = rtol == 0.0 ? std::memcmp(&x, &y, sizeof x) == 0
                                : std::fabs(x - y) <= rtol * std::fabs(x) + 1e-300;
    check(ok, name, (long long)i);
  }
}

}  // namespace

int main(int argc, char** argv) {
  const int config = argc > 1 ? std::atoi(argv[1]) : 0;
  const unsigned long long seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 0;
  pstereo_synth_spec spec;
  pstereo_synth_default(&spec, config);
  if (argc > 4) {
    spec.width = std::atoi(argv[3]);
    spec.height = std::atoi(argv[4]);
  }
  const int w = spec.width, h = spec.height, C = spec.channels;
  std::vector<std::uint8_t> l(std::size_t(w) * h * C), r(l.size());
  if (pstereo_synth_pair(&spec, seed, l.data(), r.data(), nullptr)) return 2;

  // the caller's side: Raster -> GrayImage with the reference's converter
  pstereo::Raster rl{w, h, C, l}, rr{w, h, C, r};
  const pstereo::GrayImage gl = pstereo::to_grayscale(rl), gr = pstereo::to_grayscale(rr);
  pstereo::gpu::GrayImage xl{gl.width, gl.height, gl.data, gl.valid};
  pstereo::gpu::GrayImage xr{gr.width, gr.height, gr.data, gr.valid};

  // BASELINE.json config -> PipelineConfig
  pstereo::PipelineConfig cfg;
  cfg.coarsest_exp = config == 3 ? 4 : 3;
  cfg.finest_exp = 1;
  cfg.patch_size = config == 3 ? 12 : 8;
  cfg.overlap = config == 3 ? 1.0 - 4.0 / 12.0 : 0.5;
  cfg.estimate_variance = config == 1 || config == 3;
  pstereo::gpu::PipelineConfig gcfg;
  gcfg.coarsest_exp = cfg.coarsest_exp;
  gcfg.finest_exp = cfg.finest_exp;
  gcfg.patch_size = cfg.patch_size;
  gcfg.overlap = cfg.overlap;
  gcfg.estimate_variance = cfg.estimate_variance;
  const pstereo::CameraParams cam{500.0, 5.0};
  const pstereo::gpu::CameraParams gcam{500.0, 5.0};

  const pstereo::PipelineOutput ref = pstereo::run_pipeline(gl, gr, cfg, cam);
  const pstereo::gpu::PipelineOutput gpu = pstereo::gpu::run_pipeline(xl, xr, gcfg, gcam);
  same_field(ref.disparity, gpu.disparity, "disparity", 0.0);
  same_field(ref.probability, gpu.probability, "probability", 0.0);
  same_field(ref.depth.depth, gpu.depth.depth, "depth", 0.0);
  check(ref.depth.has_sigma == gpu.depth.has_sigma, "has_sigma", -1);
  if (ref.depth.has_sigma) same_field(ref.depth.sigma, gpu.depth.sigma, "depth_sigma", 1e-3);
  check(ref.stats.levels.size() == gpu.stats.levels.size(), "stats levels", -1);
  for (std::size_t k = 0; k < ref.stats.levels.size() && k < gpu.stats.levels.size(); ++k) {
    const auto& a = ref.stats.levels[k];
    const auto& b = gpu.stats.levels[k];
    check(a.exp == b.exp && a.grid_patches == b.grid_patches && a.extracted == b.extracted &&
              a.converged == b.converged && a.accepted == b.accepted,
          "MatchStats", (long long)k);
  }
  const pstereo::MatchResult mr = pstereo::match_stereo(gl, gr, cfg);
  const pstereo::gpu::MatchResult mg = pstereo::gpu::match_stereo(xl, xr, gcfg);
  same_field(mr.disparity, mg.disparity, "match disparity", 0.0);
  same_field(mr.probability, mg.probability, "match probability", 0.0);

  long long valid = 0;
  for (auto v : gpu.disparity.valid) valid += v;
  std::printf("config %d seed %llu %dx%d: %s (%lld valid px, ref %.1f ms)\n", config, seed, w, h,
              g_fail ? "DIFFERENT" : "identical", valid, ref.runtime_ms);
  return g_fail ? 1 : 0;
}
