// TEST INFRASTRUCTURE -- a caller of the reference's public C++ API, written
// only against the reference's headers (namespace pstereo, "pstereo/*.hpp").
// tests/cpp/build.sh compiles it twice:
//   build/caller_ref : with the reference's include/ and ALL of its sources
//                      (the unmodified reference)
//   build/caller_gpu : with this repo's include/ ahead of the reference's,
//                      the reference's caller-side sources only (bench.cpp,
//                      io.cpp, metrics.cpp, runner.cpp, synth.cpp, unchanged)
//                      and libpstereo_gpu.so in place of the matcher's sources
// tests/test_gpu_dropin.py runs both on the same inputs and compares the dumps
// and the files run_match / run_bench write.
//
// Usage: caller WORKDIR LEFT.pgm RIGHT.pgm CALIB CONFIG(0..4)
// Writes WORKDIR/dump.bin (records: name, kind, count, payload) plus the
// run_match outputs under WORKDIR/match and WORKDIR/bench.csv.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "pstereo/bench.hpp"
#include "pstereo/coarse_to_fine.hpp"
#include "pstereo/config.hpp"
#include "pstereo/errors.hpp"
#include "pstereo/image.hpp"
#include "pstereo/io.hpp"
#include "pstereo/metrics.hpp"
#include "pstereo/pipeline.hpp"
#include "pstereo/runner.hpp"
#include "pstereo/synth.hpp"

using namespace pstereo;

namespace {

// record kinds: 0 = doubles compared bit for bit, 1 = doubles within 1e-3
// relative (variance-derived), 2 = bytes, 3 = int64, 4 = text
std::ofstream g_dump;

void rec(const std::string& name, int kind, const void* data, std::uint64_t count,
         std::size_t elem) {
  char n[64] = {0};
  std::snprintf(n, sizeof n, "%s", name.c_str());
  g_dump.write(n, 64);
  const std::uint8_t k = std::uint8_t(kind);
  g_dump.write(reinterpret_cast<const char*>(&k), 1);
  g_dump.write(reinterpret_cast<const char*>(&count), 8);
  g_dump.write(static_cast<const char*>(data), std::streamsize(count * elem));
}
void rec_i(const std::string& name, std::int64_t v) { rec(name, 3, &v, 1, 8); }
void rec_d(const std::string& name, double v, int kind = 0) { rec(name, kind, &v, 1, 8); }
void rec_s(const std::string& name, const std::string& s) { rec(name, 4, s.data(), s.size(), 1); }

void rec_field(const std::string& name, const ScalarField& f, int kind = 0) {
  rec_i(name + ".w", f.width);
  rec_i(name + ".h", f.height);
  rec(name + ".valid", 2, f.valid.data(), f.valid.size(), 1);
  // values at invalid pixels are unspecified: zero them before dumping
  std::vector<double> v(f.values.size(), 0.0);
  for (int y = 0; y < f.height; ++y)
    for (int x = 0; x < f.width; ++x)
      if (f.valid_at(x, y)) v[f.index(x, y)] = f.at(x, y);
  rec(name + ".values", kind, v.data(), v.size(), 8);
  rec_i(name + ".valid_count", f.valid_count());
  rec_i(name + ".size", std::int64_t(f.size()));
}

void rec_stats(const std::string& name, const MatchStats& s) {
  std::vector<std::int64_t> v;
  for (const auto& l : s.levels)
    for (int x : {l.exp, l.grid_patches, l.extracted, l.converged, l.accepted}) v.push_back(x);
  rec(name, 3, v.data(), v.size(), 8);
}

PipelineConfig config_for(int c) {
  // BASELINE.json configs -> PipelineConfig; 4 = the
  // reference's own defaults (inc/config.hpp: 5..1, s = 10, overlap 0.55)
  PipelineConfig cfg;
  if (c == 4) return cfg;
  cfg.coarsest_exp = c == 3 ? 4 : 3;
  cfg.finest_exp = 1;
  cfg.patch_size = c == 3 ? 12 : 8;
  cfg.overlap = c == 3 ? 1.0 - 4.0 / 12.0 : 0.5;
  cfg.estimate_variance = c == 1 || c == 3;
  return cfg;
}

template <class F>
std::string error_class(F&& f) {
  try {
    f();
  } catch (const ConfigError&) {
    return "ConfigError";
  } catch (const DegenerateInputError&) {
    return "DegenerateInputError";
  } catch (const IoError& e) {
    return "IoError/" + std::to_string(int(e.kind));
  } catch (const std::invalid_argument&) {
    return "invalid_argument";
  } catch (const std::exception& e) {
    return std::string("other: ") + e.what();
  }
  return "none";
}

void write_scene(const std::string& path, const std::string& body) {
  std::ofstream(path) << body;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: caller WORKDIR LEFT RIGHT CALIB CONFIG\n");
    return 2;
  }
  const std::string dir = argv[1];
  const int config = std::atoi(argv[5]);
  std::filesystem::create_directories(dir);
  g_dump.open(dir + "/dump.bin", std::ios::binary);
  const PipelineConfig cfg = config_for(config);
  const int var_kind = cfg.estimate_variance ? 1 : 0;

  // 1. the CLI's match body (src/runner.cpp:128-161): load, match, PFMs, CSV
  MatchArgs ma;
  ma.left_path = argv[2];
  ma.right_path = argv[3];
  ma.calib_path = argv[4];
  ma.out_dir = dir + "/match";
  ma.frame = "pair";
  ma.cfg = cfg;
  std::ostringstream out, err;
  rec_i("run_match.rc", run_match(ma, out, err));
  {
    // the CSV row without its runtime column
    std::string csv = out.str();
    std::istringstream is(csv);
    std::string header, row;
    std::getline(is, header);
    std::getline(is, row);
    std::vector<std::string> cells;
    std::stringstream rs(row);
    for (std::string c; std::getline(rs, c, ',');) cells.push_back(c);
    if (cells.size() > 4) cells[4] = "-";
    std::string joined;
    for (const auto& c : cells) joined += c + ",";
    rec_s("run_match.csv", header + "\n" + joined);
  }

  // 2. run_pipeline / match_stereo on the same pair (GrayImage via the
  // reference's own loader: to_grayscale of the decoded rasters)
  auto [left, right] = load_stereo_pair(argv[2], argv[3]);
  const CalibrationFile calib = load_calibration(argv[4]);
  const CameraParams cam{calib.focal_px, calib.baseline_mm};
  double gsum = 0.0;
  long long gvalid = 0;
  for (int y = 0; y < left.height; ++y)
    for (int x = 0; x < left.width; ++x)
      if (left.valid_at(x, y)) {
        gsum += left.at(x, y);
        ++gvalid;
      }
  rec_d("gray.sum", gsum);
  rec_i("gray.valid", gvalid);
  rec("gray.left", 2, left.data.data(), left.data.size() * 4, 1);

  const PipelineOutput po = run_pipeline(left, right, cfg, cam);
  rec_field("pipe.disparity", po.disparity);
  rec_field("pipe.probability", po.probability);
  rec_field("pipe.depth", po.depth.depth);
  rec_i("pipe.has_sigma", po.depth.has_sigma);
  if (po.depth.has_sigma) rec_field("pipe.sigma", po.depth.sigma, 1);
  rec_stats("pipe.stats", po.stats);

  const MatchResult mr = match_stereo(left, right, cfg);
  rec_field("match.disparity", mr.disparity);
  rec_field("match.probability", mr.probability);
  rec_i("match.has_variance", mr.has_variance);
  if (mr.has_variance) rec_field("match.var_disp", mr.var_disp, 1);
  rec_stats("match.stats", mr.stats);
  const LevelEstimate& f = mr.finest;
  rec_i("finest.level_exp", f.level_exp);
  rec_i("finest.width", f.width);
  rec_i("finest.height", f.height);
  rec_field("finest.disparity", f.disparity);
  rec_field("finest.probability", f.probability);
  rec_i("finest.has_variance", f.has_variance);
  if (f.has_variance) rec_field("finest.var_disp", f.var_disp, 1);
  {
    std::vector<double> exact, approx;
    std::vector<std::int64_t> flags;
    for (const PatchEstimate& p : f.patches) {
      for (double v : {p.cx, p.cy, p.u, p.prob, p.posterior}) exact.push_back(v);
      approx.push_back(p.sigma_k);
      flags.push_back(p.has_sigma);
    }
    rec_i("finest.n_patches", std::int64_t(f.patches.size()));
    rec("finest.patches", 0, exact.data(), exact.size(), 8);
    rec("finest.sigma_k", 1, approx.data(), approx.size(), 8);
    rec("finest.has_sigma", 3, flags.data(), flags.size(), 8);
  }

  // 2b. masked inputs (GrayImage validity, inc/image.hpp:21-26): an invalid
  // block in each view, as an RGBA alpha of 0 would give
  {
    GrayImage ml = left, mr = right;
    for (int y = left.height / 3; y < left.height / 2; ++y)
      for (int x = left.width / 4; x < left.width / 3; ++x) {
        ml.valid[std::size_t(y) * ml.width + x] = 0;
        mr.valid[std::size_t(y) * mr.width + x + 7] = 0;
      }
    const PipelineOutput mo = run_pipeline(ml, mr, cfg, cam);
    rec_field("masked.disparity", mo.disparity);
    rec_field("masked.depth", mo.depth.depth);
    rec_stats("masked.stats", mo.stats);
    const MatchResult mm = match_stereo(ml, mr, cfg);
    rec_field("masked.match", mm.disparity);
    rec_i("masked.finest_patches", std::int64_t(mm.finest.patches.size()));
  }

  // 3. run_benchmark (src/bench.cpp) over rendered scenes (src/synth.cpp)
  std::vector<SceneSpec> scenes(3);
  scenes[0].name = "plane";
  scenes[0].disparity = 6.0;
  scenes[1].name = "sphere";
  scenes[1].surface = SurfaceKind::sphere;
  scenes[1].shading = ShadingKind::nonlambertian;
  scenes[2].name = "slanted";
  scenes[2].surface = SurfaceKind::slanted_plane;
  scenes[2].disparity_gradient = 0.01;
  scenes[2].texture = TextureKind::checker;
  scenes[2].noise_std = 0.01;
  // the reference's default 5-level pyramid needs >= 320 px at the coarsest
  // level times 2^5 / patch: full-size scenes for config 4
  const int sw = config == 4 ? 640 : 320, sh = config == 4 ? 480 : 240;
  for (auto& s : scenes) {
    s.width = sw;
    s.height = sh;
  }
  const BenchResult br = run_benchmark(scenes, cfg, 2);
  for (const FrameMetrics& m : br.frames) {
    rec_s("bench.frame", m.frame);
    rec_d("bench.mean_err", m.mean_err, var_kind);
    rec_d("bench.median_err", m.median_err, var_kind);
    rec_i("bench.valid_px", m.valid_px);
    rec_d("bench.coverage", m.coverage_rate, 1);
    rec_i("bench.has_errors", m.has_errors);
  }
  rec_d("bench.avg_mean_err", br.aggregate.mean_err, var_kind);
  rec_i("bench.avg_valid_px", br.aggregate.valid_px);

  // 4. the CLI's bench body (src/runner.cpp:164-183) on scene files
  const std::string dims = config == 4 ? "width = 640\nheight = 480\n" : "width = 256\nheight = 192\n";
  write_scene(dir + "/s1.txt", "name = s1\nsurface = plane\ndisparity = 5\n" + dims);
  write_scene(dir + "/s2.txt", "name = s2\nsurface = sphere\nshading = nonlambertian\n" + dims);
  BenchArgs ba;
  ba.scene_paths = {dir + "/s1.txt", dir + "/s2.txt"};
  ba.out_csv = dir + "/bench.csv";
  ba.repetitions = 1;
  ba.cfg = cfg;
  std::ostringstream bout, berr;
  rec_i("run_bench.rc", run_bench(ba, bout, berr));

  // 5. error behaviour at the boundary
  PipelineConfig bad = cfg;
  bad.overlap = 1.5;
  rec_s("err.validate", error_class([&] { validate(bad); }));
  rec_s("err.run_pipeline_config", error_class([&] { (void)run_pipeline(left, right, bad, cam); }));
  GrayImage small = make_gray(left.width / 2, left.height);
  rec_s("err.size_mismatch", error_class([&] { (void)run_pipeline(left, small, cfg, cam); }));
  GrayImage t1 = make_gray(12, 12, 0.5f), t2 = make_gray(12, 12, 0.5f);
  rec_s("err.too_small", error_class([&] { (void)match_stereo(t1, t2, cfg); }));
  Raster two{4, 4, 2, std::vector<std::uint8_t>(32, 7)};
  rec_s("err.channels", error_class([&] { (void)to_grayscale(two); }));
  Raster rgba{3, 2, 4, {10, 20, 30, 255, 1, 2, 3, 0, 200, 100, 50, 9,
                        0, 0, 0, 0, 255, 255, 255, 255, 9, 8, 7, 6}};
  const GrayImage g4 = to_grayscale(rgba);
  rec("gray.rgba", 2, g4.data.data(), g4.data.size() * 4, 1);
  rec("gray.rgba_valid", 2, g4.valid.data(), g4.valid.size(), 1);
  MatchArgs missing = ma;
  missing.left_path = dir + "/does_not_exist.pgm";
  std::ostringstream mo, me;
  rec_i("err.run_match_missing", run_match(missing, mo, me));
  g_dump.close();
  std::printf("caller done: %s\n", dir.c_str());
  return 0;
}
