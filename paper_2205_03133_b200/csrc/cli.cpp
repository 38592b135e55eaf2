// cli.cpp -- pstereo_gpu_cli: the reference's command line (src/runner.cpp,
// inc/pstereo/runner.hpp) on the B200 path.
//
//   pstereo_gpu_cli [--config FILE.ini] match LEFT RIGHT --calib FILE
//                   [--out-dir DIR] [--frame LABEL] [pipeline flags]
//   pstereo_gpu_cli [--config FILE.ini] bench SCENE... [--out CSV] [--reps N]
//                   [pipeline flags]
//
// Pipeline flags are attach_pipeline_flags' (src/runner.cpp:17-66); --config
// reads an INI file with [match] / [bench] sections whose keys are the long
// flag names (flags on the command line override it). Exit codes follow
// inc/pstereo/runner.hpp:16-19: 0 ok, 2 ConfigError (and usage errors),
// 3 IoError, 4 DegenerateInputError, 1 anything else.
//
// `match` decodes the images on the host, converts them to grayscale on the
// device (pstereo_gpu_match_u8) and asks the kernels for the PFM payloads
// directly: fp32, -1 at invalid pixels, rows bottom to top (fill_invalid +
// flip_rows), so writing a map is a header plus one fwrite.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/pstereo_gpu.hpp"

namespace {

using namespace pstereo::gpu;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string trim(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

std::string norm_key(std::string k) {
  for (char& c : k)
    if (c == '_') c = '-';
  return k;
}

double to_double(const std::string& k, const std::string& v) {
  try {
    size_t used = 0;
    const double d = std::stod(v, &used);
    if (used != v.size()) throw std::invalid_argument(v);
    return d;
  } catch (const std::exception&) {
    throw UsageError("--" + k + ": '" + v + "' is not a number");
  }
}

long long to_int(const std::string& k, const std::string& v) {
  try {
    size_t used = 0;
    const long long d = std::stoll(v, &used);
    if (used != v.size()) throw std::invalid_argument(v);
    return d;
  } catch (const std::exception&) {
    throw UsageError("--" + k + ": '" + v + "' is not an integer");
  }
}

bool to_bool(const std::string& v) {
  return v == "1" || v == "true" || v == "on" || v == "yes";
}

// attach_pipeline_flags, src/runner.cpp:17-66. Returns false if k is not one.
bool set_pipeline(PipelineConfig& c, const std::string& k, const std::string& v) {
  if (k == "coarsest-exp") c.coarsest_exp = int(to_int(k, v));
  else if (k == "finest-exp") c.finest_exp = int(to_int(k, v));
  else if (k == "patch-size") c.patch_size = int(to_int(k, v));
  else if (k == "overlap") c.overlap = to_double(k, v);
  else if (k == "min-iterations") c.min_iterations = int(to_int(k, v));
  else if (k == "max-iterations") c.max_iterations = int(to_int(k, v));
  else if (k == "early-stop-good") c.early_stop_good = to_double(k, v);
  else if (k == "early-stop-bad") c.early_stop_bad = to_double(k, v);
  else if (k == "early-stop-improve") c.early_stop_improve = to_double(k, v);
  else if (k == "window-offsets") {
    c.window_offsets.clear();
    std::stringstream ss(v);
    std::string item;
    while (std::getline(ss, item, ',')) c.window_offsets.push_back(to_double(k, trim(item)));
  } else if (k == "sigma-s") c.sigma_s = to_double(k, v);
  else if (k == "pixel-threshold") c.pixel_threshold = to_double(k, v);
  else if (k == "gamma") c.gamma = to_double(k, v);
  else if (k == "valid-patch-ratio") c.valid_patch_ratio = to_double(k, v);
  else if (k == "estimate-variance") c.estimate_variance = to_bool(v);
  else if (k == "threads") c.threads = int(to_int(k, v));
  else if (k == "seed") c.seed = std::uint64_t(to_int(k, v));
  else return false;
  return true;
}

struct Args {
  std::string sub;
  std::vector<std::string> positional;
  std::map<std::string, std::string> opts;  // long name -> value ("1" for flags)
};

// INI sections [match] / [bench] (CLI11 config, src/runner.cpp:75-80)
std::map<std::string, std::map<std::string, std::string>> read_ini(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open config " + path);
  std::map<std::string, std::map<std::string, std::string>> out;
  std::string line, section;
  while (std::getline(in, line)) {
    const size_t h = line.find_first_of("#;");
    if (h != std::string::npos) line.erase(h);
    line = trim(line);
    if (line.empty()) continue;
    if (line.front() == '[' && line.back() == ']') {
      section = trim(line.substr(1, line.size() - 2));
      continue;
    }
    const size_t eq = line.find('=');
    if (eq == std::string::npos) throw ConfigError(path + ": expected 'key = value'");
    std::string v = trim(line.substr(eq + 1));
    if (v.size() >= 2 && v.front() == '"' && v.back() == '"') v = v.substr(1, v.size() - 2);
    if (v.size() >= 2 && v.front() == '[' && v.back() == ']') v = v.substr(1, v.size() - 2);
    out[section][norm_key(trim(line.substr(0, eq)))] = v;
  }
  return out;
}

Args parse(int argc, char** argv) {
  Args a;
  std::string config;
  std::map<std::string, std::string> cli;
  static const char* flags[] = {"estimate-variance"};
  for (int i = 1; i < argc; ++i) {
    std::string t = argv[i];
    if (t.rfind("--", 0) == 0) {
      std::string k = t.substr(2), v;
      const size_t eq = k.find('=');
      bool is_flag = false;
      for (const char* f : flags) is_flag = is_flag || k == f;
      if (eq != std::string::npos) {
        v = k.substr(eq + 1);
        k = k.substr(0, eq);
      } else if (is_flag) {
        v = "1";
      } else {
        if (i + 1 >= argc) throw UsageError("--" + k + " needs a value");
        v = argv[++i];
      }
      k = norm_key(k);
      if (k == "config") config = v;
      else cli[k] = v;
    } else if (a.sub.empty()) {
      a.sub = t;
    } else {
      a.positional.push_back(t);
    }
  }
  if (a.sub != "match" && a.sub != "bench")
    throw UsageError("a subcommand is required: match or bench");
  if (!config.empty()) {
    const auto ini = read_ini(config);
    const auto it = ini.find(a.sub);
    if (it != ini.end()) a.opts = it->second;
  }
  for (const auto& kv : cli) a.opts[kv.first] = kv.second;  // flags override the file
  return a;
}

int run_match(const Args& a, std::ostream& out) {
  if (a.positional.size() != 2) throw UsageError("match needs LEFT and RIGHT images");
  PipelineConfig cfg;
  std::string calib, out_dir = "out", frame;
  for (const auto& kv : a.opts) {
    if (kv.first == "calib") calib = kv.second;
    else if (kv.first == "out-dir") out_dir = kv.second;
    else if (kv.first == "frame") frame = kv.second;
    else if (!set_pipeline(cfg, kv.first, kv.second))
      throw UsageError("match: unknown option --" + kv.first);
  }
  if (calib.empty()) throw UsageError("match: --calib is required");
  validate(cfg);
  const std::string& lp = a.positional[0];
  const std::string& rp = a.positional[1];
  const Raster L = load_image(lp), R = load_image(rp);
  // load_stereo_pair (src/io.cpp:265-280): sizes must agree
  if (L.width != R.width || L.height != R.height)
    throw IoError(IoErrorKind::dimension_mismatch, lp + " is " + std::to_string(L.width) + "x" + std::to_string(L.height) +
                  " but " + rp + " is " + std::to_string(R.width) + "x" +
                  std::to_string(R.height));
  if (L.channels != R.channels)
    throw IoError(IoErrorKind::dimension_mismatch, lp + " and " + rp + " differ in channel count");
  const CalibrationFile cal = load_calibration(calib);
  if (cal.width != L.width || cal.height != L.height)
    throw ConfigError("calibration is for " + std::to_string(cal.width) + "x" +
                      std::to_string(cal.height) + ", images are " + std::to_string(L.width) +
                      "x" + std::to_string(L.height));
  const int w = L.width, h = L.height;
  const std::size_t px = std::size_t(w) * h;
  pstereo_ctx* ctx = detail::context_for(detail::to_c(cfg), w, h, 1);
  std::vector<float> disp(px), depth(px), sigma(cfg.estimate_variance ? px : 0);
  std::vector<std::uint8_t> dvalid(px);
  pstereo_outputs o{};
  o.dtype = PSTEREO_F32;
  o.disparity = disp.data();
  o.disparity_valid = dvalid.data();
  o.depth = depth.data();
  if (cfg.estimate_variance) o.depth_sigma = sigma.data();
  o.fill_invalid = 1;
  o.invalid_value = -1.0;
  o.flip_rows = 1;
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = pstereo_gpu_match_u8(ctx, 1, w, h, L.channels, L.pixels.data(),
                                      R.pixels.data(), 0, cal.focal_px, cal.baseline_mm, &o,
                                      nullptr);
  const auto t1 = std::chrono::steady_clock::now();
  if (rc) detail::raise(rc, pstereo_gpu_last_error(ctx));
  std::error_code ec;
  std::filesystem::create_directories(out_dir, ec);
  if (ec) throw IoError(IoErrorKind::write_failure, "cannot create " + out_dir + ": " + ec.message());
  const std::string dir = out_dir + "/";
  char msg[512];
  auto put = [&](const std::vector<float>& v, const std::string& name) {
    detail::raise_io(
        pstereo_write_pfm((dir + name).c_str(), w, h, v.data(), nullptr, 1, msg, sizeof msg),
        msg);
  };
  put(disp, "disparity.pfm");
  put(depth, "depth.pfm");
  if (cfg.estimate_variance) put(sigma, "sigma.pfm");
  FrameMetrics row;
  row.frame = frame.empty() ? std::filesystem::path(lp).stem().string() : frame;
  long long valid = 0;
  for (std::uint8_t v : dvalid) valid += v != 0;
  row.valid_px = valid;
  row.runtime_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  out << metrics_csv_header() << "\n" << format_metrics_row(row) << "\n";
  return 0;
}

int run_bench(const Args& a, std::ostream& out) {
  PipelineConfig cfg;
  std::string out_csv = "metrics.csv";
  int reps = 10;
  for (const auto& kv : a.opts) {
    if (kv.first == "out") out_csv = kv.second;
    else if (kv.first == "reps") reps = int(to_int(kv.first, kv.second));
    else if (!set_pipeline(cfg, kv.first, kv.second))
      throw UsageError("bench: unknown option --" + kv.first);
  }
  if (a.positional.empty()) throw UsageError("bench needs at least one scene file");
  validate(cfg);
  std::vector<SceneSpec> scenes;
  for (const std::string& p : a.positional) {
    SceneSpec s = load_scene_spec(p);
    if (!s.seed_explicit) s.seed = cfg.seed;  // src/runner.cpp:166-168
    scenes.push_back(s);
  }
  const BenchResult res = run_benchmark(scenes, cfg, reps);
  std::vector<FrameMetrics> rows = res.frames;
  rows.push_back(res.aggregate);
  write_metrics_csv(rows, out_csv);
  out << metrics_csv_header() << "\n";
  for (const FrameMetrics& r : rows) out << format_metrics_row(r) << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  // run_guarded, src/runner.cpp:104-124
  try {
    const Args a = parse(argc, argv);
    return a.sub == "match" ? run_match(a, std::cout) : run_bench(a, std::cout);
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const ConfigError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const IoError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const DegenerateInputError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  } catch (const std::exception& e) {
    std::cerr << "internal error: " << e.what() << "\n";
    return 1;
  }
}
