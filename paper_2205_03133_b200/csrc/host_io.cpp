// host_io.cpp -- the caller side of the matching core, host C++ (SURVEY.md
// §8f rows 3 and 4): the "key = value" reader shared by calibration and
// scene files, scene specs, image decoding (PGM/PPM, PNG), the PFM writer /
// reader and the metrics CSV, with the reference's semantics (src/io.cpp,
// src/synth.cpp:289-393). The reference's error classes map to return codes:
// ConfigError -> PSTEREO_ECONFIG, IoError -> PSTEREO_EIO.
#include <zlib.h>

#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <system_error>
#include <utility>
#include <vector>

#include "../../include/pstereo_gpu.h"

namespace {

struct Error : std::runtime_error {
  int code;
  int kind;  // IoErrorKind for PSTEREO_EIO (inc/errors.hpp:14-19)
  Error(int c, const std::string& m, int k = -1) : std::runtime_error(m), code(c), kind(k) {}
};

thread_local int t_io_kind = -1;

[[noreturn]] void config_error(const std::string& m) { throw Error(PSTEREO_ECONFIG, m); }
[[noreturn]] void io_error(int kind, const std::string& m) { throw Error(PSTEREO_EIO, m, kind); }

template <class F>
int guarded(char* msg, size_t cap, F&& body) {
  auto put = [&](const char* m) {
    if (msg && cap) {
      std::snprintf(msg, cap, "%s", m);
    }
  };
  t_io_kind = -1;
  try {
    body();
    put("");
    return PSTEREO_OK;
  } catch (const Error& e) {
    put(e.what());
    t_io_kind = e.kind;
    return e.code;
  } catch (const std::exception& e) {
    put(e.what());
    return PSTEREO_EINTERNAL;
  }
}

std::string trim(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

// ---- key = value files (src/io.cpp:24-136) --------------------------------

struct Kv {
  std::vector<std::pair<std::string, std::string>> entries;
  const std::string* find(const std::string& k) const {
    for (const auto& e : entries)
      if (e.first == k) return &e.second;
    return nullptr;
  }
};

Kv parse_kv_text(const std::string& text, const std::string& origin) {
  Kv kv;
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    const size_t hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    line = trim(line);
    if (line.empty()) continue;
    const size_t eq = line.find('=');
    if (eq == std::string::npos)
      config_error(origin + ":" + std::to_string(lineno) + ": expected 'key = value', got '" +
                   line + "'");
    std::string key = trim(line.substr(0, eq));
    std::string value = trim(line.substr(eq + 1));
    if (key.empty() || value.empty())
      config_error(origin + ":" + std::to_string(lineno) + ": empty key or value");
    if (kv.find(key))
      config_error(origin + ":" + std::to_string(lineno) + ": duplicate key '" + key + "'");
    kv.entries.emplace_back(std::move(key), std::move(value));
  }
  return kv;
}

std::string read_text(const std::string& path) {
  std::ifstream in(path);
  if (!in) io_error(PSTEREO_IO_MISSING_FILE, "cannot open " + path);
  std::ostringstream buf;
  buf << in.rdbuf();
  return buf.str();
}

double parse_double(const std::string& key, const std::string& text) {
  const std::string t = trim(text);
  double v = 0.0;
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  if (r.ec != std::errc{} || r.ptr != t.data() + t.size())
    config_error("key '" + key + "': cannot parse '" + text + "' as a number");
  return v;
}

long long parse_int(const std::string& key, const std::string& text) {
  const std::string t = trim(text);
  long long v = 0;
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  if (r.ec != std::errc{} || r.ptr != t.data() + t.size())
    config_error("key '" + key + "': cannot parse '" + text + "' as an integer");
  return v;
}

double kv_double(const Kv& kv, const std::string& key) {
  const std::string* v = kv.find(key);
  if (!v) config_error("missing key '" + key + "'");
  return parse_double(key, *v);
}
double kv_double_or(const Kv& kv, const std::string& key, double f) {
  const std::string* v = kv.find(key);
  return v ? parse_double(key, *v) : f;
}
long long kv_int(const Kv& kv, const std::string& key) {
  const std::string* v = kv.find(key);
  if (!v) config_error("missing key '" + key + "'");
  return parse_int(key, *v);
}
long long kv_int_or(const Kv& kv, const std::string& key, long long f) {
  const std::string* v = kv.find(key);
  return v ? parse_int(key, *v) : f;
}
std::string kv_string_or(const Kv& kv, const std::string& key, const std::string& f) {
  const std::string* v = kv.find(key);
  return v ? *v : f;
}

// ---- scene specs (src/synth.cpp:289-393) ----------------------------------

const char* kSceneKeys[] = {
    "name",          "surface",          "disparity",         "disparity0",
    "disparity_gradient", "sphere_depth", "sphere_radius",    "background_depth",
    "texture",       "texture_scale",    "texture_octaves",   "shading",
    "ambient",       "highlight_strength", "highlight_falloff", "noise_std",
    "seed",          "focal_px",         "baseline",          "width",
    "height",
};

void validate_scene(const pstereo_scene_spec& s, const std::string& path) {
  if (s.width < 2 || s.height < 2) config_error(path + ": width/height must be >= 2");
  if (!(s.focal_px > 0.0) || !(s.baseline > 0.0))
    config_error(path + ": focal_px and baseline must be positive");
  if (s.surface == PSTEREO_SURFACE_PLANE && !(s.disparity > 0.0))
    config_error(path + ": disparity must be positive");
  if (s.surface == PSTEREO_SURFACE_SLANTED) {
    const double dend = s.disparity0 + s.disparity_gradient * (s.width - 1);
    if (!(s.disparity0 > 0.0) || !(dend > 0.0))
      config_error(path + ": slanted plane disparity must stay positive");
    if (!(std::fabs(s.disparity_gradient) < 0.5))
      config_error(path + ": |disparity_gradient| must be < 0.5 px per px");
  }
  if (s.surface == PSTEREO_SURFACE_SPHERE &&
      (!(s.sphere_depth > 0.0) || !(s.sphere_radius > 0.0) ||
       !(s.background_depth > s.sphere_depth)))
    config_error(path + ": sphere must sit in front of the background");
  if (s.texture_octaves < 1 || s.texture_octaves > 8)
    config_error(path + ": texture_octaves must be in 1..8");
  if (!(s.texture_scale > 1.0)) config_error(path + ": texture_scale must be > 1 px");
  if (s.noise_std < 0.0) config_error(path + ": noise_std must be >= 0");
  if (s.surface < 0 || s.surface > 2 || s.texture < 0 || s.texture > 2 || s.shading < 0 ||
      s.shading > 1)
    config_error(path + ": unknown surface / texture / shading kind");
}

void load_scene(const std::string& path, pstereo_scene_spec* out) {
  const Kv kv = parse_kv_text(read_text(path), path);
  for (const auto& e : kv.entries) {
    bool known = false;
    for (const char* k : kSceneKeys) known = known || e.first == k;
    if (!known) config_error(path + ": unknown scene key '" + e.first + "'");
  }
  pstereo_scene_spec s;
  pstereo_scene_default(&s);
  const std::string name = kv_string_or(kv, "name", "scene");
  std::snprintf(s.name, sizeof s.name, "%s", name.c_str());
  const std::string surface = kv_string_or(kv, "surface", "plane");
  if (surface == "plane") s.surface = PSTEREO_SURFACE_PLANE;
  else if (surface == "slanted_plane") s.surface = PSTEREO_SURFACE_SLANTED;
  else if (surface == "sphere") s.surface = PSTEREO_SURFACE_SPHERE;
  else config_error(path + ": unknown surface '" + surface + "'");
  s.disparity = kv_double_or(kv, "disparity", s.disparity);
  s.disparity0 = kv_double_or(kv, "disparity0", s.disparity0);
  s.disparity_gradient = kv_double_or(kv, "disparity_gradient", s.disparity_gradient);
  s.sphere_depth = kv_double_or(kv, "sphere_depth", s.sphere_depth);
  s.sphere_radius = kv_double_or(kv, "sphere_radius", s.sphere_radius);
  s.background_depth = kv_double_or(kv, "background_depth", s.background_depth);
  const std::string texture = kv_string_or(kv, "texture", "perlin");
  if (texture == "perlin") s.texture = PSTEREO_TEXTURE_PERLIN;
  else if (texture == "checker") s.texture = PSTEREO_TEXTURE_CHECKER;
  else if (texture == "constant") s.texture = PSTEREO_TEXTURE_CONSTANT;
  else config_error(path + ": unknown texture '" + texture + "'");
  s.texture_scale = kv_double_or(kv, "texture_scale", s.texture_scale);
  s.texture_octaves = int(kv_int_or(kv, "texture_octaves", s.texture_octaves));
  const std::string shading = kv_string_or(kv, "shading", "diffuse");
  if (shading == "diffuse") s.shading = PSTEREO_SHADING_DIFFUSE;
  else if (shading == "nonlambertian") s.shading = PSTEREO_SHADING_NONLAMBERTIAN;
  else config_error(path + ": unknown shading '" + shading + "'");
  s.ambient = kv_double_or(kv, "ambient", s.ambient);
  s.highlight_strength = kv_double_or(kv, "highlight_strength", s.highlight_strength);
  s.highlight_falloff = kv_double_or(kv, "highlight_falloff", s.highlight_falloff);
  s.noise_std = kv_double_or(kv, "noise_std", s.noise_std);
  s.seed_explicit = kv.find("seed") != nullptr;
  s.seed = uint64_t(kv_int_or(kv, "seed", (long long)s.seed));
  s.focal_px = kv_double_or(kv, "focal_px", s.focal_px);
  s.baseline = kv_double_or(kv, "baseline", s.baseline);
  s.width = int(kv_int_or(kv, "width", s.width));
  s.height = int(kv_int_or(kv, "height", s.height));
  validate_scene(s, path);
  *out = s;
}

// ---- images (src/io.cpp:141-263) ------------------------------------------

std::vector<uint8_t> read_bytes(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) io_error(PSTEREO_IO_MISSING_FILE, "cannot open " + path);
  return std::vector<uint8_t>((std::istreambuf_iterator<char>(in)),
                              std::istreambuf_iterator<char>());
}

struct Raster {
  int w = 0, h = 0, c = 0;
  std::vector<uint8_t> px;
};

// decode_pnm, src/io.cpp:151-198
Raster decode_pnm(const std::string& path, const std::vector<uint8_t>& b) {
  auto fail = [&](const std::string& why) { io_error(PSTEREO_IO_DECODE_FAILURE, path + ": " + why); };
  size_t pos = 0;
  auto next_token = [&]() {
    while (pos < b.size()) {
      const char ch = char(b[pos]);
      if (ch == '#') {
        while (pos < b.size() && b[pos] != '\n') ++pos;
      } else if (std::isspace(static_cast<unsigned char>(ch))) {
        ++pos;
      } else {
        break;
      }
    }
    const size_t start = pos;
    while (pos < b.size() && !std::isspace(static_cast<unsigned char>(b[pos]))) ++pos;
    return std::string(b.begin() + start, b.begin() + pos);
  };
  const std::string magic = next_token();
  const int channels = magic == "P5" ? 1 : magic == "P6" ? 3 : 0;
  if (channels == 0) fail("not a binary PGM/PPM");
  int w = 0, h = 0, maxval = 0;
  try {
    w = std::stoi(next_token());
    h = std::stoi(next_token());
    maxval = std::stoi(next_token());
  } catch (const std::exception&) {
    fail("malformed header");
  }
  if (w <= 0 || h <= 0) fail("bad dimensions");
  if (maxval <= 0 || maxval > 255) fail("only 8-bit samples supported");
  ++pos;
  const size_t need = size_t(w) * h * channels;
  if (b.size() < pos + need) fail("truncated pixel data");
  Raster r;
  r.w = w;
  r.h = h;
  r.c = channels;
  r.px.assign(b.begin() + pos, b.begin() + pos + need);
  return r;
}

// PNG, decoded to what decode_png (src/io.cpp:200-249) asks libpng for:
// palette -> RGB, gray < 8 bit expanded to 8, tRNS -> alpha, 16 -> 8 bit
// (high byte, png_set_strip_16), gray+alpha -> RGBA; Adam7 de-interlaced.
uint32_t be32(const uint8_t* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | p[3];
}

uint8_t paeth(int a, int b, int c) {
  const int p = a + b - c;
  const int pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  if (pa <= pb && pa <= pc) return uint8_t(a);
  if (pb <= pc) return uint8_t(b);
  return uint8_t(c);
}

Raster decode_png(const std::string& path, const std::vector<uint8_t>& b,
                  bool header_only = false) {
  auto fail = [&](const std::string& why) { io_error(PSTEREO_IO_DECODE_FAILURE, path + ": " + why); };
  size_t pos = 8;
  uint32_t W = 0, H = 0;
  int depth = 0, ctype = -1, interlace = 0;
  std::vector<uint8_t> plte, trns, idat;
  bool seen_end = false;
  while (pos + 12 <= b.size() && !seen_end) {
    const uint32_t len = be32(&b[pos]);
    if (pos + 12 + size_t(len) > b.size()) fail("PNG decode failed (truncated chunk)");
    const uint8_t* type = &b[pos + 4];
    const uint8_t* data = &b[pos + 8];
    const bool critical = !(type[0] & 0x20);
    const uint32_t crc = be32(&b[pos + 8 + len]);
    if (critical && uint32_t(crc32(crc32(0L, Z_NULL, 0), type, len + 4)) != crc)
      fail("PNG decode failed (CRC error)");
    const std::string t(reinterpret_cast<const char*>(type), 4);
    if (t == "IHDR") {
      if (len != 13) fail("PNG decode failed (IHDR)");
      W = be32(data);
      H = be32(data + 4);
      depth = data[8];
      ctype = data[9];
      interlace = data[12];
      if (data[10] != 0 || data[11] != 0 || interlace > 1) fail("PNG decode failed (IHDR)");
    } else if (t == "PLTE") {
      plte.assign(data, data + len);
    } else if (t == "tRNS") {
      trns.assign(data, data + len);
    } else if (t == "IDAT") {
      idat.insert(idat.end(), data, data + len);
    } else if (t == "IEND") {
      seen_end = true;
    } else if (critical) {
      fail("PNG decode failed (unknown critical chunk)");
    }
    pos += 12 + size_t(len);
  }
  if (ctype < 0 || W == 0 || H == 0 || W > (1u << 24) || H > (1u << 24))
    fail("PNG decode failed (no IHDR)");
  if (uint64_t(W) * H > (uint64_t(1) << 28)) fail("PNG decode failed (image too large)");
  int spp = 0;  // samples per pixel in the file
  switch (ctype) {
    case 0: spp = 1; break;
    case 2: spp = 3; break;
    case 3: spp = 1; break;
    case 4: spp = 2; break;
    case 6: spp = 4; break;
    default: fail("PNG decode failed (color type)");
  }
  const bool depth_ok = (ctype == 0 && (depth == 1 || depth == 2 || depth == 4 || depth == 8 ||
                                        depth == 16)) ||
                        (ctype == 3 && (depth == 1 || depth == 2 || depth == 4 || depth == 8)) ||
                        ((ctype == 2 || ctype == 4 || ctype == 6) && (depth == 8 || depth == 16));
  if (!depth_ok) fail("PNG decode failed (bit depth)");
  if (ctype == 3 && (plte.empty() || plte.size() % 3)) fail("PNG decode failed (PLTE)");
  if (header_only) {  // dimensions and output channels without inflating the data
    Raster r;
    r.w = int(W);
    r.h = int(H);
    r.c = ctype == 3 ? (trns.empty() ? 3 : 4)
          : ctype == 0 ? (trns.size() >= 2 ? 4 : 1)
          : ctype == 2 ? (trns.size() >= 6 ? 4 : 3)
          : 4;
    return r;
  }
  const int bpp_bits = spp * depth;
  const size_t filt_bpp = size_t(std::max(1, bpp_bits / 8));
  // inflate
  const int passes = interlace ? 7 : 1;
  static const int sx0[7] = {0, 4, 0, 2, 0, 1, 0}, sy0[7] = {0, 0, 4, 0, 2, 0, 1};
  static const int dx[7] = {8, 8, 4, 4, 2, 2, 1}, dy[7] = {8, 8, 8, 4, 4, 2, 2};
  size_t raw_size = 0;
  for (int p = 0; p < passes; ++p) {
    const uint32_t pw = interlace ? (W + dx[p] - 1 - sx0[p]) / dx[p] : W;
    const uint32_t ph = interlace ? (H + dy[p] - 1 - sy0[p]) / dy[p] : H;
    if (pw == 0 || ph == 0) continue;
    raw_size += size_t(ph) * (1 + (size_t(pw) * bpp_bits + 7) / 8);
  }
  std::vector<uint8_t> raw(raw_size);
  z_stream zs;
  std::memset(&zs, 0, sizeof zs);
  if (inflateInit(&zs) != Z_OK) fail("PNG decode failed (zlib)");
  zs.next_in = idat.data();
  zs.avail_in = uInt(idat.size());
  zs.next_out = raw.data();
  zs.avail_out = uInt(raw.size());
  const int zr = inflate(&zs, Z_FINISH);
  const size_t got = raw.size() - zs.avail_out;
  inflateEnd(&zs);
  if ((zr != Z_STREAM_END && zr != Z_BUF_ERROR && zr != Z_OK) || got != raw.size())
    fail("PNG decode failed (image data)");
  // unfilter each pass and scatter samples (16-bit kept for tRNS compare)
  std::vector<uint16_t> samples(size_t(W) * H * spp);
  size_t off = 0;
  for (int p = 0; p < passes; ++p) {
    const uint32_t pw = interlace ? (W + dx[p] - 1 - sx0[p]) / dx[p] : W;
    const uint32_t ph = interlace ? (H + dy[p] - 1 - sy0[p]) / dy[p] : H;
    if (pw == 0 || ph == 0) continue;
    const size_t stride = (size_t(pw) * bpp_bits + 7) / 8;
    std::vector<uint8_t> prev(stride, 0), cur(stride);
    for (uint32_t y = 0; y < ph; ++y) {
      const uint8_t f = raw[off];
      const uint8_t* src = &raw[off + 1];
      off += 1 + stride;
      for (size_t i = 0; i < stride; ++i) {
        const int a = i >= filt_bpp ? cur[i - filt_bpp] : 0;
        const int up = prev[i];
        const int c = i >= filt_bpp ? prev[i - filt_bpp] : 0;
        int v = src[i];
        switch (f) {
          case 0: break;
          case 1: v += a; break;
          case 2: v += up; break;
          case 3: v += (a + up) >> 1; break;
          case 4: v += paeth(a, up, c); break;
          default: fail("PNG decode failed (filter)");
        }
        cur[i] = uint8_t(v);
      }
      const uint32_t yy = interlace ? sy0[p] + y * dy[p] : y;
      for (uint32_t x = 0; x < pw; ++x) {
        const uint32_t xx = interlace ? sx0[p] + x * dx[p] : x;
        for (int s = 0; s < spp; ++s) {
          uint16_t v;
          if (depth == 16) {
            const size_t o = (size_t(x) * spp + s) * 2;
            v = uint16_t((cur[o] << 8) | cur[o + 1]);
          } else if (depth == 8) {
            v = cur[size_t(x) * spp + s];
          } else {
            const size_t bit = size_t(x) * depth;
            v = uint16_t((cur[bit / 8] >> (8 - depth - bit % 8)) & ((1 << depth) - 1));
          }
          samples[(size_t(yy) * W + xx) * spp + s] = v;
        }
      }
      std::swap(prev, cur);
    }
  }
  // colour conversion
  Raster r;
  r.w = int(W);
  r.h = int(H);
  const size_t n = size_t(W) * H;
  auto to8 = [&](uint16_t v) -> uint8_t {
    if (depth == 16) return uint8_t(v >> 8);
    if (depth == 8) return uint8_t(v);
    return uint8_t(v * (255 / ((1 << depth) - 1)));  // 1/2/4-bit gray expansion
  };
  if (ctype == 3) {
    const size_t ncol = plte.size() / 3;
    const bool alpha = !trns.empty();
    r.c = alpha ? 4 : 3;
    r.px.resize(n * r.c);
    for (size_t i = 0; i < n; ++i) {
      const size_t k = samples[i];
      uint8_t* o = &r.px[i * r.c];
      if (k < ncol) {
        o[0] = plte[3 * k];
        o[1] = plte[3 * k + 1];
        o[2] = plte[3 * k + 2];
      } else {
        o[0] = o[1] = o[2] = 0;
      }
      if (alpha) o[3] = k < trns.size() ? trns[k] : 255;
    }
  } else if (ctype == 0) {
    const bool key = trns.size() >= 2;
    const uint16_t kv = key ? uint16_t((trns[0] << 8) | trns[1]) : 0;
    r.c = key ? 4 : 1;  // gray + tRNS alpha -> gray+alpha -> RGBA
    r.px.resize(n * r.c);
    for (size_t i = 0; i < n; ++i) {
      const uint8_t g = to8(samples[i]);
      if (key) {
        uint8_t* o = &r.px[i * 4];
        o[0] = o[1] = o[2] = g;
        o[3] = samples[i] == kv ? 0 : 255;
      } else {
        r.px[i] = g;
      }
    }
  } else if (ctype == 2) {
    const bool key = trns.size() >= 6;
    r.c = key ? 4 : 3;
    r.px.resize(n * r.c);
    for (size_t i = 0; i < n; ++i) {
      const uint16_t* s = &samples[i * 3];
      uint8_t* o = &r.px[i * r.c];
      for (int c = 0; c < 3; ++c) o[c] = to8(s[c]);
      if (key) {
        const bool hit = s[0] == uint16_t((trns[0] << 8) | trns[1]) &&
                         s[1] == uint16_t((trns[2] << 8) | trns[3]) &&
                         s[2] == uint16_t((trns[4] << 8) | trns[5]);
        o[3] = hit ? 0 : 255;
      }
    }
  } else if (ctype == 4) {
    r.c = 4;
    r.px.resize(n * 4);
    for (size_t i = 0; i < n; ++i) {
      uint8_t* o = &r.px[i * 4];
      o[0] = o[1] = o[2] = to8(samples[i * 2]);
      o[3] = to8(samples[i * 2 + 1]);
    }
  } else {
    r.c = 4;
    r.px.resize(n * 4);
    for (size_t i = 0; i < n * 4; ++i) r.px[i] = to8(samples[i]);
  }
  return r;
}

// load_image, src/io.cpp:253-263 (header_only: dimensions and channels)
Raster load_image(const std::string& path, bool header_only = false) {
  const std::vector<uint8_t> b = read_bytes(path);
  static const uint8_t sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1A, '\n'};
  if (b.size() >= 8 && std::memcmp(b.data(), sig, 8) == 0)
    return decode_png(path, b, header_only);
  if (b.size() >= 2 && b[0] == 'P' && (b[1] == '5' || b[1] == '6')) return decode_pnm(path, b);
  io_error(PSTEREO_IO_DECODE_FAILURE, path + ": unrecognized image format (PNG/PGM/PPM supported)");
}

// ---- metrics CSV (src/io.cpp:346-439) -------------------------------------

const char kCsvHeader[] = "frame,mean_err,median_err,valid_px,runtime_ms,coverage_rate";

std::string format_double(double v) {
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, r.ptr);
}

std::string format_row(const pstereo_metrics_row& m) {
  std::string row = m.frame;
  row += ',';
  row += format_double(m.mean_err);
  row += ',';
  row += format_double(m.median_err);
  row += ',';
  row += std::to_string(m.valid_px);
  row += ',';
  row += format_double(m.runtime_ms);
  row += ',';
  row += format_double(m.coverage_rate);
  return row;
}

double parse_csv_double(const std::string& cell, const std::string& path) {
  if (cell == "nan" || cell == "-nan") return std::numeric_limits<double>::quiet_NaN();
  try {
    size_t used = 0;
    const double v = std::stod(cell, &used);
    if (used != cell.size()) throw std::invalid_argument(cell);
    return v;
  } catch (const std::exception&) {
    io_error(PSTEREO_IO_DECODE_FAILURE, path + ": bad numeric cell '" + cell + "'");
  }
}

std::vector<pstereo_metrics_row> read_csv(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) io_error(PSTEREO_IO_MISSING_FILE, "cannot open " + path);
  std::string line;
  if (!std::getline(in, line) || trim(line) != kCsvHeader)
    io_error(PSTEREO_IO_DECODE_FAILURE, path + ": missing metrics header");
  std::vector<pstereo_metrics_row> rows;
  while (std::getline(in, line)) {
    line = trim(line);
    if (line.empty()) continue;
    std::vector<std::string> cells;
    size_t start = 0;
    for (size_t i = 0; i <= line.size(); ++i)
      if (i == line.size() || line[i] == ',') {
        cells.push_back(line.substr(start, i - start));
        start = i + 1;
      }
    if (cells.size() != 6)
      io_error(PSTEREO_IO_DECODE_FAILURE, path + ": expected 6 cells, got " + std::to_string(cells.size()));
    pstereo_metrics_row m;
    std::memset(&m, 0, sizeof m);
    std::snprintf(m.frame, sizeof m.frame, "%s", cells[0].c_str());
    m.mean_err = parse_csv_double(cells[1], path);
    m.median_err = parse_csv_double(cells[2], path);
    try {
      m.valid_px = parse_int("valid_px", cells[3]);
    } catch (const Error& e) {
      io_error(PSTEREO_IO_DECODE_FAILURE, path + ": " + e.what());
    }
    m.runtime_ms = parse_csv_double(cells[4], path);
    m.coverage_rate = parse_csv_double(cells[5], path);
    m.has_errors = !std::isnan(m.mean_err);
    rows.push_back(m);
  }
  return rows;
}

}  // namespace

extern "C" {

int pstereo_last_io_kind(void) { return t_io_kind; }

void pstereo_scene_default(pstereo_scene_spec* s) {
  std::memset(s, 0, sizeof *s);
  std::snprintf(s->name, sizeof s->name, "scene");
  s->surface = PSTEREO_SURFACE_PLANE;
  s->disparity = 8.0;
  s->disparity0 = 8.0;
  s->disparity_gradient = 0.0;
  s->sphere_depth = 60.0;
  s->sphere_radius = 20.0;
  s->background_depth = 90.0;
  s->texture = PSTEREO_TEXTURE_PERLIN;
  s->texture_scale = 32.0;
  s->texture_octaves = 4;
  s->shading = PSTEREO_SHADING_DIFFUSE;
  s->ambient = 0.3;
  s->highlight_strength = 0.7;
  s->highlight_falloff = 6.0;
  s->noise_std = 0.0;
  s->seed = 1;
  s->seed_explicit = 0;
  s->focal_px = 500.0;
  s->baseline = 5.0;
  s->width = 640;
  s->height = 480;
}

int pstereo_scene_validate(const pstereo_scene_spec* s, char* msg, size_t cap) {
  return guarded(msg, cap, [&] {
    if (!s) config_error("null scene spec");
    validate_scene(*s, s->name);
  });
}

int pstereo_load_scene_spec(const char* path, pstereo_scene_spec* out, char* msg, size_t cap) {
  return guarded(msg, cap, [&] { load_scene(path, out); });
}

int pstereo_load_calibration(const char* path, double* focal_px, double* baseline_mm,
                             int* width, int* height, char* msg, size_t cap) {
  // load_calibration, src/io.cpp:266-281
  return guarded(msg, cap, [&] {
    const std::string p = path;
    const Kv kv = parse_kv_text(read_text(p), p);
    const double f = kv_double(kv, "focal_px");
    const double b = kv_double(kv, "baseline_mm");
    const int w = int(kv_int(kv, "width"));
    const int h = int(kv_int(kv, "height"));
    if (!(f > 0.0)) config_error(p + ": focal_px must be positive");
    if (!(b > 0.0)) config_error(p + ": baseline_mm must be positive");
    if (w <= 0 || h <= 0) config_error(p + ": width/height must be positive");
    *focal_px = f;
    *baseline_mm = b;
    *width = w;
    *height = h;
  });
}

int pstereo_load_image(const char* path, int* width, int* height, int* channels,
                       uint8_t* pixels, size_t cap, char* msg, size_t msg_cap) {
  return guarded(msg, msg_cap, [&] {
    const Raster r = load_image(path, pixels == nullptr);
    *width = r.w;
    *height = r.h;
    *channels = r.c;
    if (pixels) {
      if (cap < r.px.size()) throw Error(PSTEREO_EINTERNAL, "pixel buffer too small");
      std::memcpy(pixels, r.px.data(), r.px.size());
    }
  });
}

int pstereo_write_pfm(const char* path, int w, int h, const float* values, const uint8_t* valid,
                      int rows_bottom_up, char* msg, size_t cap) {
  // write_pfm, src/io.cpp:297-310
  return guarded(msg, cap, [&] {
    const std::string p = path;
    if (w < 0 || h < 0 || (!values && w * h > 0)) throw Error(PSTEREO_EINTERNAL, "bad PFM plane");
    std::ofstream out(p, std::ios::binary);
    if (!out) io_error(PSTEREO_IO_WRITE_FAILURE, "cannot write " + p);
    out << "Pf\n" << w << " " << h << "\n-1.0\n";
    if (!valid && rows_bottom_up) {
      out.write(reinterpret_cast<const char*>(values), std::streamsize(sizeof(float)) * w * h);
    } else {
      std::vector<float> row(static_cast<size_t>(w));
      for (int k = 0; k < h; ++k) {
        const int y = rows_bottom_up ? k : h - 1 - k;  // source row written k-th
        const float* src = values + size_t(y) * w;
        const uint8_t* ok = valid ? valid + size_t(y) * w : nullptr;
        for (int x = 0; x < w; ++x) row[size_t(x)] = (!ok || ok[x]) ? src[x] : -1.0f;
        out.write(reinterpret_cast<const char*>(row.data()),
                  std::streamsize(row.size() * sizeof(float)));
      }
    }
    if (!out) io_error(PSTEREO_IO_WRITE_FAILURE, "write failed: " + p);
  });
}

int pstereo_read_pfm(const char* path, int* width, int* height, float* values, size_t cap,
                     char* msg, size_t msg_cap) {
  // read_pfm, src/io.cpp:312-341
  return guarded(msg, msg_cap, [&] {
    const std::string p = path;
    std::ifstream in(p, std::ios::binary);
    if (!in) io_error(PSTEREO_IO_MISSING_FILE, "cannot open " + p);
    std::string magic;
    in >> magic;
    if (magic != "Pf") io_error(PSTEREO_IO_DECODE_FAILURE, p + ": not a grayscale PFM");
    int w = 0, h = 0;
    double scale = 0.0;
    in >> w >> h >> scale;
    if (!in || w <= 0 || h <= 0) io_error(PSTEREO_IO_DECODE_FAILURE, p + ": malformed header");
    if (!(scale < 0.0)) io_error(PSTEREO_IO_DECODE_FAILURE, p + ": big-endian PFM unsupported");
    in.get();
    *width = w;
    *height = h;
    if (!values) return;
    if (cap < size_t(w) * h) throw Error(PSTEREO_EINTERNAL, "value buffer too small");
    for (int y = h - 1; y >= 0; --y) {
      in.read(reinterpret_cast<char*>(values + size_t(y) * w), std::streamsize(w) * 4);
      if (!in) io_error(PSTEREO_IO_DECODE_FAILURE, p + ": truncated pixel data");
    }
  });
}

const char* pstereo_metrics_csv_header(void) { return kCsvHeader; }

int pstereo_format_metrics_row(const pstereo_metrics_row* row, char* buf, size_t cap) {
  const std::string s = format_row(*row);
  if (!buf || cap < s.size() + 1) return -1;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return int(s.size());
}

int pstereo_write_metrics_csv(const char* path, const pstereo_metrics_row* rows, int n_rows,
                              char* msg, size_t cap) {
  return guarded(msg, cap, [&] {
    const std::string p = path;
    std::ofstream out(p, std::ios::binary);
    if (!out) io_error(PSTEREO_IO_WRITE_FAILURE, "cannot write " + p);
    out << kCsvHeader << "\n";
    for (int i = 0; i < n_rows; ++i) out << format_row(rows[i]) << "\n";
    if (!out) io_error(PSTEREO_IO_WRITE_FAILURE, "write failed: " + p);
  });
}

int pstereo_read_metrics_csv(const char* path, pstereo_metrics_row* rows, int cap, int* n_rows,
                             char* msg, size_t msg_cap) {
  return guarded(msg, msg_cap, [&] {
    const std::vector<pstereo_metrics_row> r = read_csv(path);
    *n_rows = int(r.size());
    if (rows) {
      if (cap < int(r.size())) throw Error(PSTEREO_EINTERNAL, "row buffer too small");
      std::memcpy(rows, r.data(), r.size() * sizeof(pstereo_metrics_row));
    }
  });
}

}  // extern "C"
