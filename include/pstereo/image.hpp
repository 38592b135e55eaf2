// pstereo/image.hpp -- drop-in for proj/include/pstereo/image.hpp:12-45:
// Raster (decoder output), GrayImage (fp32 [0,1] + validity) with its
// accessors, make_gray and to_grayscale. to_grayscale runs the match path's
// k_gray_u8 kernel on the current device (Rec.601 luma in double, rounded to
// fp32; RGBA alpha == 0 marks a pixel invalid: src/image.cpp:16-43).
// The reference's inline sample_bilinear / sample_plane_bilinear
// (inc/image.hpp:53-90) are internals of the matcher, evaluated on the
// device here, and are not re-exported.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "gpu_runtime.hpp"

namespace pstereo {

struct Raster {
  int width = 0;
  int height = 0;
  int channels = 0;                  // 1 gray, 3 RGB, 4 RGBA
  std::vector<std::uint8_t> pixels;  // row-major, interleaved
};

struct GrayImage {
  int width = 0;
  int height = 0;
  std::vector<float> data;          // row-major
  std::vector<std::uint8_t> valid;  // 1 = usable

  float at(int x, int y) const { return data[std::size_t(y) * std::size_t(width) + x]; }
  float& at(int x, int y) { return data[std::size_t(y) * std::size_t(width) + x]; }
  bool valid_at(int x, int y) const {
    return valid[std::size_t(y) * std::size_t(width) + x] != 0;
  }
  bool in_bounds(double x, double y) const {
    return x >= 0.0 && x <= width - 1.0 && y >= 0.0 && y <= height - 1.0;
  }
};

inline GrayImage make_gray(int width, int height, float fill = 0.0f, bool valid = true) {
  GrayImage img;
  img.width = width;
  img.height = height;
  img.data.assign(std::size_t(width) * std::size_t(height), fill);
  img.valid.assign(std::size_t(width) * std::size_t(height), valid ? 1 : 0);
  return img;
}

inline GrayImage to_grayscale(const Raster& raster) {
  if (raster.channels != 1 && raster.channels != 3 && raster.channels != 4)
    throw std::invalid_argument("to_grayscale: unsupported channel count " +
                                std::to_string(raster.channels));
  GrayImage img = make_gray(raster.width, raster.height);
  if (img.data.empty()) return img;
  const int rc = pstereo_gpu_to_grayscale(gpu::device(), raster.width, raster.height,
                                          raster.channels, raster.pixels.data(), img.data.data(),
                                          img.valid.data());
  if (rc != PSTEREO_OK) gpu::detail::raise(rc, "to_grayscale failed on the device");
  return img;
}

}  // namespace pstereo
