// image.hpp for the oracle build — TEST INFRASTRUCTURE ONLY.
//
// The reference's image.cpp needs OpenCV (imgcodecs), absent from this image,
// for its PNG I/O. The oracle build links dataset.cpp / eval.cpp (for
// synth_from_grid, evaluate_map_quality and the metrics) against this file
// instead: the PNG functions throw (file I/O is out of scope), and
// the two quantisers restate image.cpp:13-30 (round half-up to 8-bit colour /
// 16-bit depth units, clamped; invalid depth stays 0).
#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "voxrf/image.hpp"

namespace voxrf {

double quantize_color(double v) {
  const double scaled = std::floor(v * 255.0 + 0.5);
  return double(int(std::clamp(scaled, 0.0, 255.0))) / 255.0;
}

double quantize_depth(double meters, double depth_scale) {
  if (!(meters > 0.0)) return 0.0;
  const double units = std::floor(meters * depth_scale + 0.5);
  return int(std::clamp(units, 0.0, 65535.0)) / depth_scale;
}

static void no_png(const char* what) {
  throw std::runtime_error(std::string(what) + ": PNG I/O is not part of the oracle build");
}
void write_color_png(const std::filesystem::path&, const ImageF&) { no_png("write_color_png"); }
ImageF read_color_png(const std::filesystem::path&) {
  no_png("read_color_png");
  return {};
}
void write_depth_png(const std::filesystem::path&, const ImageF&, double) {
  no_png("write_depth_png");
}
ImageF read_depth_png(const std::filesystem::path&, double) {
  no_png("read_depth_png");
  return {};
}

}  // namespace voxrf
